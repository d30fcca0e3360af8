#!/bin/bash
# steady-state rate vs Verlet skin over the first 600 ticks (30 s) of the C3 train
for sk in ${SKINS:-0.15 0.25 0.35 0.5}; do
  timeout -s KILL 900 python bench.py --long-horizon --horizon-ticks 600 --skin $sk > gpurun_out/hz_$sk.json 2> gpurun_out/hz_$sk.err
done
