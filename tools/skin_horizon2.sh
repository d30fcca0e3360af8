#!/bin/bash
for cfg in "0.5 2" "0.7 0" "0.3 2" "0.15 2"; do
  set -- $cfg
  timeout -s KILL 900 python bench.py --long-horizon --horizon-ticks 400 --skin $1 --rebuild-path $2 > gpurun_out/hz2_$1_$2.json 2> gpurun_out/hz2_$1_$2.err
done
