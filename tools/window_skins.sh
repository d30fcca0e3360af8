#!/bin/bash
for cfg in "0.15 0" "0.5 0" "0.15 0.5" "0.15 0.35"; do
  set -- $cfg
  timeout -s KILL 900 python bench.py --no-cpu-baseline --skin $1 --skin-max $2 > gpurun_out/win_$1_$2.json 2> gpurun_out/win_$1_$2.err
done
