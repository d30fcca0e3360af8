#!/bin/bash
for cfg in ${CFGS:-"0.15 0.8 1"}; do
  set -- $cfg
  timeout -s KILL 900 python bench.py --workload C4 --no-cpu-baseline --steps 3 --warmup 1 --skin $1 --skin-max $2 --skin-mode $3 > gpurun_out/c4_$1_$2_$3.json 2> gpurun_out/c4_$1_$2_$3.err
done
