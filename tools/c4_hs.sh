#!/bin/bash
for v in base 20 40; do
  if [ $v = base ]; then L=paper_2604_12505_b200/libsphb200.so; else L=paper_2604_12505_b200/libsphb200_hs$v.so; fi
  SPH_LIB_PATH=$L timeout -s KILL 900 python bench.py --workload C4 --no-cpu-baseline --steps 3 --warmup 1 > gpurun_out/c4hs_$v.json 2> gpurun_out/c4hs_$v.err
done
