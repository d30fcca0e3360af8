#!/bin/bash
# Phase stamps of the resident path (diagnostic builds abso/<v>_t.so, -DSPH_RES_TIMING) on C2
for v in ${VARIANTS:-new}; do
  rm -f gpurun_out/rt_$v.bin
  SPH_LIB_PATH=abso/${v}_t.so SPH_RES_TIMING_FILE=gpurun_out/rt_$v.bin timeout -s KILL 600 \
    python bench.py --workload ${WL:-C2} --no-cpu-baseline --steps 3 --warmup 3 > gpurun_out/rt_$v.json 2>&1
  echo "== $v"; python tools/res_phases.py gpurun_out/rt_$v.bin
done
