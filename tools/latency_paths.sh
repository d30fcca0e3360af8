#!/bin/bash
# latency-bound single tanks: cooperative tick (default) vs resident clusters
for ex in ${EXS:-0 3}; do
  timeout -s KILL 600 python bench.py --workload C2 --no-cpu-baseline --exec-path $ex > gpurun_out/lat_c2_$ex.json 2> gpurun_out/lat_c2_$ex.err
  timeout -s KILL 600 python bench.py --workload C1 --no-cpu-baseline --exec-path $ex > gpurun_out/lat_c1_$ex.json 2> gpurun_out/lat_c1_$ex.err
  timeout -s KILL 900 python bench.py --workload P0 --exec-path $ex > gpurun_out/lat_p0_$ex.json 2> gpurun_out/lat_p0_$ex.err
  timeout -s KILL 900 python bench.py --workload C2CL --exec-path $ex > gpurun_out/lat_c2cl_$ex.json 2> gpurun_out/lat_c2cl_$ex.err
done
