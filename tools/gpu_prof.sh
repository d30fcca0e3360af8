#!/bin/bash
# ncu captures (run only after the same command exited 0 in this call).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
TAG=${TAG:-r01}
CMD="python tools/prof_kernels.py ${PROF_ARGS}"
$CMD > gpurun_out/prof_plain_${TAG}.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_force|k_density" -s 6 -c 2 \
    -o gpurun_out/prof_${TAG} -f $CMD > gpurun_out/ncu_${TAG}.log 2>&1
echo "ncu exit $?"; tail -3 gpurun_out/ncu_${TAG}.log
