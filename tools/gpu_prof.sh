#!/bin/bash
# ncu captures (run only after the same command exited 0 in this call).
# prof_kernels.py: the bench's settled snapshot, the C3 context at the bench's skin, then direct
# substeps (k_density + two k_force launches each): skip 3 substeps, capture one substep's three.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
TAG=${TAG:-r01}
CMD="python tools/prof_kernels.py --settle-steps -1 --skin 0.15 --substeps 6 ${PROF_ARGS}"
$CMD > gpurun_out/prof_plain_${TAG}.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_force|k_density" -s 9 -c 3 \
    -o gpurun_out/prof_${TAG} -f $CMD > gpurun_out/ncu_${TAG}.log 2>&1
echo "ncu exit $?"; tail -3 gpurun_out/ncu_${TAG}.log
