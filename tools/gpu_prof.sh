#!/bin/bash
# ncu captures (run only after the same command exited 0 in this call).
# prof_kernels.py: 200 settle substeps (1 rollout) then the C3 context: substep 1 rebuilds,
# substeps 2.. are steady-state -> skip 200 settle launches of each profiled kernel + 2 substeps.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
TAG=${TAG:-r01}
CMD="python tools/prof_kernels.py --settle-steps 200 --substeps 6 ${PROF_ARGS}"
$CMD > gpurun_out/prof_plain_${TAG}.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_force|k_density" -s 404 -c 2 \
    -o gpurun_out/prof_${TAG} -f $CMD > gpurun_out/ncu_${TAG}.log 2>&1
echo "ncu exit $?"; tail -3 gpurun_out/ncu_${TAG}.log
