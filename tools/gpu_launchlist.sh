#!/bin/bash
# ncu launch list (gpu__time_duration per launch) of the profiling driver, summarised.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
TAG=${TAG:-ll}
CMD="python tools/prof_kernels.py --settle-steps ${SETTLE:-50} --substeps ${SUBSTEPS:-40} ${PROF_ARGS}"
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
$CMD > gpurun_out/ll_plain_${TAG}.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -s ${SKIP:-0} --csv \
    --log-file gpurun_out/ll_${TAG}.csv $CMD > gpurun_out/ll_ncu_${TAG}.log 2>&1
echo "ncu exit $?"
