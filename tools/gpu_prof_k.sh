#!/bin/bash
# ncu full capture of kernels matching $KREGEX (after a plain run of the same command).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
TAG=${TAG:-rk}
CMD="python tools/prof_kernels.py --settle-steps ${SETTLE:-200} --substeps ${SUBSTEPS:-6} ${PROF_ARGS}"
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
$CMD > gpurun_out/prof_plain_${TAG}.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"${KREGEX}" -s ${SKIP:-0} -c ${COUNT:-1} \
    -o gpurun_out/prof_${TAG} -f $CMD > gpurun_out/ncu_${TAG}.log 2>&1
echo "ncu exit $?"; tail -2 gpurun_out/ncu_${TAG}.log
