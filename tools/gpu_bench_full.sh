#!/bin/bash
# Full default bench line + reference arm + ncu launch list of the same bench command
# (launches of the timed region only: NVTX range "timed").
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
TAG=${TAG:-r01}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo BUILD FAILED; exit 1; }
python bench.py $BENCH_ARGS > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err; echo "bench exit $?"; tail -1 gpurun_out/bench_${TAG}.json | cut -c1-600
if [ -z "$NO_REF" ]; then
python bench.py --impl reference > gpurun_out/bench_ref_${TAG}.json 2> gpurun_out/bench_ref_${TAG}.err; echo "ref exit $?"; tail -1 gpurun_out/bench_ref_${TAG}.json | cut -c1-400
fi
if [ -n "$LAUNCHES" ]; then
python bench.py --no-cpu-baseline --steps 2 > gpurun_out/bench_plain_${TAG}.json 2>&1 && \
ncu --nvtx --nvtx-include "timed/" --metrics gpu__time_duration.sum --clock-control none -c ${LAUNCHES} --csv \
    --log-file gpurun_out/launches_${TAG}.csv python bench.py --no-cpu-baseline --steps 2 > gpurun_out/ncu_bench_${TAG}.log 2>&1
echo "ncu exit $?"
fi
