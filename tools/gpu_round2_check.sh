#!/bin/bash
# GPU tests + sanitizers + a bench line (one gpurun call)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gputest.log 2>&1
echo "pytest exit $?" >> gpurun_out/gputest.log
for tool in memcheck synccheck racecheck; do
  timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 python tools/sanitize.py ${SAN_SCEN:-coop_c1 kernels_multikernel_c1 kernels_small_c1 kernels_small_c2} > gpurun_out/san_$tool.log 2>&1
  echo "exit $?" >> gpurun_out/san_$tool.log
done
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err
