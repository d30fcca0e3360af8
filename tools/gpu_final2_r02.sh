#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo "exit $?" >> gpurun_out/smoke.log
timeout -s KILL 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gputest_final.log 2>&1; echo "exit $?" >> gpurun_out/gputest_final.log
for i in 1 2; do timeout -s KILL 900 python bench.py --no-cpu-baseline > gpurun_out/bench_rep_$i.json 2> gpurun_out/bench_rep_$i.err; done
timeout -s KILL 900 python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err
