#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo "exit $?" >> gpurun_out/smoke.log
timeout -s KILL 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gputest_final.log 2>&1; echo "exit $?" >> gpurun_out/gputest_final.log
timeout -s KILL 900 python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err
timeout -s KILL 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout -s KILL 1500 python bench.py --long-horizon > gpurun_out/horizon_final.json 2> gpurun_out/horizon_final.err
python tools/prof_c3.py 2 1 > gpurun_out/plain_c3.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:"k_force|k_density" -s 900 -c 4 -o gpurun_out/c3_full python tools/prof_c3.py 2 1 > gpurun_out/ncu_c3.log 2>&1
