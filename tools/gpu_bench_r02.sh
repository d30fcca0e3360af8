#!/bin/bash
mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests/test_gpu_ensemble.py -q -x -p no:cacheprovider > gpurun_out/ens_test.log 2>&1; echo "exit $?" >> gpurun_out/ens_test.log
timeout -s KILL 600 python bench.py --no-cpu-baseline > gpurun_out/b_c3_w0.json 2> gpurun_out/b_c3_w0.err
timeout -s KILL 600 python bench.py --no-cpu-baseline --window-start 1000 > gpurun_out/b_c3_w1000.json 2> gpurun_out/b_c3_w1000.err
timeout -s KILL 900 python bench.py --no-cpu-baseline --workload C5 --scaling strong > gpurun_out/b_c5.json 2> gpurun_out/b_c5.err
timeout -s KILL 1200 python bench.py --long-horizon > gpurun_out/horizon.json 2> gpurun_out/horizon.err
