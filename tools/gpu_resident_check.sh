#!/bin/bash
# resident-path tests (short timeouts: a cluster-barrier deadlock must not hang the box)
mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests/test_gpu_resident.py -q -x -p no:cacheprovider ${RES_K:+-k "$RES_K"} > gpurun_out/res_test.log 2>&1
echo "pytest exit $?" >> gpurun_out/res_test.log
