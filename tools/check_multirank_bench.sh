#!/bin/bash
# Control-flow check of bench.py's multi-rank path on a 1-GPU box: 2 ranks on device 0 with gloo
# collectives (barrier, max-reduction of the timings, trajectory gather).  Not a measurement.
cd "$(dirname "$0")/.."
BENCH_SINGLE_DEVICE_CHECK=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
    --master-addr 127.0.0.1 --master-port 29555 bench.py --gpus 2 --steps 2 --warmup 3 --rollouts 64 \
    --no-cpu-baseline
echo "multi-rank bench exit $?"
BENCH_SINGLE_DEVICE_CHECK=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
    --master-addr 127.0.0.1 --master-port 29556 bench.py --impl reference --gpus 2 --steps 1 --warmup 0
echo "multi-rank reference exit $?"
BENCH_SINGLE_DEVICE_CHECK=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
    --master-addr 127.0.0.1 --master-port 29557 bench.py --workload C4DD --gpus 2 --steps 1 --warmup 1
echo "multi-rank C4DD exit $?"
