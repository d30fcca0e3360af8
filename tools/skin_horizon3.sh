#!/bin/bash
timeout -s KILL 1200 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/gputest2.log 2>&1; echo "exit $?" >> gpurun_out/gputest2.log
for cfg in "0.15 0.5" "0.15 0.7" "0.2 0.5"; do
  set -- $cfg
  timeout -s KILL 900 python bench.py --long-horizon --horizon-ticks 400 --skin $1 --skin-max $2 > gpurun_out/hz3_$1_$2.json 2> gpurun_out/hz3_$1_$2.err
done
