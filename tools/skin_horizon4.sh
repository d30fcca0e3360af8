#!/bin/bash
#timeout -s KILL 1200 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/gputest3.log 2>&1; echo "exit $?" >> gpurun_out/gputest3.log
for cfg in "0.15 0.5" "0.15 0.8" "0.15 1.0" "0.1 0.8"; do
  set -- $cfg
  timeout -s KILL 900 python bench.py --long-horizon --horizon-ticks 400 --skin $1 --skin-max $2 > gpurun_out/hz4_$1_$2.json 2> gpurun_out/hz4_$1_$2.err
done
