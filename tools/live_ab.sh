#!/bin/bash
for i in 1 2; do
timeout -s KILL 600 python bench.py --no-cpu-baseline > gpurun_out/ab_live_$i.json 2>/dev/null
timeout -s KILL 600 python bench.py --no-cpu-baseline --live-every 0 > gpurun_out/ab_nolive_$i.json 2>/dev/null
done
python tools/prof_c3.py 3 10 > gpurun_out/ab_prof.log 2>&1
