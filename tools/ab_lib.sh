#!/bin/bash
# A/B of two builds of libsphb200.so on the same box: tools/prof_c3.py 3 10 alternately
for i in 1 2 3; do
  SPH_LIB_PATH=paper_2604_12505_b200/libsphb200_base.so python tools/prof_c3.py 3 10 >> gpurun_out/ab_base.log 2>&1
  python tools/prof_c3.py 3 10 >> gpurun_out/ab_new.log 2>&1
done
