#!/bin/bash
# A/B of library builds abso/<v>.so on the latency workloads, alternating on one box
#   VARIANTS="old new" WLS="C2 C2CL P0" STEPS=5 bash tools/ab_latency.sh
for i in 1 2; do
  for v in ${VARIANTS:-old new}; do
    for w in ${WLS:-C2 C2CL P0}; do
      SPH_LIB_PATH=abso/$v.so timeout -s KILL 600 python bench.py --workload $w --no-cpu-baseline --steps ${STEPS:-5} \
        > gpurun_out/ab_${v}_${w}_$i.json 2> gpurun_out/ab_${v}_${w}_$i.err
    done
  done
done
python - <<'P'
import json, glob
for f in sorted(glob.glob("gpurun_out/ab_*_*_*.json")):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
        print(f, round(d["ms_per_step"], 4), d["clocks"]["sm_mhz"], d["clocks"]["reasons"])
    except Exception as e:
        print(f, "ERR", e)
P
