#!/bin/bash
# usage: sweep_build.sh "<nvcc extra flags>|<bench args>" ...   (rebuilds per variant)
# env RUNENV="A=1 B=2" is applied to every bench run.
cd "$(dirname "$0")/.."
for spec in "$@"; do
  flags="${spec%%|*}"; args="${spec#*|}"
  echo "== flags[$flags] args[$args]"
  SPH_NVCC_EXTRA="$flags" python -c "from paper_2604_12505_b200 import build; build.build(force=True)" || { echo build failed; continue; }
  grep -A3 "7k_forceENS" paper_2604_12505_b200/csrc/ptxas_info.txt | grep -E "Used|spill" | tr '\n' ' '; echo
  env $RUNENV timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline $args 2>&1 | tail -1 | python -c "
import sys,json
l=sys.stdin.read().strip()
try:
  d=json.loads(l); r=d['roofline']
  print('value %.3e' % d['value'], 'chk %.9e' % d['config'].get('y_checksum',0), 'reb/sub %.1f' % d['config']['substeps_per_rebuild'],
        'live', {k: round(v*1e3,1) for k,v in r['live_ms'].items()}, 'isolated', {k: round(v*1e3,1) for k,v in r['isolated_ms'].items()})
except Exception as e: print('ERR', l[-800:])
"
done
python -c "from paper_2604_12505_b200 import build; build.build(force=True)"
