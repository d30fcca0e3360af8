#!/bin/bash
# parameter sweep of the bench (device value only).  Each argument: "ENV=.. ENV2=..|bench args"
# (either side may be empty), e.g. "SPH_RING=0|--steps 10" or "|--skin 0.2".
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
for spec in "$@"; do
  envs="${spec%%|*}"; args="${spec#*|}"
  [ "$envs" == "$spec" ] && { envs=""; args="$spec"; }
  echo "== env[$envs] args[$args]"
  env $envs timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline $args 2>&1 | tail -1 | python -c "
import sys,json
l=sys.stdin.read().strip()
try:
  d=json.loads(l); r=d['roofline']
  print('value %.3e' % d['value'], 'chk %.9e' % d['config'].get('y_checksum',0), 'reb/sub %.1f' % d['config']['substeps_per_rebuild'],
        'live', {k: (round(v*1e3,1) if v is not None else None) for k,v in r['live_ms'].items()}, 'isolated', {k: round(v*1e3,1) for k,v in r['isolated_ms'].items()}, 'ms/step %.3f' % d['ms_per_step'], 'frac %.3f' % r['frac'])
except Exception as e: print('ERR', l[-800:])
"
done
