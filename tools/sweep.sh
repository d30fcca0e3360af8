#!/bin/bash
# parameter sweep of the bench (device value only)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
for args in "$@"; do
  echo "== $args"
  timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline $args 2>&1 | tail -1 | python -c "
import sys,json
l=sys.stdin.read().strip()
try:
  d=json.loads(l); r=d['roofline']
  print('value %.3e' % d['value'], 'chk %.9e' % d['config'].get('y_checksum',0), 'reb/sub %.1f' % d['config']['substeps_per_rebuild'], {k: round(v*1e3,1) for k,v in r['kernel_ms_all'].items()}, 'sub_us', round(r['substep_ms_profiled']*1e3,1))
except Exception as e: print('ERR', l[-500:])
"
done
