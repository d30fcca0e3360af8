# A/B: rebuild branch (side stream) at the highest stream priority (SPH_SIDE_PRIO=1) on C3
run() {
  lbl=$1; shift
  env "$@" timeout 200 python bench.py --no-cpu-baseline 2>/dev/null | grep "^{" | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$lbl', round(d['value']/1e9,3), d['config']['y_checksum'], {k: round(v*1000,1) for k,v in d['roofline']['live_ms'].items()})" >> gpurun_out/prio.log 2>&1
}
for r in 1 2 3; do
run base X=1
run prio SPH_SIDE_PRIO=1
done
