# A/B of the warp-persistent density / force kernels (SPH_WP bit 0 / bit 1; bit 2 = no L2 prefetch) on C3
run() {
  lbl=$1; shift
  env "$@" timeout 200 python bench.py --no-cpu-baseline 2>/dev/null | grep "^{" | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$lbl', round(d['value']/1e9,3), d['config']['y_checksum'], {k: round(v*1000,1) for k,v in d['roofline']['live_ms'].items()})" >> gpurun_out/wp2.log 2>&1
}
for r in 1 2; do
run base X=1
run wp1 SPH_WP=1
run wp5 SPH_WP=5
run wp6 SPH_WP=6
done
