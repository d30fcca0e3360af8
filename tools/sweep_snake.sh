# A/B of the snake rollout order of k_force (SPH_SNAKE=1) on C3, plus parity with it on
run() {
  lbl=$1; shift
  env "$@" timeout 200 python bench.py --no-cpu-baseline 2>/dev/null | grep "^{" | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$lbl', round(d['value']/1e9,3), d['config']['y_checksum'], {k: round(v*1000,1) for k,v in d['roofline']['live_ms'].items()})" >> gpurun_out/snake.log 2>&1
}
for r in 1 2 3; do
run base X=1
run snake SPH_SNAKE=1
done
SPH_SNAKE=1 timeout 600 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/snake_parity.log 2>&1; echo rc=$? >> gpurun_out/snake_parity.log
