# SM clock / power / throttle reasons sampled every 20 ms during the default bench and during a
# run with the warp-persistent density kernel (SPH_WP=5), to test the power-headroom hypothesis
for v in base 5; do
  nvidia-smi --query-gpu=timestamp,clocks.sm,clocks.mem,power.draw,clocks_throttle_reasons.active --format=csv,noheader -lms 20 > gpurun_out/power_$v.csv &
  P=$!
  if [ $v = base ]; then python bench.py --no-cpu-baseline > gpurun_out/power_bench_$v.json 2>/dev/null
  else SPH_WP=$v python bench.py --no-cpu-baseline > gpurun_out/power_bench_$v.json 2>/dev/null; fi
  kill $P
done
