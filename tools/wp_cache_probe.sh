# Launch lists (one metric pass, --cache-control none: L2 state kept between launches) of the
# C3 timed region with the grid density kernel and with k_density_wp (SPH_WP=5)
for v in 0 5; do
  SPH_WP=$v ncu --nvtx --nvtx-include "timed/" --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
      --clock-control none --cache-control none -c 1401 --csv --log-file gpurun_out/wpcache_$v.csv \
      python bench.py --no-cpu-baseline --steps 1 > gpurun_out/wpcache_$v.log 2>&1
  echo "wp=$v ncu exit $?"
done
