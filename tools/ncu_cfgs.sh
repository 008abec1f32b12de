set -x
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed,sm__warps_active.avg.pct_of_peak_sustained_active,launch__registers_per_thread,launch__grid_size
for c in c4 c2s c2c c5; do
  timeout 300 ncu --metrics $M --clock-control none --csv --log-file gpurun_out/ncu_$c.csv python tools/profile_target.py $c 6 > gpurun_out/ncu_$c.log 2>&1
done
