set -u
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --cache-control none --csv \
  --log-file gpurun_out/r01_step_launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r01_step_ncu.out 2>&1
echo "rc=$?"
