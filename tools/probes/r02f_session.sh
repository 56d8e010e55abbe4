#!/usr/bin/env bash
# r02f GPU session: parity, key-scan A/B (dual vs 32-bit only), adaptive item size, launch lists.
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest -q -m gpu tests > gpurun_out/t_all.log 2>&1; tail -2 gpurun_out/t_all.log
for v in main k32 main k32; do
  if [ $v = main ]; then L=; else L=ab_$v/libsgb200.so; fi
  echo "== $v" >> gpurun_out/ab.log
  SGB200_LIB=$L timeout 300 python tools/bench_configs.py --only hwf7,clutrr --no-cpu >> gpurun_out/ab.log 2>&1
done
M="--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,launch__registers_per_thread,launch__grid_size --clock-control none --csv"
timeout 300 ncu --nvtx --nvtx-include "step/" $M --log-file gpurun_out/launches_hwf_r02f.csv python tools/probes/dtkp_step.py hwf > /dev/null 2>&1
timeout 300 ncu --nvtx --nvtx-include "step/" $M --log-file gpurun_out/launches_clutrr_r02f.csv python tools/probes/dtkp_step.py clutrr > /dev/null 2>&1
echo session done
