#!/usr/bin/env bash
# r02e GPU session: parity, chain-bwd prefetch A/B, DTKP key A/B, launch lists, ncu issue captures.
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest -q -m gpu tests > gpurun_out/t_all.log 2>&1; tail -2 gpurun_out/t_all.log
for v in main nopf main nopf; do
  if [ $v = main ]; then L=; else L=ab_$v/libsgb200.so; fi
  echo "== $v" >> gpurun_out/pf.log
  SGB200_LIB=$L timeout 300 python tools/chain_bench.py --batch 16384 >> gpurun_out/pf.log 2>&1
  SGB200_LIB=$L timeout 300 python bench.py --no-configs --no-train --no-cpu-baseline --steps 30 --warmup 5 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('step_ms', d['ms_per_step'], 'bwd_us', d['roofline']['avg_launch_us'])" >> gpurun_out/pf.log 2>&1
done
for v in main old main; do
  if [ $v = main ]; then L=; else L=ab_$v/libsgb200.so; fi
  echo "== $v" >> gpurun_out/ab.log
  SGB200_LIB=$L timeout 300 python tools/bench_configs.py --only hwf7,clutrr --no-cpu >> gpurun_out/ab.log 2>&1
done
M="--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,launch__registers_per_thread,launch__grid_size --clock-control none --csv"
timeout 300 ncu --nvtx --nvtx-include "step/" $M --log-file gpurun_out/launches_hwf_r02e.csv python tools/probes/dtkp_step.py hwf > /dev/null 2>&1
timeout 300 ncu --nvtx --nvtx-include "step/" $M --log-file gpurun_out/launches_clutrr_r02e.csv python tools/probes/dtkp_step.py clutrr > /dev/null 2>&1
timeout 600 ncu --set full --import-source on --clock-control none --nvtx --nvtx-include "step/" -k regex:k_dtkp_apply --launch-skip 6 --launch-count 2 -o gpurun_out/hwf_r02e -f python tools/probes/dtkp_step.py hwf > gpurun_out/ncu_hwf_r02e.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none --nvtx --nvtx-include "step/" -k regex:k_dtkp_apply --launch-skip 6 --launch-count 2 -o gpurun_out/clutrr_r02e -f python tools/probes/dtkp_step.py clutrr > gpurun_out/ncu_clutrr_r02e.log 2>&1
echo session done
