#!/usr/bin/env bash
# Final round-2 session: parity, smoke, full bench line, reference arm, launch lists.
set -u
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/r02i_smi.txt 2>&1
timeout 900 python -m pytest -q -m gpu tests > gpurun_out/r02i_pytest_gpu.txt 2>&1; tail -2 gpurun_out/r02i_pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r02i_smoke.txt 2>&1; tail -1 gpurun_out/r02i_smoke.txt
timeout 900 python bench.py > gpurun_out/r02i_bench.json 2> gpurun_out/r02i_bench.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r02i_reference_arm.json 2> gpurun_out/r02i_ref.err; echo "ref rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02i_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-configs --no-train > gpurun_out/r02i_ncu_bench.out 2>&1; echo "ncu rc=$?"
M="--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,launch__registers_per_thread,launch__grid_size --clock-control none --csv"
timeout 300 ncu --nvtx --nvtx-include "step/" $M --log-file gpurun_out/launches_hwf_r02i.csv python tools/probes/dtkp_step.py hwf > /dev/null 2>&1
timeout 300 ncu --nvtx --nvtx-include "step/" $M --log-file gpurun_out/launches_clutrr_r02i.csv python tools/probes/dtkp_step.py clutrr > /dev/null 2>&1
timeout 600 ncu --set full --import-source on --clock-control none --nvtx --nvtx-include "step/" -k regex:k_dtkp_apply --launch-skip 8 --launch-count 2 -o gpurun_out/hwf_r02i -f python tools/probes/dtkp_step.py hwf > gpurun_out/ncu_hwf_r02i.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none --nvtx --nvtx-include "step/" -k regex:k_dtkp_apply --launch-skip 6 --launch-count 2 -o gpurun_out/clutrr_r02i -f python tools/probes/dtkp_step.py clutrr > gpurun_out/ncu_clutrr_r02i.log 2>&1
echo session done
