#!/usr/bin/env bash
# One GPU session: parity tests, bench line, ncu launch list and one full capture of the
# dominant kernel.  Everything lands in gpurun_out/ (merged back by gpurun).
set -u
mkdir -p gpurun_out
TAG=${TAG:-r01}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/${TAG}_smi.txt 2>&1
if [ "${SKIP_TESTS:-0}" != "1" ]; then
  timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_pytest_gpu.txt 2>&1
  echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest_gpu.txt
  tail -3 gpurun_out/${TAG}_pytest_gpu.txt
fi
timeout 900 python bench.py ${BENCH_ARGS:-} > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
echo "bench rc=$?"; tail -c 3000 gpurun_out/${TAG}_bench.json; tail -5 gpurun_out/${TAG}_bench.err
if [ "${SKIP_NCU:-0}" != "1" ]; then
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file gpurun_out/${TAG}_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline \
      > gpurun_out/${TAG}_ncu_bench.out 2>&1
  echo "ncu launches rc=$?"
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:${NCU_KERNEL:-k_conv_bwd} -s ${NCU_SKIP:-20} -c ${NCU_COUNT:-2} \
      -o gpurun_out/${TAG}_full -f python bench.py --steps 2 --warmup 1 --no-cpu-baseline \
      > gpurun_out/${TAG}_ncu_full.out 2>&1
  echo "ncu full rc=$?"
fi
