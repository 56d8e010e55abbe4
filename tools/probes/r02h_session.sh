#!/usr/bin/env bash
# r02h: first-fill fast path A/B (HWF), keyed K=5 conj A/B (CLUTRR), parity.
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest -q -m gpu tests > gpurun_out/t_all.log 2>&1; tail -2 gpurun_out/t_all.log
for v in main nofill k5 main nofill k5; do
  if [ $v = main ]; then L=; else L=ab_$v/libsgb200.so; fi
  echo "== $v" >> gpurun_out/ab.log
  SGB200_LIB=$L timeout 300 python tools/bench_configs.py --only hwf7,clutrr --no-cpu >> gpurun_out/ab.log 2>&1
done
SGB200_LIB=ab_k5/libsgb200.so timeout 600 python -m pytest -q -m gpu tests/test_gpu_golden.py tests/test_gpu_full_size.py tests/test_fixpoint.py 2>&1 | tail -1
echo session done
