#!/usr/bin/env bash
# ncu evidence for profiles/: launch list of the captured Sum-15 step (in-step, warm L2 as
# in the real run) and one --set full capture of each hot kernel.
set -u
mkdir -p gpurun_out
TAG=${TAG:-r01}
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  --cache-control none --csv --log-file gpurun_out/${TAG}_step_launches.csv \
  python bench.py --quick --steps 2 --warmup 1 > gpurun_out/${TAG}_ncu_quick.out 2>&1; echo "launches rc=$?"
# --set full of one launch of each hot kernel inside the captured Sum-15 step (B=16384);
# default cache control (flushed before the launch): the cold per-launch roofline case
for KS in k_chain_bwd:4 k_chain_fwd:4 k_nll_fwd_given:4 k_nll_bwd:4; do
  K=${KS%%:*}; S=${KS##*:}
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:$K -s $S -c 1 \
    -o gpurun_out/${TAG}_full_$K -f python bench.py --quick --steps 2 --warmup 1 > gpurun_out/${TAG}_ncu_$K.out 2>&1
  echo "$K rc=$?"
done
timeout 400 ncu --set full --clock-control none --import-source on -k regex:k_dtkp_apply -s 30 -c 2 \
  -o gpurun_out/${TAG}_full_k_dtkp_apply -f python tools/bench_configs.py --only hwf7 --iters 2 > gpurun_out/${TAG}_ncu_dtkp.out 2>&1
echo "dtkp rc=$?"
