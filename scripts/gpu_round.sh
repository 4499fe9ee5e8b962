#!/bin/bash
# Full round: smoke + GPU tests + bench (N=1) + ncu list + ncu full, the EP path at one rank
# (p2p and NCCL transports), the reference arm, the product sweep.
TAG=${1:-r}
bash scripts/gpu_check.sh $TAG tests bench ncu full perm
for t in p2p nccl; do
  timeout 600 python bench.py --ep --transport $t --steps 20 --warmup 5 > gpurun_out/bench_${TAG}_ep1_$t.json 2> gpurun_out/bench_${TAG}_ep1_$t.err
  echo "ep1_${t}_exit=$?"; tail -2 gpurun_out/bench_${TAG}_ep1_$t.err
done
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_${TAG}_ref.json 2>&1
echo "ref_exit=$?"
timeout 600 python scripts/product_sweep.py --out gpurun_out/sweep_${TAG}.json > gpurun_out/sweep_${TAG}.log 2>&1
echo "sweep_exit=$?"
nproc > gpurun_out/host_${TAG}.txt; lscpu | grep "Model name" >> gpurun_out/host_${TAG}.txt
timeout 300 python scripts/micro/hbm_rw.py > gpurun_out/hbm_rw_${TAG}.txt 2>&1
