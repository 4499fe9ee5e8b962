#!/bin/bash
# Full round: smoke + GPU tests + bench (N=1) + EP path at one rank + reference arm + ncu list + ncu full.
TAG=${1:-r}
bash scripts/gpu_check.sh $TAG tests bench ncu full
timeout 600 python bench.py --ep --steps 10 --warmup 3 > gpurun_out/bench_${TAG}_ep1.json 2> gpurun_out/bench_${TAG}_ep1.err
echo "ep1_exit=$?"; tail -2 gpurun_out/bench_${TAG}_ep1.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_${TAG}_ref.json 2>&1
echo "ref_exit=$?"
nproc > gpurun_out/host_${TAG}.txt; lscpu | grep "Model name" >> gpurun_out/host_${TAG}.txt
