#!/bin/bash
# ncu --set full of chosen GEMM launches in one bench step (1 GPU).
# usage: bash scripts/gpu_ncu_kernel.sh TAG "regex on demangled name" [skip] [count]
TAG=$1; RE=$2; SKIP=${3:-2}; CNT=${4:-1}
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:$RE" -s $SKIP -c $CNT \
  -o gpurun_out/prof_$TAG python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_$TAG.log 2>&1
echo "ncu_exit=$?"; grep -E "PROF|WARN|ERR" gpurun_out/ncu_$TAG.log | tail -3
