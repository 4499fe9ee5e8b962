#!/bin/bash
# A/B the GEMM pipeline parts: MOE_GEMM_DBG = 0 (normal), 1 (no epilogue work), 2 (no MMA), 4 (no act math)
mkdir -p gpurun_out; TAG=${1:-dbg}; shift
for d in ${@:-0 1 2 3 4}; do
  MOE_GEMM_DBG=$d timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_${TAG}_$d.json 2> gpurun_out/bench_${TAG}_$d.err
  echo "dbg=$d exit=$?"
done
