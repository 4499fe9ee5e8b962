#!/bin/bash
# Bottleneck matrix of the CTA-pair SDD / SDD^T under MOE_GEMM_DBG knobs (timing only; outputs are garbage):
# 1 no epilogue, 2 no MMA, 4 no activation math, 8 no operand loads, 16 no epilogue stores.
mkdir -p gpurun_out; TAG=${1:-dbg}; shift
for d in ${@:-0 1 2 4 8 16 20 10 26}; do
  MOE_GEMM_DBG=$d timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e $BENCH_FLAGS > gpurun_out/dbg_${TAG}_$d.json 2>/dev/null
  python - "$TAG" "$d" <<'PY'
import json, sys
try:
    b = json.load(open(f"gpurun_out/dbg_{sys.argv[1]}_{sys.argv[2]}.json"))["breakdown_ms"]
    print(f"dbg {sys.argv[2]:>3}: " + " ".join(f"{k}={b[k]['ms']*1000:.1f}" for k in ("sdd", "dsd+scatter", "sddT", "dsTd", "ddTs", "dsdT+dx") if k in b))
except Exception as e:
    print("dbg", sys.argv[2], "failed", e)
PY
done
