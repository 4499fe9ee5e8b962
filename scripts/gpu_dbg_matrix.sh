#!/bin/bash
# Bottleneck matrix of the tcgen05 GEMMs with the runtime experiment knobs
# (MOE_GEMM_DBG bits: 1 = no epilogue work, 2 = no MMA, 4 = no activation,
# 8 = no TMA operand loads). Outputs are garbage under a knob; only the
# per-kernel times of the bench breakdown are read.
# usage (under gpurun): bash scripts/gpu_dbg_matrix.sh TAG [bits ...]
TAG=${1:-x}
shift
BITS="${@:-0 1 2 4 8 3 9 10}"
mkdir -p gpurun_out
for b in $BITS; do
  MOE_GEMM_DBG=$b timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/dbg_${TAG}_$b.json 2>/dev/null
  python - "$TAG" "$b" <<'PY'
import json, sys
try:
    d = json.load(open(f"gpurun_out/dbg_{sys.argv[1]}_{sys.argv[2]}.json"))
    print("dbg", sys.argv[2], round(d["ms_per_step"], 4), " ".join(f"{k}={v['ms']*1000:.1f}" for k, v in d["breakdown_ms"].items()))
except Exception as e:
    print("dbg", sys.argv[2], "failed", e)
PY
done
