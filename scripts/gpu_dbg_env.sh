#!/bin/bash
# dbg matrix under an extra environment: bash scripts/gpu_dbg_env.sh TAG "ENV=1 ENV2=2" bits...
TAG=$1; ENVS=$2; shift 2
for b in "$@"; do
  env $ENVS MOE_GEMM_DBG=$b timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/dbge_${TAG}_$b.json 2>/dev/null
  python - "gpurun_out/dbge_${TAG}_$b.json" "$b" "$ENVS" <<'PY'
import json, sys
try:
    d = json.load(open(sys.argv[1]))
    print(sys.argv[3], "dbg", sys.argv[2], round(d["ms_per_step"], 4), " ".join(f"{k}={v['ms']*1000:.1f}" for k, v in d["breakdown_ms"].items()))
except Exception as e:
    print(sys.argv[3], "dbg", sys.argv[2], "failed", e)
PY
done
