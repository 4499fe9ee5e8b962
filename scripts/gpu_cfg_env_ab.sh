#!/bin/bash
# configs x env variants: bash scripts/gpu_cfg_env_ab.sh "C2 C3 C4" "A=1" "B=2" ...
CFGS=$1; shift
mkdir -p gpurun_out
for c in $CFGS; do
  for v in "$@"; do
    env $v timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/cfgab.json 2>/dev/null
    python - gpurun_out/cfgab.json "$c" "$v" <<'PY'
import json, sys
try:
    d = json.load(open(sys.argv[1]))
    print(sys.argv[2], sys.argv[3], round(d["ms_per_step"], 4), " ".join(f"{k}={v['ms']*1000:.1f}" for k, v in d["breakdown_ms"].items()))
except Exception as e:
    print(sys.argv[2], sys.argv[3], "failed", e)
PY
  done
done
