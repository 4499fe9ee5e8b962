#!/bin/bash
# A/B of library builds (abvariants/libmoe_<name>.so), 2 reps each, bench breakdown
mkdir -p gpurun_out
cp paper_2211_15841_b200/libmoe.so /tmp/libmoe_current.so
for rep in 1 2; do
  for v in "$@"; do
    cp abvariants/libmoe_$v.so paper_2211_15841_b200/libmoe.so
    timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/ab_$v.json 2>/dev/null
    python - "$v" <<'PY'
import json, sys
try:
    d = json.load(open(f"gpurun_out/ab_{sys.argv[1]}.json"))
    print(sys.argv[1], round(d["ms_per_step"], 4), " ".join(f"{k}={v['ms']*1000:.1f}" for k, v in d["breakdown_ms"].items()))
except Exception as e:
    print(sys.argv[1], "failed", e)
PY
  done
done
cp /tmp/libmoe_current.so paper_2211_15841_b200/libmoe.so
