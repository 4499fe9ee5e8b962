#!/bin/bash
# A/B of library builds: bash scripts/gpu_variant_ab.sh name1 name2 ... (abvariants/libmoe_<name>.so)
mkdir -p gpurun_out
cp paper_2211_15841_b200/libmoe.so /tmp/libmoe_current.so
for v in "$@"; do
  for rep in 1 2; do
    cp abvariants/libmoe_$v.so paper_2211_15841_b200/libmoe.so
    timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/ab_$v.json 2>/dev/null
    python - "$v" <<'PY'
import json, sys
d = json.load(open(f"gpurun_out/ab_{sys.argv[1]}.json"))
print(sys.argv[1], round(d["ms_per_step"], 4), " ".join(f"{k}={v['ms']*1000:.1f}" for k, v in d["breakdown_ms"].items()))
PY
  done
done
cp /tmp/libmoe_current.so paper_2211_15841_b200/libmoe.so
