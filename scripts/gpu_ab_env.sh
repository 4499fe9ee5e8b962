#!/bin/bash
# A/B of bench variants on one box: bash scripts/gpu_ab_env.sh TAG "VARIANT1" "VARIANT2" ... where a variant is
# "VAR=VALUE ...;--bench-flag ..." (either part may be empty); prints value, ms and the per-kernel breakdown of each.
mkdir -p gpurun_out; TAG=$1; shift
i=0
for v in "$@"; do
  i=$((i+1))
  envs="${v%%;*}"; flags=""; [[ "$v" == *\;* ]] && flags="${v#*;}"
  env $envs timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e $flags > gpurun_out/ab_${TAG}_$i.json 2> gpurun_out/ab_${TAG}_$i.err
  python - "$TAG" "$i" "$v" <<'PY'
import json, sys
try:
    d = json.load(open(f"gpurun_out/ab_{sys.argv[1]}_{sys.argv[2]}.json"))
    print(f"[{sys.argv[3]}] value {d['value']/1e6:.2f} Mtok/s ms {d['ms_per_step']}")
    print("   " + " ".join(f"{k}={v['ms']*1000:.1f}" for k, v in d["breakdown_ms"].items()))
except Exception as e:
    print(f"[{sys.argv[3]}] failed {e}")
PY
done
