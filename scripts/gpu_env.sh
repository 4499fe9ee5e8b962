#!/bin/bash
# Bench under several environment settings: bash scripts/gpu_env.sh TAG "VAR=val ..." "VAR=val" ...
mkdir -p gpurun_out; TAG=$1; shift
i=0
for v in "$@"; do
  env $v timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/bench_${TAG}_$i.json 2> gpurun_out/bench_${TAG}_$i.err
  python - "$TAG" "$i" "$v" <<'PY'
import json, sys
try:
    d = json.load(open(f"gpurun_out/bench_{sys.argv[1]}_{sys.argv[2]}.json"))
    print(sys.argv[3], "| value %.1fM" % (d["value"] / 1e6), " ".join(f"{k}={v['ms']*1000:.0f}" for k, v in d["breakdown_ms"].items()))
except Exception as e:
    print(sys.argv[3], "| failed", e)
PY
  i=$((i+1))
done
