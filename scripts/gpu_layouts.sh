#!/bin/bash
# padded vs unpadded (P:297 fringe) layout on every BASELINE config, same harness
mkdir -p gpurun_out
for c in ${CONFIGS:-C1 C2 C3 C4}; do
  for l in padded unpadded; do
    timeout 300 python bench.py --config $c --layout $l --steps 20 --warmup 5 --no-cpu-baseline --no-e2e \
      > gpurun_out/layout_${c}_${l}.json 2>/dev/null
    python - gpurun_out/layout_${c}_${l}.json $c $l <<'PY'
import json, sys
try:
    d = json.load(open(sys.argv[1]))
    print(sys.argv[2], sys.argv[3], f"{d['value']/1e6:.2f} Mtok/s", round(d["ms_per_step"], 4),
          " ".join(f"{k}={v['ms']*1000:.1f}" for k, v in d["breakdown_ms"].items()))
except Exception as e:
    print(sys.argv[2], sys.argv[3], "failed", e)
PY
  done
done
