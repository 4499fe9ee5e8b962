#!/bin/bash
# quick GPU check of a kernel change: a parity subset, the bench breakdown, optional env A/B
TAG=${1:-q}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x --timeout 600 -k "${TESTS:-six_products or dsd_scatter or dsd_dx or layer_forward_backward or full_size_every_output and C1}" -p no:cacheprovider > gpurun_out/qt_$TAG.log 2>&1
echo "tests_exit=$?"; tail -3 gpurun_out/qt_$TAG.log
for v in "" ${AB}; do
  env $v timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/qb_${TAG}_${v//=/_}.json 2>/dev/null
  python - gpurun_out/qb_${TAG}_${v//=/_}.json "$v" <<'PY'
import json, sys
try:
    d = json.load(open(sys.argv[1]))
    print("bench", sys.argv[2] or "default", round(d["ms_per_step"], 4), " ".join(f"{k}={v['ms']*1000:.1f}" for k, v in d["breakdown_ms"].items()))
except Exception as e:
    print("bench", sys.argv[2], "failed", e)
PY
done
