#!/bin/bash
# CTA-pair SDD^T (wide in-place act'(H) ring) check: parity under MOE_SDD_PAIR=1, bench A/B
mkdir -p gpurun_out
MOE_SDD_PAIR=1 timeout 900 python -m pytest tests/test_gpu_parity.py -q -x --timeout 600 -p no:cacheprovider \
  -k "six_products or layer_forward_backward or full_size_every_output or degenerate or autograd" > gpurun_out/qt_sddt.log 2>&1
echo "tests_exit=$?"; tail -3 gpurun_out/qt_sddt.log
for rep in 1 2; do
  for v in "MOE_DEFAULT=1" "MOE_SDD_PAIR=1"; do
    env $v timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/qb_sddt.json 2>/dev/null
    python - gpurun_out/qb_sddt.json "$v" <<'PY'
import json, sys
try:
    d = json.load(open(sys.argv[1]))
    print("bench", sys.argv[2], round(d["ms_per_step"], 4), " ".join(f"{k}={v['ms']*1000:.1f}" for k, v in d["breakdown_ms"].items()))
except Exception as e:
    print("bench", sys.argv[2], "failed", e)
PY
  done
done
