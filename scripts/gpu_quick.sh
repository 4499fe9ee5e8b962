#!/bin/bash
# Quick GPU iteration: product/layer parity subset + bench breakdown (no CPU baseline / e2e).
mkdir -p gpurun_out; TAG=${1:-q}
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x --timeout 200 -p no:cacheprovider ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/tests_$TAG.log 2>&1
echo "tests_exit=$?"; tail -3 gpurun_out/tests_$TAG.log
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
echo "bench_exit=$?"
python - "$TAG" <<'PY'
import json, sys
d = json.load(open(f"gpurun_out/bench_{sys.argv[1]}.json"))
print("value", d["value"], "ms", d["ms_per_step"])
print(" ".join(f"{k}={v['ms']*1000:.0f}" for k, v in d["breakdown_ms"].items()))
PY
