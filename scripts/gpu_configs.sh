#!/bin/bash
# Single-GPU bench of every BASELINE config (C0..C4) — throughput beyond the headline C1.
mkdir -p gpurun_out; TAG=${1:-cfg}
for c in C0 C1 C2 C3 C4; do
  timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_${TAG}_$c.json 2> gpurun_out/bench_${TAG}_$c.err
  python - "$TAG" "$c" <<'PY'
import json, sys
try:
    d = json.load(open(f"gpurun_out/bench_{sys.argv[1]}_{sys.argv[2]}.json"))
    print(sys.argv[2], "| %.2f Mtok/s  %.3f ms/step  roofline %s %.3f  gemm %.0f TF" % (
        d["value"] / 1e6, d["ms_per_step"], d["roofline"]["kernel"], d["roofline"].get("frac") or 0,
        d["gemm"]["useful_tflops"]), d["config"].get("expert_load_max_over_mean"))
    print("   ", " ".join(f"{k}={v['ms']*1000:.0f}" for k, v in d["breakdown_ms"].items()))
except Exception as e:
    print(sys.argv[2], "| failed", e)
PY
done
