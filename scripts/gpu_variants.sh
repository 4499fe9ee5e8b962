#!/bin/bash
# Build and bench compile-time variants of the GEMM engine on the GPU box.
# usage: bash scripts/gpu_variants.sh TAG "-DFOO=1 -DBAR=2" "-DFOO=2" ...
mkdir -p gpurun_out; TAG=$1; shift
i=0
for v in "$@"; do
  rm -f build/*.o
  make -s EXTRA="$v" > gpurun_out/build_${TAG}_$i.log 2>&1 || { echo "build $v failed"; continue; }
  timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/bench_${TAG}_$i.json 2> gpurun_out/bench_${TAG}_$i.err
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
rm -f build/*.o; make -s > /dev/null 2>&1
