#!/bin/bash
# A/B of the CTA-pair experiment switches (MOE_SDD_PAIR, MOE_GEMM_PAIR_ROWS) on the product sweep and the bench
mkdir -p gpurun_out
for v in base MOE_SDD_PAIR MOE_GEMM_PAIR_ROWS; do
  if [ $v = base ]; then E=""; else E="$v=1"; fi
  env $E timeout 300 python scripts/product_sweep.py --problems XS,Medium --reps 10 > gpurun_out/ab_$v.log 2>&1
  echo "== $v"; python - $v <<'PY'
import json,sys
for l in open(f"gpurun_out/ab_{sys.argv[1]}.log"):
    if l.startswith("{"):
        d=json.loads(l)
        if "product" in d: print(d["problem"], d["product"], d["ours_ms"], d["bmm_ms"])
PY
  env $E timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/abb_$v.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/abb_$v.json'));print('bench',d['value'],d['ms_per_step'],{k:round(v['ms']*1000,1) for k,v in d['breakdown_ms'].items()})"
done
