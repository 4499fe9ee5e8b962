#!/bin/bash
# A/B perf: pair vs 1-SM kernels (bench only, no CPU baseline)
mkdir -p gpurun_out; TAG=${1:-ab}
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x --timeout 120 -k "six_products or layer_forward_backward" -p no:cacheprovider > gpurun_out/tests_$TAG.log 2>&1
echo "tests_exit=$?"; tail -3 gpurun_out/tests_$TAG.log
MOE_GEMM_PAIR=0 timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/bench_${TAG}_1sm.json 2>&1
echo "b1=$?"
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/bench_${TAG}_pair.json 2>&1
echo "b2=$?"
