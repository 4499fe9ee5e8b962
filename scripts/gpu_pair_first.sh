#!/bin/bash
# First run of the CTA-pair kernels: guarded, short timeouts.
mkdir -p gpurun_out
timeout 180 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_p1.log 2>&1
echo "smoke_exit=$?"; tail -3 gpurun_out/smoke_p1.log
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x --timeout 120 -k "six_products or empty_expert" -p no:cacheprovider > gpurun_out/tests_p1a.log 2>&1
echo "prod_exit=$?"; tail -15 gpurun_out/tests_p1a.log
timeout 900 python -m pytest tests -m gpu -q --timeout 200 -rf -p no:cacheprovider > gpurun_out/tests_p1.log 2>&1
echo "tests_exit=$?"; tail -5 gpurun_out/tests_p1.log
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_p1.json 2> gpurun_out/bench_p1.err
echo "bench_exit=$?"; tail -3 gpurun_out/bench_p1.err
MOE_GEMM_PAIR=0 timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/bench_p1_nopair.json 2>&1
echo "bench_nopair_exit=$?"
