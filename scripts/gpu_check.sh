#!/bin/bash
# One GPU round trip: smoke, GPU tests, bench, ncu launch list (+ optional full capture).
# usage (under gpurun): bash scripts/gpu_check.sh TAG [tests|bench|ncu|full]...
TAG=${1:-x}
shift
STEPS="${@:-tests bench ncu}"
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,temperature.gpu --format=csv > gpurun_out/gpu_$TAG.txt
for s in $STEPS; do
  case $s in
    tests)
      timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1
      echo "smoke_exit=$?"
      timeout 1200 python -m pytest tests -m gpu -q --timeout 300 -rf -p no:cacheprovider > gpurun_out/tests_$TAG.log 2>&1
      echo "tests_exit=$?"; tail -5 gpurun_out/tests_$TAG.log ;;
    bench)
      timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
      echo "bench_exit=$?"; tail -3 gpurun_out/bench_$TAG.err ;;
    ncu)
      timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv \
        python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_list_$TAG.log 2>&1
      echo "ncu_list_exit=$?" ;;
    full)
      # the 8 tcgen05 GEMM launches of the third eager warm-up step
      timeout 900 ncu --set full --clock-control none --import-source on -k regex:bsgemm -s 16 -c 8 \
        -o gpurun_out/prof_$TAG python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_full_$TAG.log 2>&1
      echo "ncu_full_exit=$?" ;;
    perm)
      # topology, padded gather and scatter backward of the third warm-up step
      timeout 900 ncu --set full --clock-control none -k "regex:topo|scatter" -s 6 -c 3 \
        -o gpurun_out/prof_perm_$TAG python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_perm_$TAG.log 2>&1
      echo "ncu_perm_exit=$?" ;;
  esac
done
