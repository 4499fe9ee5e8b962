#!/bin/bash
# compute-sanitizer racecheck / synccheck / memcheck over smoke() and a set of
# parity tests (one GPU). Logs under gpurun_out/sanitizer_<tool>_<what>.txt
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in ${TOOLS:-racecheck synccheck}; do
  timeout 900 $CS --tool $tool --print-limit 50 python -c "import __graft_entry__ as g; g.smoke()" \
    > gpurun_out/sanitizer_${tool}_smoke.txt 2>&1
  echo "$tool smoke exit=$?: $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' gpurun_out/sanitizer_${tool}_smoke.txt | tail -2 | tr '\n' ' ')"
  timeout 1500 $CS --tool $tool --print-limit 50 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider \
    -k "${TESTS:-six_products and case0 or dsd_scatter and case0 or dsd_dx and case0 or permutation or topology_bit_exact or layer_forward_backward and C0- or capacity_forward_backward and C0-cf1}" \
    > gpurun_out/sanitizer_${tool}_tests.txt 2>&1
  echo "$tool tests exit=$?: $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|passed|failed' gpurun_out/sanitizer_${tool}_tests.txt | tail -3 | tr '\n' ' ')"
done
