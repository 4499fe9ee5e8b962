#!/bin/bash
# EP paths on one GPU: p2p tests (ranks sharing cuda:0), bench --ep for both transports, per-phase profile.
mkdir -p gpurun_out; TAG=${1:-ep}
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "p2p or ep_ or expert_parallel" -p no:cacheprovider > gpurun_out/t_$TAG.log 2>&1
echo tests=$?; tail -4 gpurun_out/t_$TAG.log
for t in nccl p2p; do
  timeout 300 python bench.py --ep --transport $t --steps 20 --warmup 5 > gpurun_out/bench_${TAG}_$t.json 2>gpurun_out/bench_${TAG}_$t.err
  echo ep_$t=$?; tail -2 gpurun_out/bench_${TAG}_$t.err
  python -c "import json;d=json.load(open('gpurun_out/bench_${TAG}_$t.json'));print(d['value'],d['ms_per_step'],d['config'].get('launch_mode'),d['gpu_launches'],(d.get('e2e') or {}).get('value'))"
done
