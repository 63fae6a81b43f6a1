#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_loopback.py tests/test_gpu_dist.py tests/test_gpu_dump.py tests/test_gpu_species.py -m gpu -x -q 2>&1 | tail -3
for L in 128 64; do
  timeout 300 python tools/group_overhead.py $L 1,1,1 50 loopback >> gpurun_out/lb_halo.jsonl 2>> gpurun_out/lb_halo.err
done
timeout 300 python tools/group_breakdown.py 128 1,1,1 20 loopback >> gpurun_out/lb_halo.jsonl 2>>gpurun_out/lb_halo.err
cat gpurun_out/lb_halo.jsonl
