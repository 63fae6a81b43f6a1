#!/bin/bash
mkdir -p gpurun_out
timeout 300 python tools/group_breakdown.py 128 1,1,1 20 loopback > gpurun_out/loopback_breakdown2.jsonl 2>gpurun_out/lb2.err
timeout 300 python tools/group_breakdown.py 64 1,1,1 20 loopback >> gpurun_out/loopback_breakdown2.jsonl 2>>gpurun_out/lb2.err
for L in 128 64; do
  timeout 300 python tools/group_overhead.py $L 1,1,1 50 loopback >> gpurun_out/loopback_overhead2.jsonl 2>> gpurun_out/lb2.err
done
timeout 300 python tools/group_overhead.py 128 2,2,2 20 graph >> gpurun_out/loopback_overhead2.jsonl 2>> gpurun_out/lb2.err
cat gpurun_out/loopback_breakdown2.jsonl gpurun_out/loopback_overhead2.jsonl
timeout 600 python -m pytest tests/test_gpu_loopback.py tests/test_gpu_dist.py -m gpu -x -q 2>&1 | tail -3
