#!/bin/bash
# Loopback NCCL data plane on the box: its tests, the full GPU suite, and the overhead runs.
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_loopback.py -m gpu -x -q 2>&1 | tail -15
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -5
for L in 128 64; do
  timeout 300 python tools/group_overhead.py $L 1,1,1 50 loopback >> gpurun_out/loopback_overhead.jsonl 2> gpurun_out/loopback_$L.err
  timeout 300 python tools/group_overhead.py $L 2,2,2 50 graph >> gpurun_out/loopback_overhead.jsonl 2>> gpurun_out/loopback_$L.err
done
cat gpurun_out/loopback_overhead.jsonl
