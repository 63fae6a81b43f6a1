#!/bin/bash
# Loopback breakdown + force-kernel source capture (v62) for the region table.
mkdir -p gpurun_out
timeout 300 python tools/group_breakdown.py 128 1,1,1 20 loopback > gpurun_out/loopback_breakdown.jsonl 2>gpurun_out/lb.err
timeout 300 python tools/group_breakdown.py 64 1,1,1 20 loopback >> gpurun_out/loopback_breakdown.jsonl 2>>gpurun_out/lb.err
NCCL_DEBUG=INFO timeout 300 python tools/group_overhead.py 128 1,1,1 20 loopback > gpurun_out/lb_nccl_info.log 2>&1
cat gpurun_out/loopback_breakdown.jsonl
timeout 400 ncu --set full --import-source on --clock-control none -k regex:k_force_tile -s 3 -c 1 -o gpurun_out/force_v62 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_v62.log 2>&1
tail -2 gpurun_out/ncu_v62.log
