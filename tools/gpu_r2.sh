#!/bin/bash
# One round-2 iteration on the box: parity tests, bench, launch list, ncu capture of the force kernel.
# usage: tools/gpu_r2.sh tag [pytest files...]
tag=${1:-it}; shift
tests=${@:-tests/test_gpu_parity.py}
mkdir -p gpurun_out
timeout 900 python -m pytest $tests -m gpu -x -q 2>&1 | tail -12
timeout 300 python bench.py --steps 200 --warmup 20 --no-cpu-baseline --no-e2e > gpurun_out/b_$tag.json 2> gpurun_out/b_$tag.err
python tools/bench_brief.py gpurun_out/b_$tag.json
timeout 300 ncu --set full --import-source on --clock-control none -k regex:k_force_tile -s 3 -c 1 -o gpurun_out/force_$tag python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_$tag.log 2>&1
tail -1 gpurun_out/ncu_$tag.log
