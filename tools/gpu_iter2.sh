#!/bin/bash
# One iteration: GPU tests (all unless files given), bench, force-kernel ncu capture.
# usage: tools/gpu_iter2.sh tag [pytest files...]
tag=${1:-it}; shift
tests=${@:-tests}
mkdir -p gpurun_out
timeout 900 python -m pytest $tests -m gpu -x -q 2>&1 | tail -8
timeout 300 python bench.py --steps 200 --warmup 20 --no-cpu-baseline --no-e2e > gpurun_out/b_$tag.json 2> gpurun_out/b_$tag.err
python tools/bench_brief.py gpurun_out/b_$tag.json
timeout 400 ncu --set full --import-source on --clock-control none -k regex:k_force_tile -s 3 -c 1 -o gpurun_out/force_$tag python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_$tag.log 2>&1
tail -1 gpurun_out/ncu_$tag.log
