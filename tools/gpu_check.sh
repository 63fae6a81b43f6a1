#!/bin/bash
# One gpurun round: gpu tests, bench, ncu full capture of the force kernel, launch list.
# usage (on the box): tools/gpu_check.sh [tag] [pytest-args]
tag=${1:-run}; shift
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q "$@" 2>&1 | tail -15
timeout 300 python bench.py --steps 200 --warmup 20 --no-cpu-baseline > gpurun_out/bench_$tag.json 2> gpurun_out/bench_$tag.err
python tools/bench_brief.py gpurun_out/bench_$tag.json
timeout 300 ncu --set full --import-source on --clock-control none -k regex:k_force_tile -s 3 -c 1 -o gpurun_out/force_$tag python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_$tag.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 80 --csv --log-file gpurun_out/launches_$tag.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
