#!/bin/bash
# Round artifacts on the box: default bench line, reference arm, launch list, ncu full capture
# of one step's kernels (traffic), all under gpurun_out/.  usage: tools/round_artifacts.sh tag
tag=${1:-r01}
mkdir -p gpurun_out
timeout 600 python bench.py > gpurun_out/bench_default_$tag.json 2> gpurun_out/bench_default_$tag.err
tail -c 600 gpurun_out/bench_default_$tag.json; echo
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_reference_$tag.json 2> gpurun_out/bench_reference_$tag.err
tail -c 300 gpurun_out/bench_reference_$tag.json; echo
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -s 820 -c 200 --csv --log-file gpurun_out/launches_$tag.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-weak-point > /dev/null 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_bin|k_scan|k_scatter|k_force_tile" -s 816 -c 4 -o gpurun_out/step_$tag python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_step_$tag.log 2>&1
tail -2 gpurun_out/ncu_step_$tag.log
