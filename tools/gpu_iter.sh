#!/bin/bash
# One iteration on the box: parity + dist tests, bench (kernel $2), ncu capture of the force kernel.
# usage: tools/gpu_iter.sh tag [force_kernel] [test-files...]
tag=${1:-it}; fk=${2:-0}; shift 2
tests=${@:-tests/test_gpu_parity.py tests/test_gpu_dist.py}
mkdir -p gpurun_out
timeout 900 python -m pytest $tests -m gpu -x -q 2>&1 | tail -12
timeout 300 python bench.py --steps 200 --warmup 20 --no-cpu-baseline --no-e2e --force-kernel $fk > gpurun_out/b_$tag.json 2> gpurun_out/b_$tag.err
python tools/bench_brief.py gpurun_out/b_$tag.json
kre=k_force_tile; [ "$fk" = "2" ] && kre=k_force_cells
timeout 300 ncu --set full --import-source on --clock-control none -k regex:$kre -s 3 -c 1 -o gpurun_out/force_$tag python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --force-kernel $fk > gpurun_out/ncu_$tag.log 2>&1
tail -1 gpurun_out/ncu_$tag.log
