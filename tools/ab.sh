#!/bin/bash
# A/B timing of prebuilt library variants on the box: tools/ab.sh tag variant.so [variant.so ...]
# Each variant is copied over the in-tree libdpd.so and timed with bench.py (kernel times).
tag=${1:-ab}; shift
mkdir -p gpurun_out
cp paper_1911_04712_b200/libdpd.so /tmp/libdpd_orig.so
for v in "$@"; do
  cp "$v" paper_1911_04712_b200/libdpd.so
  touch paper_1911_04712_b200/libdpd.so
  for rep in 1 2; do
    timeout 300 python bench.py --steps 200 --warmup 20 --no-cpu-baseline --no-e2e $BENCH_ARGS > gpurun_out/ab_${tag}_$(basename $v .so)_$rep.json 2>/dev/null
    echo "$(basename $v) rep$rep: $(python tools/bench_brief.py gpurun_out/ab_${tag}_$(basename $v .so)_$rep.json | tr "\n" " ")"
  done
done
cp /tmp/libdpd_orig.so paper_1911_04712_b200/libdpd.so
