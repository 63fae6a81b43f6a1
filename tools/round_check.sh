#!/bin/bash
# Round check on the box: compute-sanitizer (memcheck / racecheck / synccheck) of tools/sanitize.py,
# then bench lines for the scaling configs on one GPU.  usage: tools/round_check.sh tag
tag=${1:-r01}
mkdir -p gpurun_out
out=gpurun_out/sanitizer_$tag.txt
echo "# compute-sanitizer on tools/sanitize.py ($(date -u +%F))" > $out
for tool in memcheck racecheck synccheck; do
  r=$(timeout 900 compute-sanitizer --tool $tool python tools/sanitize.py 2>&1 | grep -E "sanitize run ok|ERROR SUMMARY|RACECHECK SUMMARY|Error|error" | tail -3 | tr '\n' ' ')
  echo "== $tool: $r" >> $out
done
cat $out
for w in weak128 strong256; do
  timeout 600 python bench.py --config $w --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_${w}_$tag.json 2> gpurun_out/bench_${w}_$tag.err
  python tools/bench_brief.py gpurun_out/bench_${w}_$tag.json
done
