#!/bin/bash
# Build libdpd.so variants for tools/ab.sh: tools/build_variants.sh name "flags" [name "flags" ...]
# Each lands in tools/scratch/v/<name>.so; the in-tree libdpd.so is rebuilt without flags at the end.
set -e
cd "$(dirname "$0")/.."
mkdir -p tools/scratch/v
while [ $# -ge 2 ]; do
  name=$1; flags=$2; shift 2
  DPD_NVCC_FLAGS="$flags" python -c "from paper_1911_04712_b200 import build as b; b.build(force=True)"
  cp paper_1911_04712_b200/libdpd.so tools/scratch/v/$name.so
  echo "built $name ($flags)"
done
python -c "from paper_1911_04712_b200 import build as b; b.build(force=True)"
