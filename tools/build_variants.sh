#!/bin/bash
# Build variants/<name>.so from EXTRA_NVFLAGS sets:  tools/build_variants.sh name1 "-DX=1" name2 "-DY=2" ...
# (the in-tree build is restored at the end).
set -e
cd "$(dirname "$0")/.."
mkdir -p variants
while [ $# -ge 2 ]; do
  name=$1; flags=$2; shift 2
  touch paper_2409_08669_b200/csrc/*.cu
  make -s -C paper_2409_08669_b200/csrc -j8 EXTRA_NVFLAGS="$flags" 2>&1 | grep -i error || true
  cp paper_2409_08669_b200/_build/libadrsplat.so variants/$name.so
done
touch paper_2409_08669_b200/csrc/*.cu
make -s -C paper_2409_08669_b200/csrc -j8 2>&1 | grep -i error || true
