#!/bin/bash
# Build library variants of one source file with sed substitutions, for A/B timing on the GPU box.
# usage: tools/variants.sh <src.cu> <name> 'sed-expr' [<name> 'sed-expr' ...]
# leaves build/variants/<name>.so; the in-tree library is rebuilt from the unmodified source.
set -e
src=$1; shift
mkdir -p build/variants
cp "$src" /tmp/variant_orig.cu
while [ $# -gt 0 ]; do
  name=$1; expr=$2; shift 2
  sed -e "$expr" /tmp/variant_orig.cu > "$src"
  make -s >/dev/null
  cp paper_2411_19588_b200/libuwsplat_b200.so build/variants/$name.so
done
cp /tmp/variant_orig.cu "$src"
make -s >/dev/null
