#!/bin/bash
# Build a variant of the library with one translation unit recompiled with extra flags:
#   tools/variant.sh NAME UNIT "-DFOO=1 ..."   -> build/variants/NAME.so
name=$1; unit=$2; flags=$3
mkdir -p build/variants/obj_$name
exact="preprocess preprocess_bwd densify backscatter"
extra=""; for e in $exact; do [ "$e" = "$unit" ] && extra="-fmad=false"; done
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr $extra $flags \
  -c paper_2411_19588_b200/csrc/$unit.cu -o build/variants/obj_$name/$unit.o || exit 1
objs=""; for o in build/obj/*.o; do b=$(basename $o); [ "$b" = "$unit.o" ] && objs="$objs build/variants/obj_$name/$unit.o" || objs="$objs $o"; done
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o build/variants/$name.so $objs
