#!/bin/bash
# Build an experimental libcarve_cuda.so (tools only): tools/build_variant.sh NAME SRCDIR [nvcc defines...]
# -> build/exp/NAME/libcarve_cuda.so, loaded with CARVE_LIB=build/exp/NAME/libcarve_cuda.so
set -eu
NAME=$1; SRC=$2; shift 2
OUT=build/exp/$NAME
mkdir -p $OUT
FLAGS="-O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -fmad=false -Xcompiler -fPIC -Iinclude $*"
pids=()
for f in carve_cuda dp_variants_a dp_variants_b dp_variants_c dp_variants_d; do
  nvcc $FLAGS -c -o $OUT/$f.o $SRC/$f.cu & pids+=($!)
done
for p in "${pids[@]}"; do wait $p; done
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $OUT/libcarve_cuda.so $OUT/*.o
rm -f $OUT/*.o
echo built $OUT/libcarve_cuda.so
