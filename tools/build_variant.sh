#!/bin/bash
# Build an A/B variant of libfga.so with extra -D flags into
# paper_2009_14005_b200/_lib/libfga_<name>.so (objects under _lib/obj_<name>).
# usage: tools/build_variant.sh NAME "-DFOO=1 -DBAR=2"
set -e
NAME=$1; DEFS=$2
cd "$(dirname "$0")/../paper_2009_14005_b200/csrc"
OBJ=../_lib/obj_$NAME; mkdir -p $OBJ
NV="/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O2 --expt-relaxed-constexpr $DEFS"
pids=()
for f in tree forces rigid setup batched knn rbf capi; do $NV -c $f.cu -o $OBJ/$f.o & pids+=($!); done
$NV -Xcompiler -fopenmp -c io.cu -o $OBJ/io.o & pids+=($!)
for p in "${pids[@]}"; do wait $p; done
$NV -shared -o ../_lib/libfga_$NAME.so $OBJ/*.o -lcudart_static -lgomp -Xlinker -Bsymbolic
echo built libfga_$NAME.so
