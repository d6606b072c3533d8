#!/bin/bash
# Build an A/B variant of the native library with extra nvcc defines:
#   tools/build_variant.sh NAME -DFOO=1 ...   -> paper_2411_12690_b200/_lib/variants/libtsv_NAME.so
# Run with TSV_B200_LIB=<that path>.
set -e
name=$1; shift
d=paper_2411_12690_b200/_lib/variants/$name; mkdir -p $d
F="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O3 --expt-relaxed-constexpr -I include $*"
C=paper_2411_12690_b200/csrc
for f in context.cu local_stage.cu host_index.cpp rom_io.cpp; do nvcc $F -c $C/$f -o $d/${f%.*}.o & done; wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o $d/../libtsv_$name.so $d/*.o -lcusolver -lcublas -lcrypto -Xlinker -rpath,/usr/local/cuda/lib64
rm -rf $d
echo paper_2411_12690_b200/_lib/variants/libtsv_$name.so
