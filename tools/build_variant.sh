#!/bin/bash
# Build a variant libhadr.so with extra -D flags on kernels.cu (A/B runs in one gpurun call):
#   tools/build_variant.sh NAME -DHADR_MARCH_THREADS=256 ...   ->  tools/var/NAME/libhadr.so
# (run `make -C paper_1712_06091_b200/csrc` first: the other objects are reused)
set -e
name=$1; shift
cs=paper_1712_06091_b200/csrc
mkdir -p tools/var/$name
nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo --fmad=false -Xcompiler -fPIC,-ffp-contract=off \
  -Xptxas -v "$@" -c -o tools/var/$name/kernels.o $cs/kernels.cu 2> tools/var/$name/kernels.ptxas.log
objs=$(ls $cs/build/*.o | grep -v kernels.o)
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o tools/var/$name/libhadr.so tools/var/$name/kernels.o $objs -ldl
rm -f tools/var/$name/kernels.o  # the snapshot sent to the GPU box is capped at 512 MiB
grep -A2 "k_stencil_march" tools/var/$name/kernels.ptxas.log | grep -E "registers|spill" | sort | uniq -c | sort -rn | head -4
