#!/bin/bash
# tools/build_variant.sh OUT.so -DFLAG=... : build an experimental copy of the engine
out=$1; shift
cd "$(dirname "$0")/../paper_2104_08865_b200/csrc" && /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O3,-fopenmp -Xptxas -v --expt-relaxed-constexpr -shared "$@" -o "$out" halftime.cu -lgomp 2> "$out.ptxas.log"
grep -A2 "hash_kernelILi40ELb0" "$out.ptxas.log" | grep -E "Used|spill" | sed 's/ptxas info    ://'
