#!/bin/bash
# build an experimental libbdfb variant: tpc.cu with extra -D flags, linked with the current bdfb.o
# usage: exp/build_variant.sh NAME [nvcc flags...]   -> exp/lib_NAME.so  (load with BDFB_LIB=...)
name=$1; shift
cd /root/repo/paper_2405_01713_b200
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -fmad=false -Xcompiler -fPIC \
  -Xptxas -v -c -o /tmp/tpc_$name.o csrc/tpc.cu "$@" > /tmp/ptxas_$name.txt 2>&1 || { tail -20 /tmp/ptxas_$name.txt; exit 1; }
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a --shared -o /root/repo/exp/lib_$name.so build/bdfb.o /tmp/tpc_$name.o -lnccl
grep -A2 "Function properties for _ZN4bdfb20integrate_tpc_kernelINS_15Tpc_drm19" /tmp/ptxas_$name.txt | tail -2
