#!/bin/bash
# build an experimental libbdfb variant: split.cu with extra -D flags, linked with the other current objects
# usage: exp/build_split_variant.sh NAME [nvcc flags...]   -> exp/lib_NAME.so  (load with BDFB_LIB=...)
name=$1; shift
cd /root/repo/paper_2405_01713_b200
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -fmad=false -Xcompiler -fPIC \
  -Xptxas -v -c -o /tmp/split_$name.o csrc/split.cu "$@" > /tmp/ptxas_split_$name.txt 2>&1 || { tail -20 /tmp/ptxas_split_$name.txt; exit 1; }
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a --shared -o /root/repo/exp/lib_$name.so build/bdfb.o build/tpc.o \
  build/split_mf.o build/erk.o build/rhs.o /tmp/split_$name.o -lnccl
grep -A2 "Function properties for _ZN4bdfb16split_ctl_kernelINS_15Tpc_drm19" /tmp/ptxas_split_$name.txt | tail -2
