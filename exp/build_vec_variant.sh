#!/bin/bash
# build an experimental libbdfb variant in which split.cu, split_mf.cu and rhs.cu (every unit that touches the
# SPLIT slot records) get extra -D flags; other objects are the current ones.
# usage: exp/build_vec_variant.sh NAME [nvcc flags...]   -> exp/lib_NAME.so  (load with BDFB_LIB=...)
name=$1; shift
cd /root/repo/paper_2405_01713_b200
F="-gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -fmad=false -Xcompiler -fPIC -Xptxas -v"
for u in split split_mf rhs; do
  /usr/local/cuda/bin/nvcc $F -c -o /tmp/${u}_$name.o csrc/$u.cu "$@" > /tmp/ptxas_${u}_$name.txt 2>&1 &
done
wait
for u in split split_mf rhs; do test -s /tmp/${u}_$name.o || { tail -20 /tmp/ptxas_${u}_$name.txt; exit 1; }; done
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a --shared -o /root/repo/exp/lib_$name.so build/bdfb.o \
  build/tpc.o build/erk.o /tmp/split_$name.o /tmp/split_mf_$name.o /tmp/rhs_$name.o -lnccl
grep -A2 "Function properties for _ZN4bdfb16split_ctl_kernelINS_15Tpc_drm19" /tmp/ptxas_split_$name.txt | tail -2
