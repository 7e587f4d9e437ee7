#!/bin/bash
# compile only csrc/tpc.cu (fast iteration on the thread-per-cell kernel); extra nvcc args pass through
cd /root/repo/paper_2405_01713_b200 && /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -fmad=false -Xcompiler -fPIC -Xptxas -v -c -o /tmp/tpc_test.o csrc/tpc.cu "$@" 2>&1 | grep -A2 "Function properties" | grep -A2 "integrate_tpc\|tpc_factorILi22ELb1\|3jac" | grep -v "^--"
