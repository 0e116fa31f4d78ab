#!/bin/bash
# usage: build_var.sh NAME "-DFLAG ..."
cd /root/repo
mkdir -p build/var_$1
nvcc -gencode arch=compute_100a,code=sm_100a -std=c++20 -O3 -lineinfo -Xcompiler -fPIC,-fvisibility=hidden -Iinclude -Ithird_party -Ipaper_2505_13211_b200/csrc -Xptxas -v --expt-relaxed-constexpr $2 -c paper_2505_13211_b200/csrc/kernels/ffa_bwd.cu -o build/var_$1/ffa_bwd.o 2> build/var_$1/ptxas.log || { cat build/var_$1/ptxas.log; exit 1; }
objs=$(ls build/obj/*.o | grep -v kernels_ffa_bwd)
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o build/var_$1/libmagiplan.so $objs build/var_$1/ffa_bwd.o -lcudart_static
echo built $1
