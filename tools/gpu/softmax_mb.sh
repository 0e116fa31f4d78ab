# softmax-phase microbenchmark: 128 columns per thread at 1, 2, 4 warps per SM sub-partition
cd $GRAFT_REPO_ROOT/tools/microbench
for th in 128 256 512; do echo "== threads $th" >> ../../gpurun_out/softmax_mb.log; timeout 120 ./softmax_128_$th >> ../../gpurun_out/softmax_mb.log 2>&1; done
