# peer-memory GroupCast: CP tests at 2 and 4 ranks, then the N=4 bench in both transports back to back
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_cp.py -q -s -p no:cacheprovider -k "p2p" > gpurun_out/p2p_tests.log 2>&1; echo "rc=$?" >> gpurun_out/p2p_tests.log
for rep in 1 2; do
for m in magi p2p; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 2964$rep \
    bench.py --gpus 4 --steps 3 --warmup 3 --cp-mode $m > gpurun_out/bench_n4_${m}_$rep.json 2> gpurun_out/bench_n4_${m}_$rep.err
done
done
