# peer-memory CP vs NCCL CP: the N=2 and N=4 bench in both transports back to back
cd $GRAFT_REPO_ROOT
for n in 4 2; do
for rep in 1 2; do
for m in magi p2p; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 296$n$rep \
    bench.py --gpus $n --steps 3 --warmup 3 --cp-mode $m > gpurun_out/bench_n${n}_${m}_$rep.json 2> gpurun_out/bench_n${n}_${m}_$rep.err
done
done
done
