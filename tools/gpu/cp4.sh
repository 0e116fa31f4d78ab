# 4-GPU context-parallel validation: NCCL parity suite (2 and 4 ranks), the
# per-stage timeline at 4 ranks, and the CP bench at N = 2 and 4.
cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=index,name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/cp4_smi.txt
timeout 1500 python -m pytest tests/test_gpu_cp.py -q -s -p no:cacheprovider > gpurun_out/cp4_tests.log 2>&1; echo "cp tests rc=$?" >> gpurun_out/cp4_tests.log
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29512 tools/cp_timeline.py --per-rank 32768 --stages 4 --out gpurun_out/cp_timeline_n4.json > gpurun_out/cp_timeline_n4.log 2>&1; echo "timeline rc=$?" >> gpurun_out/cp_timeline_n4.log
for n in 2 4; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2952$n bench.py --gpus $n --steps 5 --warmup 3 > gpurun_out/bench_n$n.json 2> gpurun_out/bench_n$n.err; echo "bench n=$n rc=$?" >> gpurun_out/bench_n$n.err
done
