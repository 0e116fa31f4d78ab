# Driver-style scaling run on this box: bench N=1,2,4 (torchrun for N>1) and
# the reference arm at N=1 and N=4; then the multi-GPU GPU suite (NCCL path).
cd $GRAFT_REPO_ROOT
TAG=${1:-scale}
nvidia-smi --query-gpu=index,name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi_$TAG.txt
timeout 900 python bench.py > gpurun_out/bench_${TAG}_n1.json 2> gpurun_out/bench_${TAG}_n1.err
for n in 2 4; do
  timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2961$n \
    bench.py --gpus $n > gpurun_out/bench_${TAG}_n$n.json 2> gpurun_out/bench_${TAG}_n$n.err
  echo "n=$n rc=$?" >> gpurun_out/bench_${TAG}_n$n.err
done
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29619 \
  bench.py --gpus 4 --impl reference > gpurun_out/bench_${TAG}_ref_n4.json 2> gpurun_out/bench_${TAG}_ref_n4.err
echo "ref rc=$?" >> gpurun_out/bench_${TAG}_ref_n4.err
timeout 1800 python -m pytest tests/test_gpu_cp.py -q -p no:cacheprovider > gpurun_out/cp_tests_${TAG}.log 2>&1; echo "tests rc=$?" >> gpurun_out/cp_tests_${TAG}.log
