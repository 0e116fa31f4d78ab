# Strong scaling: 1M tokens (block-causal 8192, 48q/8kv) at cp 1, 2, 4 on one box.
cd $GRAFT_REPO_ROOT
for n in 1 2 4; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2963$n \
    tools/cp_strong.py --steps 1 --warmup 1 >> gpurun_out/cp_strong.jsonl 2> gpurun_out/cp_strong_n$n.err
  echo "n=$n rc=$?" >> gpurun_out/cp_strong_n$n.err
  nvidia-smi --query-gpu=index,clocks.sm,power.draw --format=csv,noheader >> gpurun_out/cp_strong_n$n.err
done
