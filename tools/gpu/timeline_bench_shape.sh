# Per-stage CP timeline at the bench's per-rank shape (131072 tokens, 48q/8kv,
# block-causal 8192) with the packages forced to 4, at 2 and 4 ranks.
cd $GRAFT_REPO_ROOT
for n in 2 4; do
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2955$n tools/cp_timeline.py --per-rank 131072 --block 8192 --stages 4 --out gpurun_out/cp_timeline_bench_n$n.json > gpurun_out/cp_timeline_bench_n$n.log 2>&1; echo "timeline rc=$?" >> gpurun_out/cp_timeline_bench_n$n.log
done
