# Per-stage CP timeline of the bench's own scenario (solver-chosen stages) at 2 and 4 ranks.
cd $GRAFT_REPO_ROOT
for n in 2 4; do
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2956$n tools/cp_timeline.py --bench --out gpurun_out/cp_timeline_benchsolver_n$n.json > gpurun_out/cp_timeline_benchsolver_n$n.log 2>&1; echo "timeline rc=$?" >> gpurun_out/cp_timeline_benchsolver_n$n.log
done
