# Re-fit the B200 cost model on the current kernels (2 ranks for the
# collectives), then the per-stage CP timeline at 2 and 4 ranks against it.
cd $GRAFT_REPO_ROOT
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29531 tools/calibrate_cost_model.py > gpurun_out/calib.log 2>&1; echo "calib rc=$?" >> gpurun_out/calib.log
cp configs/cost_model_b200.json gpurun_out/cost_model_b200.json
for n in 2 4; do
timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2954$n tools/cp_timeline.py --per-rank 32768 --stages 4 --out gpurun_out/cp_timeline_n$n.json > gpurun_out/cp_timeline_n$n.log 2>&1; echo "timeline rc=$?" >> gpurun_out/cp_timeline_n$n.log
done
