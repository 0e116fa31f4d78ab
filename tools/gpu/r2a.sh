cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt
timeout 1500 python -m pytest tests -m gpu -x -q -s -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests.log
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 tools/cp_timeline.py --per-rank 32768 --stages 4 --out gpurun_out/cp_timeline_n2.json > gpurun_out/cp_timeline_n2.log 2>&1; echo "timeline rc=$?" >> gpurun_out/cp_timeline_n2.log
