# Full GPU suite on this box's GPUs (CP cases run at 2 and 4 ranks when 4
# GPUs are visible) + smoke.
cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=index,name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/final_smi.txt
timeout 2400 python -m pytest tests -m gpu -q -s -p no:cacheprovider > gpurun_out/final_gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/final_gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/final_smoke.log
