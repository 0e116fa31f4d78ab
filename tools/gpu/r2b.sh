cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -x -q -s -p no:cacheprovider -k "not cp_" > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests.log
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
