cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_cp.py -k capi -x -q -s -p no:cacheprovider > gpurun_out/capi_cp.log 2>&1; echo "rc=$?" >> gpurun_out/capi_cp.log
