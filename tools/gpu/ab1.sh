cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_ffa_fwd.py tests/test_gpu_fullsize.py tests/test_gpu_guard.py -x -q -p no:cacheprovider > gpurun_out/fwd_tests.log 2>&1; echo "rc=$?" >> gpurun_out/fwd_tests.log
for rep in 1 2; do
for lib in paper_2505_13211_b200/libmagiplan.so build/var_old/libmagiplan.so build/var_nw2/libmagiplan.so build/var_nw2qs2/libmagiplan.so build/var_nw4qs2/libmagiplan.so; do
  timeout 120 python tools/time_bwd.py $lib >> gpurun_out/t.log 2>&1
done
done
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw --format=csv >> gpurun_out/t.log
