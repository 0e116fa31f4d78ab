# forward-variant check + timing: the variant's forward tests (swapped in),
# then alternate the in-tree library with build/fv_*/ variants (configs 2, 3, 4)
cd $GRAFT_REPO_ROOT
cp paper_2505_13211_b200/libmagiplan.so build/lib_keep.so
for v in build/fv_*/libmagiplan.so; do
  cp $v paper_2505_13211_b200/libmagiplan.so
  timeout 150 python -m pytest tests/test_gpu_ffa_fwd.py tests/test_gpu_fullsize.py -x -q -p no:cacheprovider >> gpurun_out/fv_tests.log 2>&1; echo "$v rc=$?" >> gpurun_out/fv_tests.log
done
cp build/lib_keep.so paper_2505_13211_b200/libmagiplan.so
for rep in 1 2 3; do
for wl in magi1_4.5b_layer_s32k_b4096 magi1_24b_layer_s32k_b4096 varlen_packed_s32k; do
for lib in paper_2505_13211_b200/libmagiplan.so build/fv_*/libmagiplan.so; do
  timeout 90 python tools/time_bwd.py $lib $wl >> gpurun_out/fv.log 2>&1
done
done
done
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw --format=csv >> gpurun_out/fv.log
