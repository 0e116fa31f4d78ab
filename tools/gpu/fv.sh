# kernel-variant timing: alternate the in-tree library with build/fv_*/
# variants on config 2 (and 3)
cd $GRAFT_REPO_ROOT
for rep in 1 2 3; do
for wl in magi1_4.5b_layer_s32k_b4096 magi1_24b_layer_s32k_b4096; do
for lib in paper_2505_13211_b200/libmagiplan.so build/fv_*/libmagiplan.so; do
  timeout 90 python tools/time_bwd.py $lib $wl >> gpurun_out/fv.log 2>&1
done
done
done
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw --format=csv >> gpurun_out/fv.log
