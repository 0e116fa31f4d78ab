# same-box A/B of two library builds: 1-GPU kernel timings (configs 2, 4) and
# the 4-GPU CP bench (the in-tree library vs build/fv_hm, swapped into place)
cd $GRAFT_REPO_ROOT
for rep in 1 2; do
for wl in varlen_packed_s32k magi1_4.5b_layer_s32k_b4096; do
for lib in paper_2505_13211_b200/libmagiplan.so build/fv_hm/libmagiplan.so; do
  timeout 180 python tools/time_bwd.py $lib $wl >> gpurun_out/fv.log 2>&1
done
done
done
cp paper_2505_13211_b200/libmagiplan.so build/lib_new.so
for rep in 1 2; do
for v in new hm; do
  if [ $v = new ]; then cp build/lib_new.so paper_2505_13211_b200/libmagiplan.so; else cp build/fv_hm/libmagiplan.so paper_2505_13211_b200/libmagiplan.so; fi
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 2962$rep \
    bench.py --gpus 4 --steps 3 --warmup 3 > gpurun_out/ab_${v}_$rep.json 2> gpurun_out/ab_${v}_$rep.err
done
done
cp build/lib_new.so paper_2505_13211_b200/libmagiplan.so
