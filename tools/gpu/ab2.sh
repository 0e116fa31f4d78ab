cd $GRAFT_REPO_ROOT
for rep in 1 2 3; do
for lib in build/var_old/libmagiplan.so build/var_nored/libmagiplan.so build/var_nw2qs2/libmagiplan.so; do
  timeout 120 python tools/time_bwd.py $lib >> gpurun_out/t.log 2>&1
done
done
