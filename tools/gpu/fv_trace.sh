# per-role forward traces of the diagnostics build (one CTA each)
cd $GRAFT_REPO_ROOT
for lib in build/trace/libmagiplan.so build/ft_*/libmagiplan.so; do
  [ -f $lib ] || continue
  echo "== $lib" >> gpurun_out/fv_trace.log
  MAGI_LIB=$lib timeout 120 python tools/trace_fwd.py 0 >> gpurun_out/fv_trace.log 2>&1
  MAGI_LIB=$lib timeout 120 python tools/trace_fwd.py 1000 >> gpurun_out/fv_trace.log 2>&1
done
