# per-role backward traces of the diagnostics build (dK/dV CTA 0 and 500, dQ CTA 0 and 1000)
cd $GRAFT_REPO_ROOT
MAGI_LIB=build/trace/libmagiplan.so timeout 120 python tools/trace_bwd.py 0 > gpurun_out/bwd_trace.log 2>&1
MAGI_LIB=build/trace/libmagiplan.so timeout 120 python tools/trace_bwd.py 500 >> gpurun_out/bwd_trace.log 2>&1
MAGI_LIB=build/trace/libmagiplan.so timeout 120 python tools/trace_dq.py 0 >> gpurun_out/bwd_trace.log 2>&1
MAGI_LIB=build/trace/libmagiplan.so timeout 120 python tools/trace_dq.py 1000 >> gpurun_out/bwd_trace.log 2>&1
