#!/bin/bash
# ncu --set full capture of one launch of each FFA kernel (config 2 shapes).
# usage: bash tools/ncu_capture.sh TAG
cd "${GRAFT_REPO_ROOT:-.}"
TAG=${1:-dev}
for K in ffa_fwd ffa_bwd_dkdv ffa_bwd_dq; do
  timeout 300 ncu --set full --import-source on --clock-control none -k regex:$K -c 1 \
    -o gpurun_out/prof_${TAG}_$K python -c "
import sys; sys.path.insert(0, '.')
from tools.perf_fwd import run
run(32768, 24, 8, 128, 4096, bwd=True, iters=1)
" > gpurun_out/ncu_${TAG}_$K.log 2>&1
  tail -1 gpurun_out/ncu_${TAG}_$K.log
done
