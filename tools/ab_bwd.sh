#!/bin/bash
# A/B of dK/dV exp2 polynomial shares on one box (development helper).
for V in "$@"; do
  echo "== MAGI_BWD_POLY=$V"
  MAGI_BWD_POLY=$V timeout 90 python -c "
import sys; sys.path.insert(0, '.')
from tools.perf_fwd import run
run(32768, 24, 8, 128, 4096, bwd=True, iters=10)
" | grep bwd
done
