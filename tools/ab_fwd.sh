#!/bin/bash
# A/B of forward softmax variants on one box (development helper).
for V in "$@"; do
  echo "== variant $V"
  MAGI_FWD_VARIANT=$V timeout 60 python -c "
import sys; sys.path.insert(0, '.')
from tools.perf_fwd import run
run(32768, 24, 8, 128, 4096, iters=20)
run(32768, 24, 8, 128, 4096, iters=20)
"
done
