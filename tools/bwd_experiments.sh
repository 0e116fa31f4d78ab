#!/bin/bash
# Backward pipeline diagnostics: time the dK/dV and dQ kernels with the
# elementwise work removed (1) or the gradient MMAs removed (2).
for e in 0 1 2; do
  echo "experiment $e"
  MAGI_BWD_EXPERIMENT=$e python bench.py --steps 3 --warmup 2 --no-cpu-baseline | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); k=d['kernels']
print({n: round(v['ms'],2) for n,v in k.items()})"
done
