#!/bin/bash
# Same-box A/B of environment knobs on the 1-GPU bench (development helper).
# usage: bash tools/ab_env.sh "A=1" "A=2" ...   (each run twice, interleaved)
cd "${GRAFT_REPO_ROOT:-.}"
for rep in 1 2; do
  for E in "$@"; do
    echo -n "[$E] "
    env $E timeout 200 python bench.py --steps 10 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1), {k:round(v['ms'],2) for k,v in d['kernels'].items()}, d['clocks']['sm_mhz'])"
  done
done
