#!/bin/bash
# Same-box A/B of the current build against build/ab/libmagiplan_base.so
# (development helper; MAGIPLAN_LIB selects the library _lib.py loads).
cd "${GRAFT_REPO_ROOT:-.}"
for L in new base new base; do
  if [ $L = base ]; then export MAGIPLAN_LIB=$PWD/build/ab/libmagiplan_base.so; else unset MAGIPLAN_LIB; fi
  echo -n "$L: "; timeout 200 python bench.py --steps 10 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1), {k:round(v['ms'],2) for k,v in d['kernels'].items()}, d['clocks']['sm_mhz'])"
done
