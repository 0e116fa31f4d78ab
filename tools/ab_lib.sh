cd $GRAFT_REPO_ROOT
for L in new old new old; do
  if [ $L = old ]; then export MAGIPLAN_LIB=$PWD/build/ab/libmagiplan_old_dq.so; else unset MAGIPLAN_LIB; fi
  echo -n "$L: "; timeout 200 python bench.py --steps 10 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1), {k:round(v['ms'],2) for k,v in d['kernels'].items()}, d['clocks']['sm_mhz'])"
done
