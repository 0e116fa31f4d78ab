#!/bin/bash
# Bench + ncu launch list + one --set full capture of every FFA kernel.
# usage: bash tools/profile_round.sh TAG   (outputs under gpurun_out/)
cd "${GRAFT_REPO_ROOT:-.}"
TAG=${1:-dev}
timeout 300 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_$TAG.log 2>&1 && tail -1 gpurun_out/bench_$TAG.log
timeout 400 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 2 --warmup 1 > gpurun_out/ncu_list_$TAG.log 2>&1
echo "launch list rc=$?"
timeout 400 ncu --set full --import-source on --clock-control none -k regex:"ffa_|bwd_preprocess" -c 4 \
  -o gpurun_out/prof_$TAG python tools/one_step.py > gpurun_out/ncu_full_$TAG.log 2>&1
echo "full capture rc=$?"
