# One-GPU round check: GPU suite, smoke, bench (all fields), extra workloads,
# ncu launch list and one --set full capture of every FFA kernel.
# usage: bash tools/gpu/round_check.sh TAG   (outputs under gpurun_out/)
cd $GRAFT_REPO_ROOT
TAG=${1:-dev}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/smi_$TAG.txt
timeout 1200 python -m pytest tests -m gpu -q -s -p no:cacheprovider > gpurun_out/gpu_tests_$TAG.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke_$TAG.log
timeout 900 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo "bench rc=$?" >> gpurun_out/bench_$TAG.err
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref_$TAG.json 2> gpurun_out/bench_ref_$TAG.err
for W in magi1_24b_layer_s32k_b4096 varlen_packed_s32k; do
  timeout 300 python bench.py --workload $W --no-weak-anchor --no-cpu-baseline > gpurun_out/bench_${W}_$TAG.json 2>> gpurun_out/bench_$TAG.err
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 2 --warmup 1 --no-weak-anchor --no-cpu-baseline > gpurun_out/ncu_list_$TAG.log 2>&1
echo "launch list rc=$?" >> gpurun_out/ncu_list_$TAG.log
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"ffa_|bwd_preprocess" -c 4 \
  -o gpurun_out/prof_$TAG python tools/one_step.py > gpurun_out/ncu_full_$TAG.log 2>&1
echo "full capture rc=$?" >> gpurun_out/ncu_full_$TAG.log
