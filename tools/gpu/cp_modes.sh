# CP bench of every mode at N = 4 (and the C-ABI executor at N = 2), back to back on one box.
cd $GRAFT_REPO_ROOT
port=29600
for spec in "4 magi" "4 capi" "4 ring" "4 ulysses" "2 capi"; do
  set -- $spec; n=$1; m=$2; port=$((port+1))
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $port \
    bench.py --gpus $n --steps 5 --warmup 2 --cp-mode $m > gpurun_out/bench_n${n}_$m.json 2> gpurun_out/bench_n${n}_$m.err
  echo "n=$n mode=$m rc=$?" >> gpurun_out/cp_modes.log
done
