# sync phase breakdown at N=4: cfg2 (H=50) and cfg5 (H=1)
for c in "cfg2 50" "cfg5 1"; do set -- $c
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29531 \
    bench.py --gpus 4 --config $1 --H $2 --steps 2 --warmup 3 > gpurun_out/sync_$1.json 2> gpurun_out/sync_$1_err.log
  echo "$1 rc=$? $(grep -c . gpurun_out/sync_$1.json)"; grep -E "sync" gpurun_out/sync_$1_err.log | head -8
done
