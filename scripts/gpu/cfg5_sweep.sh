# cfg5 sync-interval sweep (H at N in {2, 4}) on a 4-GPU box, one torchrun per
# point; each point's JSON line goes to gpurun_out/sweep/cfg5_n<N>_h<H>.json
mkdir -p gpurun_out/sweep
for n in 2 4; do
  for h in 1 5 50 200; do
    timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
      --master-port 2960$n bench.py --gpus $n --config cfg5 --H $h --steps 2 --warmup 3 --prof-rounds 0 \
      > gpurun_out/sweep/cfg5_n${n}_h${h}.json 2> gpurun_out/sweep/cfg5_n${n}_h${h}_err.log
    echo "n=$n h=$h rc=$? $(head -c 160 gpurun_out/sweep/cfg5_n${n}_h${h}.json | tail -c 60)"
  done
done
