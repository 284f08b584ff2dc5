# bench.py at N=2 and N=4 under torchrun (one process per GPU, NCCL + NVLink sync)
for n in 2 4; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2957$n bench.py --gpus $n --steps 3 --warmup 3 2> gpurun_out/bench${n}_err.log > gpurun_out/bench${n}.json
  echo "n=$n rc=$?"
done
