# 4-GPU box: the multi-rank GPU tests (2 and 4 ranks), then bench.py at N=2 and N=4 under
# torchrun over NCCL (one process per GPU)
nvidia-smi -L | wc -l
timeout 900 python -m pytest tests/test_gpu_multi.py -x -q -p no:cacheprovider 2>&1 | tail -4
for n in 2 4; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2951$n bench.py --gpus $n --steps 3 --warmup 3 2> gpurun_out/bench${n}_err.log > gpurun_out/bench${n}.json
  head -c 300 gpurun_out/bench${n}.json; echo; grep -E "sync|adamw" gpurun_out/bench${n}_err.log | head -3
done
