nvidia-smi -L
timeout 600 python -m pytest tests/test_gpu_multi.py -x -q -p no:cacheprovider 2>&1 | tail -6
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 3 --warmup 3 2> gpurun_out/bench2_err.log | tee gpurun_out/bench2.json | head -c 400; echo; tail -5 gpurun_out/bench2_err.log
