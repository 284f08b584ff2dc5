nvidia-smi -L | wc -l
timeout 600 python -m pytest tests/test_gpu_multi.py -x -q -p no:cacheprovider 2>&1 | tail -4
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 4 --steps 3 --warmup 3 2> gpurun_out/bench4_err.log | tee gpurun_out/bench4.json | head -c 300; echo; grep -E "sync|adamw" gpurun_out/bench4_err.log | head -3
