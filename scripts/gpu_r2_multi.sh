nvidia-smi --query-gpu=name --format=csv | head -3
timeout 1200 python -m pytest tests/test_gpu_multi.py -m gpu -q -p no:cacheprovider 2>&1 | tail -15 > gpurun_out/r2_m1_pytest.txt
for N in 2 4; do
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus $N --steps 3 --warmup 2 --e2e-steps 1 > gpurun_out/r2_m1_cfg5_n$N.json 2> gpurun_out/r2_m1_cfg5_n$N.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus $N --config cfg5 --H 1 --steps 3 --warmup 2 --e2e-steps 1 > gpurun_out/r2_m1_cfg5_H1_n$N.json 2> gpurun_out/r2_m1_cfg5_H1_n$N.err
done
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29513 bench.py --gpus 4 --config cfg2 --steps 10 --warmup 3 > gpurun_out/r2_m1_cfg2_n4.json 2> gpurun_out/r2_m1_cfg2_n4.err
for f in gpurun_out/r2_m1_*.json; do python -c "
import json,sys;d=json.load(open('$f'));print('$f',d['value'],d['ms_per_step'],d.get('sync'))"; done
cat gpurun_out/r2_m1_pytest.txt
