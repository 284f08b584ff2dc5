O=gpurun_out/ev5m
mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_multi.py -m gpu -q -p no:cacheprovider 2>&1 | tail -5 > $O/pytest_gpu_multi.txt
cat $O/pytest_gpu_multi.txt
for N in 2 4; do
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2951$N bench.py --gpus $N --steps 3 --warmup 3 > $O/bench_cfg5_n$N.json 2> $O/bench_cfg5_n$N.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2952$N bench.py --gpus $N --impl reference --steps 2 --warmup 1 > $O/bench_reference_n$N.json 2> $O/bench_reference_n$N.err
done
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 4 --config cfg2 --steps 10 --warmup 3 > $O/bench_cfg2_n4.json 2> $O/bench_cfg2_n4.err
for f in $O/*.json; do python -c "
import json;d=json.load(open('$f'));print('$f',d.get('value'),d.get('ms_per_step'),(d.get('e2e') or {}).get('value'),(d.get('sync') or {}).get('ms'),(d.get('sync') or {}).get('frac'))" 2>/dev/null; done
