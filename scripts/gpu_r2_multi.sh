for cfg in "17 1" "20 1" "20 0"; do set -- $cfg
SPES_SYNC_CHUNK=$1 SPES_SYNC_ORDER=$2 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 4 --config cfg5 --H 1 --steps 3 --warmup 2 --e2e-steps 0 --prof-rounds 0 --no-cpu-baseline > gpurun_out/r2_m6_$1_$2.json 2> gpurun_out/r2_m6_$1_$2.err
python -c "
import json;d=json.load(open('gpurun_out/r2_m6_$1_$2.json'));print('chunk $1 order $2',d['value'],d['ms_per_step'],d['sync']['ms'],d['sync']['frac'])"
done
timeout 900 python -m pytest tests/test_gpu_multi.py -m gpu -q -p no:cacheprovider 2>&1 | tail -3
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29513 bench.py --gpus 4 --config cfg2 --steps 10 --warmup 3 --e2e-steps 0 --prof-rounds 0 --no-cpu-baseline > gpurun_out/r2_m6_cfg2_n4.json 2> gpurun_out/r2_m6_cfg2_n4.err
python -c "
import json;d=json.load(open('gpurun_out/r2_m6_cfg2_n4.json'));print('cfg2 n4',d['value'],d['ms_per_step'],d['sync']['ms'],d['sync']['frac'])"
