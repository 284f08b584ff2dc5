timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "local_step or stream_overlap" 2>&1 | tail -3
timeout 600 python bench.py --steps 3 --warmup 2 --e2e-steps 0 --no-cpu-baseline > gpurun_out/r2_v16_cfg5.json 2> gpurun_out/r2_v16_cfg5.err
timeout 600 python bench.py --config cfg2 --steps 10 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/r2_v16_cfg2.json 2> gpurun_out/r2_v16_cfg2.err
grep -h "combine_bwd\|router_bwd" gpurun_out/r2_v16_cfg5.err gpurun_out/r2_v16_cfg2.err
python -c "
import json
for c in ['cfg5','cfg2']:
    d=json.load(open('gpurun_out/r2_v16_%s.json'%c));print(c,d['value'],d['ms_per_step'])"
