O=gpurun_out/m14
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -s -p no:cacheprovider -k "router_gradient_paths" 2>&1 | grep -E "GRADERR|passed|failed|Error|^E " | tail -20 > $O/pytest.txt
cat $O/pytest.txt
for c in cfg4; do for tc in 0 1; do
SPES_ROUTER_TC=$tc timeout 600 python bench.py --config $c --steps 5 --warmup 3 --e2e-steps 0 --no-cpu-baseline > $O/bench_${c}_tc$tc.json 2> $O/bench_${c}_tc$tc.err
python -c "
import json;d=json.load(open('$O/bench_${c}_tc$tc.json'));print('$c tc$tc',d['value'],d['ms_per_step'])"
grep -E "norm_router|router_grad" $O/bench_${c}_tc$tc.err
done; done
