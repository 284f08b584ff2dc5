O=gpurun_out/m11
mkdir -p $O
for v in 1 2 3; do
SPES_RF_SHAPE=$v timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_large.py -m gpu -q -p no:cacheprovider -x -k "rout or local_step_cfg1 or cfg5" 2>&1 | tail -2 > $O/pytest_v$v.txt
echo "shape $v: $(tail -1 $O/pytest_v$v.txt)"
for c in cfg5 cfg2; do
SPES_RF_SHAPE=$v timeout 600 python bench.py --config $c --steps 3 --warmup 3 --e2e-steps 0 --no-cpu-baseline > $O/bench_${c}_v$v.json 2> $O/bench_${c}_v$v.err
python -c "
import json;d=json.load(open('$O/bench_${c}_v$v.json'));print('$c v$v',d['value'],d['ms_per_step'])"
grep -E "router_fwd" $O/bench_${c}_v$v.err
done; done
