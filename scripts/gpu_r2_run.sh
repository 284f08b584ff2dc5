O=gpurun_out/m25
mkdir -p $O
SPES_GEMM_BAND=8 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_large.py -m gpu -q -p no:cacheprovider -k "local_step or fused or overlap" 2>&1 | tail -1
for c in cfg5 cfg2; do for rep in 1 2; do for b in 0 8 4; do
SPES_GEMM_BAND=$b timeout 600 python bench.py --config $c --steps 3 --warmup 3 --e2e-steps 0 --no-cpu-baseline > $O/bench_${c}_b${b}_$rep.json 2> $O/bench_${c}_b${b}_$rep.err
python -c "
import json;d=json.load(open('$O/bench_${c}_b${b}_$rep.json'));print('$c band$b rep$rep',round(d['value']),round(d['ms_per_step'],2),d['clocks']['sm_mhz'],round(d['roofline']['frac'],3))"
done; done; done
