# N=1 evidence set: the driver's default bench (cfg5, with cpu_baseline), the reference arm,
# the other BASELINE configurations, and the GPU test suite
O=gpurun_out/ev2
mkdir -p $O
timeout 900 python bench.py > $O/bench_default.json 2> $O/bench_default.err; echo default rc=$?
timeout 900 python bench.py --impl reference > $O/bench_reference.json 2> $O/bench_reference.err; echo ref rc=$?
for c in cfg2 cfg3 cfg4; do
timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > $O/bench_${c}_n1.json 2> $O/bench_${c}_n1.err; echo $c rc=$?
done
SPES_DSWIGLU_TMA=0 timeout 600 python bench.py --config cfg4 --steps 10 --warmup 3 --e2e-steps 0 --no-cpu-baseline > $O/bench_cfg4_n1_unstaged.json 2> $O/bench_cfg4_n1_unstaged.err
grep -h gemm_bwd_dh $O/bench_cfg4_n1.err $O/bench_cfg4_n1_unstaged.err
timeout 1500 python -m pytest tests -m gpu -q -s -p no:cacheprovider 2>&1 | grep -E "GRADERR|passed|failed|Error|error|^E |FAIL" | tail -40 > $O/pytest_gpu.txt
for f in $O/*.json; do python -c "
import json;d=json.load(open('$f'));print('$f',d.get('value'),d.get('ms_per_step'),(d.get('e2e') or {}).get('value'),(d.get('cpu_baseline') or {}).get('value'))"; done
tail -3 $O/pytest_gpu.txt
