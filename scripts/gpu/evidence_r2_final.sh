# Round-2 evidence set on one B200: the GPU test suite, the driver's default bench (cfg5,
# with cpu_baseline), the reference arm, the other configurations at N=1, and the ncu
# launch lists of a cfg5 and a cfg2 step (per-launch time and DRAM bytes -> roofline.traffic)
O=gpurun_out/ev5
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -s -p no:cacheprovider 2>&1 | grep -E "GRADERR|passed|failed|Error|error|^E |FAIL|PASS" | tail -60 > $O/pytest_gpu.txt
timeout 900 python bench.py > $O/bench_default.json 2> $O/bench_default.err; echo default rc=$?
timeout 900 python bench.py --impl reference > $O/bench_reference.json 2> $O/bench_reference.err; echo ref rc=$?
for c in cfg2 cfg3 cfg4; do
timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > $O/bench_${c}_n1.json 2> $O/bench_${c}_n1.err; echo $c rc=$?
done
for c in cfg5 cfg2; do
CMD="python bench.py --config $c --steps 1 --warmup 2 --H 2 --prof-rounds 0 --e2e-steps 1 --no-cpu-baseline"
timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $O/launches_$c.csv $CMD > /dev/null 2>&1; echo ncu $c rc=$?
python scripts/ncu_summary.py launches $O/launches_$c.csv $O/ncu_launches_$c.txt $O/ncu_traffic.json $c "$CMD"
rm -f $O/launches_$c.csv
done
for f in $O/*.json; do python -c "
import json;d=json.load(open('$f'));print('$f',d.get('value'),d.get('ms_per_step'),(d.get('e2e') or {}).get('value'),(d.get('cpu_baseline') or {}).get('value'))" 2>/dev/null; done
tail -3 $O/pytest_gpu.txt
# the smoke the driver runs
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1; tail -1 $O/smoke.txt
# ncu --set full of the top kernel families of one cfg5 step (summarised on the box)
C=cfg5
CMD="python bench.py --config $C --steps 1 --warmup 2 --H 2 --prof-rounds 0 --e2e-steps 1 --no-cpu-baseline"
timeout 1800 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:adamw_k|grouped_gemm_2cta_kernel|router_fwd_k|normed_grad_k|norm_router_partial_k|combine_bwd_k|combine_fwd_k|permute_tma_k|router_scalar_bwd_k" -s 140 -c 44 -o $O/full $CMD > $O/ncu_full.log 2>&1; echo full rc=$?
python scripts/ncu_summary.py full $O/full.ncu-rep $O/ncu_full_$C.txt "$CMD"
find $O -name '*.ncu-rep' -size +40M -delete
