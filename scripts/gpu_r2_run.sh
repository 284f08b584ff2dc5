O=gpurun_out/m23
mkdir -p $O
for c in cfg5 cfg2; do for rep in 1 2; do for v in 0 1; do
SPES_NG_ALLK=$v timeout 600 python bench.py --config $c --steps 3 --warmup 3 --e2e-steps 0 --no-cpu-baseline > $O/bench_${c}_v${v}_$rep.json 2> $O/bench_${c}_v${v}_$rep.err
python -c "
import json;d=json.load(open('$O/bench_${c}_v${v}_$rep.json'));print('$c v$v rep$rep',round(d['value']),round(d['ms_per_step'],2))"
grep -E "router_bwd" $O/bench_${c}_v${v}_$rep.err
done; done; done
