O=gpurun_out/m26
mkdir -p $O
for rep in 1 2 3; do for v in 0 1; do
SPES_ADAM_TAIL_FG=$v timeout 600 python bench.py --steps 3 --warmup 3 --e2e-steps 0 --no-cpu-baseline --prof-rounds 0 > $O/bench_cfg5_t${v}_$rep.json 2> $O/bench_cfg5_t${v}_$rep.err
python -c "
import json;d=json.load(open('$O/bench_cfg5_t${v}_$rep.json'));print('cfg5 tail_fg=$v rep$rep',round(d['value']),round(d['ms_per_step'],2),d['clocks']['sm_mhz'])"
done; done
SPES_ADAM_TAIL_FG=1 timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "overlap or local_step_cfg1" 2>&1 | tail -1
