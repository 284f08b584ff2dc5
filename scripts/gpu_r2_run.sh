O=gpurun_out/m18
mkdir -p $O
run() {  # name env...
  n=$1; shift
  env "$@" timeout 600 python bench.py --steps 3 --warmup 3 --e2e-steps 0 --no-cpu-baseline --prof-rounds 0 > $O/bench_$n.json 2> $O/bench_$n.err
  python -c "
import json;d=json.load(open('$O/bench_$n.json'));print('$n',d['value'],d['ms_per_step'],d['clocks']['sm_mhz'])"
}
run carve1 SPES_SIDE_CARVEOUT=1
run carve0 SPES_SIDE_CARVEOUT=0
run nooverlap SPES_OPT_OVERLAP=0
run carve1b SPES_SIDE_CARVEOUT=1
run carve1_bg256 SPES_SIDE_CARVEOUT=1 SPES_ADAM_BG=256,8,0,2
