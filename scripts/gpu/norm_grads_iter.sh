# norm/router-gradient kernels: parity tests, a default bench line, then ncu --set full
# (with source) of one launch each of normed_grad_k and norm_router_partial_k
O=gpurun_out/ng
mkdir -p $O
timeout 900 python -m pytest tests -m gpu -x -q > $O/tests.log 2>&1; echo tests rc=$?; tail -2 $O/tests.log
timeout 600 python bench.py > $O/bench.json 2> $O/bench_err.log; echo bench rc=$?
python -c "import json;d=json.loads([l for l in open('$O/bench.json') if l.startswith('{')][0]);print('value',d['value'],'e2e',d['e2e']['value'],d['clocks'])"
grep -E "norm_router|router_bwd|adamw " $O/bench_err.log
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:normed_grad_k|norm_router_partial_k" -s 4 -c 2 -o $O/ng python bench.py --steps 1 --warmup 3 --H 2 --prof-rounds 0 --no-cpu-baseline > $O/ncu.log 2>&1; echo ncu rc=$?
