timeout 600 python -m pytest tests -m gpu -x -q -p no:cacheprovider 2>&1 | tail -3
timeout 600 python bench.py --config cfg4 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/bench_cfg4.json 2> gpurun_out/bench_cfg4_err.log; echo cfg4 rc=$?
head -c 250 gpurun_out/bench_cfg4.json; echo; head -8 gpurun_out/bench_cfg4_err.log
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench_err.log; head -c 250 gpurun_out/bench.json; echo; grep router_fwd gpurun_out/bench_err.log
