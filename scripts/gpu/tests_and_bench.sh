timeout 600 python -m pytest tests -m gpu -x -q -p no:cacheprovider 2>&1 | tail -5
timeout 300 python bench.py --no-cpu-baseline 2>gpurun_out/bench_err.log > gpurun_out/bench.json; head -c 300 gpurun_out/bench.json; echo; head -25 gpurun_out/bench_err.log
