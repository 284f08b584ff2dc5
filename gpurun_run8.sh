timeout 120 ./build/gemm_selftest 2>&1 | grep -E "FAIL|TFLOP|SELFTEST"
timeout 600 python -m pytest tests -m gpu -x -q -p no:cacheprovider 2>&1 | tail -4
timeout 300 python bench.py --no-cpu-baseline 2>gpurun_out/bench_err.log > gpurun_out/bench.json; head -c 200 gpurun_out/bench.json; echo; head -24 gpurun_out/bench_err.log
