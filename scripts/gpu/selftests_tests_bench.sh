timeout 120 ./build/gemm2_selftest 2>&1 | tail -12
timeout 120 ./build/gemm_selftest 2>&1 | tail -6
bash scripts/gpu/tests_and_bench.sh
