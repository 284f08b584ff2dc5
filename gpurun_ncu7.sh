set -x
python bench.py --no-cpu-baseline --steps 1 --warmup 3 > /dev/null 2>&1 || echo bench failed
timeout 900 ncu --set full --import-source on --clock-control none -k regex:grouped_gemm_2cta -s 6 -c 6 -o gpurun_out/gemm2_lib python bench.py --no-cpu-baseline --steps 1 --warmup 3 > gpurun_out/ncu7.log 2>&1
tail -5 gpurun_out/ncu7.log
