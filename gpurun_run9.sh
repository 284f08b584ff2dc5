CMD="python bench.py --steps 1 --warmup 1 --H 2 --no-cpu-baseline"
timeout 300 $CMD > gpurun_out/plain9.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:grouped_gemm" -s 18 -c 9 -o gpurun_out/prof9 $CMD > gpurun_out/ncu9.log 2>&1
echo rc=$?; tail -2 gpurun_out/ncu9.log
