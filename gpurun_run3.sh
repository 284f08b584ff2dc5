set -x
timeout 600 python -m pytest tests -m gpu -x -q -p no:cacheprovider 2>&1 | tail -5
CMD="python bench.py --steps 1 --warmup 1 --H 2 --no-cpu-baseline"
timeout 300 $CMD > gpurun_out/plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu1.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:grouped_gemm -s 18 -c 9 -o gpurun_out/prof_gemm $CMD > gpurun_out/ncu2.log 2>&1
echo rc=$?
tail -3 gpurun_out/plain.log
ls -la gpurun_out
