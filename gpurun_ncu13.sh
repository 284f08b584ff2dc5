CMD="python bench.py --steps 1 --warmup 3 --H 2 --no-cpu-baseline"
timeout 300 $CMD > gpurun_out/plain13.log 2>&1 || echo plain failed
timeout 1200 ncu --set full --clock-control none --import-source on -s 200 -c 32 -o gpurun_out/prof13 $CMD > gpurun_out/ncu13.log 2>&1
echo rc=$?; tail -2 gpurun_out/ncu13.log
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches13.csv $CMD > /dev/null 2>&1; echo rc=$?
