CMD="python bench.py --steps 1 --warmup 3 --H 2 --no-cpu-baseline"
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches16.csv $CMD > /dev/null 2>&1; echo rc=$?
