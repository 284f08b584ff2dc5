CMD="python bench.py --steps 1 --warmup 3 --H 2 --prof-rounds 0 --no-cpu-baseline"
timeout 300 $CMD > gpurun_out/plain19.log 2>&1 || echo plain failed
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches19.csv $CMD > /dev/null 2>&1; echo rc1=$?
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:adamw_k|EpiSwiGLU|EpiDSwiGLU" -s 6 -c 3 -o gpurun_out/prof19 $CMD > gpurun_out/ncu19.log 2>&1; echo rc2=$?
