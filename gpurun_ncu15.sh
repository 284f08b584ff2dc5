CMD="python bench.py --steps 1 --warmup 3 --H 2 --no-cpu-baseline"
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:EpiDSwiGLU -s 2 -c 1 -o gpurun_out/prof15 $CMD > gpurun_out/ncu15.log 2>&1
echo rc=$?; tail -2 gpurun_out/ncu15.log
