CMD="python bench.py --steps 1 --warmup 3 --H 2 --no-cpu-baseline"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:router_fwd -s 4 -c 1 -o gpurun_out/prof14 $CMD > gpurun_out/ncu14.log 2>&1
echo rc=$?; tail -2 gpurun_out/ncu14.log
