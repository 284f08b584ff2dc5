CMD="python bench.py --config cfg4 --steps 1 --warmup 3 --H 2 --prof-rounds 0 --no-cpu-baseline"
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:router_fwd" -s 3 -c 1 -o gpurun_out/prof24 $CMD > gpurun_out/ncu24.log 2>&1; echo rc=$?
