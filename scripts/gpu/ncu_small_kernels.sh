CMD="python bench.py --steps 1 --warmup 3 --H 2 --prof-rounds 0 --no-cpu-baseline"
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:route_scan|vocab_scan|losses_finish" -s 3 -c 3 -o gpurun_out/prof26 $CMD > gpurun_out/ncu26.log 2>&1; echo rc=$?
