CMD="python bench.py --steps 1 --warmup 3 --H 2 --prof-rounds 0 --no-cpu-baseline"
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:normed_grad|combine_fwd|norm_router_partial|combine_bwd" -s 8 -c 4 -o gpurun_out/prof22 $CMD > gpurun_out/ncu22.log 2>&1; echo rc=$?
