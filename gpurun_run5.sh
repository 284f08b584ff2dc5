CMD="python bench.py --steps 1 --warmup 1 --H 2 --no-cpu-baseline"
timeout 300 $CMD > gpurun_out/plain5.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:router_bwd|norm_router|router_fwd|head_ce|losses_k|route_scatter|embed_grad|route_scan|adamw" -s 18 -c 10 -o gpurun_out/prof_misc $CMD > gpurun_out/ncu5.log 2>&1
echo rc=$?; tail -3 gpurun_out/ncu5.log
