# ncu --set full of the exact router / norm kernels (cfg2 shapes)
CMD="python bench.py --steps 1 --warmup 3 --H 2 --prof-rounds 0 --no-cpu-baseline"
timeout 300 $CMD > gpurun_out/plain_router.log 2>&1 || echo plain failed
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:router_fwd_k|router_scalar_bwd_k|normed_grad_k|norm_router_partial_k|combine_bwd_k|embed_grad_k" -s 12 -c 6 -o gpurun_out/prof_router $CMD > gpurun_out/ncu_router.log 2>&1; echo rc=$?
