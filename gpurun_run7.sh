CMD="python bench.py --steps 1 --warmup 1 --H 2 --no-cpu-baseline"
timeout 300 $CMD > gpurun_out/plain7.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:router_fwd|normed_grad|norm_router_partial|adamw|expert_shadows|head_shadows|embed_grad" -s 20 -c 8 -o gpurun_out/prof8 $CMD > gpurun_out/ncu7.log 2>&1
echo rc=$?; tail -2 gpurun_out/ncu7.log
