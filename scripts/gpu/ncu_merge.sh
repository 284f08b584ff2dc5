# ncu --set full of the merge kernels (cfg3: merge every round)
CMD="python bench.py --config cfg3 --steps 1 --warmup 3 --prof-rounds 0 --no-cpu-baseline"
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:gram_partial_k|gram_finish_k|merge_apply_k|refresh_shadows_k" -s 4 -c 4 -o gpurun_out/prof_merge $CMD > gpurun_out/ncu_merge.log 2>&1; echo rc=$?
