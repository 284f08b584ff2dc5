# ncu --set full of the dW GEMMs with MaskedAdamW in the epilogue (SPES_FUSED_OPT=1)
CMD="python bench.py --steps 1 --warmup 3 --H 2 --prof-rounds 0 --no-cpu-baseline"
export SPES_FUSED_OPT=1
timeout 300 $CMD > gpurun_out/plain_fused.log 2>&1 || echo plain failed
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:EpiAdamW" -s 4 -c 2 -o gpurun_out/prof_fused $CMD > gpurun_out/ncu_fused.log 2>&1; echo rc=$?
