O=gpurun_out/m31
mkdir -p $O
C=cfg5
CMD="python bench.py --config $C --steps 1 --warmup 2 --H 2 --prof-rounds 0 --e2e-steps 1 --no-cpu-baseline"
timeout 1500 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:EpiGradW1|normed_grad_k|norm_router_partial_k|EpiStoreF32<128>|EpiDSwiGLUInPlace" -s 20 -c 10 -o $O/full $CMD > $O/ncu_full.log 2>&1; echo full rc=$?
python scripts/ncu_summary.py full $O/full.ncu-rep $O/ncu_full_cfg5_bwd.txt "$CMD"
find $O -name '*.ncu-rep' -size +40M -delete
