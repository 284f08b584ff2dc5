# ncu --set full of one launch of each top kernel of a cfg2 local step (the launch list
# is in evidence.sh); summarise with scripts/ncu_summary.py full
O=gpurun_out/ev
mkdir -p $O
CMD="python bench.py --steps 1 --warmup 3 --H 2 --prof-rounds 0 --no-cpu-baseline"
timeout 1500 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:adamw_k|grouped_gemm_2cta_kernel|router_fwd_k|normed_grad_k|norm_router_partial_k|combine_bwd_k|combine_fwd_k" -s 40 -c 16 -o $O/full2 $CMD > $O/ncu_full2.log 2>&1; echo full rc=$?
