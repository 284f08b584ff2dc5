# Round-2 ncu evidence for one configuration ($1, default cfg5): the launch list of one local
# step (per-launch time + DRAM bytes -> profiles/r02/ncu_launches_$1.txt and the
# configuration's roofline.traffic in profiles/ncu_traffic.json), then --set full of one
# launch of each top kernel family, summarised on the box.
C=${1:-cfg5}
O=gpurun_out/ncu_$C
mkdir -p $O
CMD="python bench.py --config $C --steps 1 --warmup 2 --H 2 --prof-rounds 0 --e2e-steps 1 --no-cpu-baseline"
timeout 600 $CMD > $O/plain.json 2> $O/plain.err || echo plain failed
timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $O/launches.csv $CMD > /dev/null 2>&1; echo launches rc=$?
python scripts/ncu_summary.py launches $O/launches.csv $O/ncu_launches_$C.txt $O/ncu_traffic.json $C "$CMD"
timeout 1800 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:adamw_k|grouped_gemm_2cta_kernel|router_fwd_k|normed_grad_k|norm_router_partial_k|combine_bwd_k|combine_fwd_k|permute_tma_k|router_scalar_bwd_k" -s ${SKIP:-140} -c ${COUNT:-40} -o $O/full $CMD > $O/ncu_full.log 2>&1; echo full rc=$?
python scripts/ncu_summary.py full $O/full.ncu-rep $O/ncu_full_$C.txt "$CMD"
# keep the report only when it fits the pull-back limit (the summary above is what is committed)
find $O -name '*.ncu-rep' -size +40M -delete
ls -la $O
