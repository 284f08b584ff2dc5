# Round-end evidence on one B200: default bench line (with cpu_baseline), the reference
# arm, the ncu launch list of one local step and one --set full capture of the top
# kernels, and the other BASELINE configs. Summarise here with scripts/ncu_summary.py.
O=gpurun_out/ev
mkdir -p $O
timeout 600 python bench.py > $O/default.json 2> $O/default_err.log; echo default rc=$?
timeout 600 python bench.py --impl reference > $O/reference.json 2> $O/reference_err.log; echo reference rc=$?
CMD="python bench.py --steps 1 --warmup 3 --H 2 --prof-rounds 0 --no-cpu-baseline"
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $O/launches.csv $CMD > /dev/null 2>&1; echo launches rc=$?
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:adamw_k|EpiSwiGLU|EpiDSwiGLU|EpiHeadCE|router_fwd_k|norm_router_partial_k" -s 12 -c 6 -o $O/full $CMD > $O/ncu_full.log 2>&1; echo full rc=$?
for c in cfg3 cfg4 cfg5; do
  timeout 600 python bench.py --config $c --steps 2 --warmup 3 --no-cpu-baseline > $O/$c.json 2> $O/${c}_err.log; echo $c rc=$?
done
head -c 400 $O/default.json; echo
