O=gpurun_out/ncu_dsw
mkdir -p $O
CMD="python bench.py --config cfg2 --steps 1 --warmup 2 --H 2 --prof-rounds 0 --e2e-steps 0 --no-cpu-baseline"
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:EpiDSwiGLU" -s 2 -c 1 -o $O/dsw $CMD > $O/ncu.log 2>&1; echo rc=$?
ncu -i $O/dsw.ncu-rep --page details --csv 2>/dev/null | grep -E "Duration|Tensor|Issue Slots Busy|Warp Cycles Per Issued|Stall|DRAM Throughput|Compute \(SM\)|Memory Throughput" | head -40 > $O/details.txt
ncu -i $O/dsw.ncu-rep --page raw --csv 2>/dev/null > $O/raw.csv
python - <<'PY'
import csv,io
rows=list(csv.reader(io.StringIO(open('gpurun_out/ncu_dsw/raw.csv').read())))
hdr,units,data=rows[0],rows[1],rows[2:]
d=dict(zip(hdr,data[0]))
for k in sorted(d):
    if any(x in k for x in ['smsp__pcsamp_warps_issue_stalled','tc_cycles_active','gpu__time_duration.sum','dram__bytes_read.sum','dram__bytes_write.sum','issue_active.avg.pct','smsp__average_warp']):
        print(k, d[k])
PY
