CMD="python bench.py --steps 1 --warmup 3 --H 2 --no-cpu-baseline"
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k "regex:vocab|embed_grad|route_|losses|norm_router|head_ce" --csv --log-file gpurun_out/launches17.csv $CMD > /dev/null 2>&1; echo rc=$?
