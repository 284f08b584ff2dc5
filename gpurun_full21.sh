start=$(date +%s)
timeout 900 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default_err.log; echo rc=$? secs=$(( $(date +%s) - start ))
start=$(date +%s)
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref_err.log; echo rc=$? secs=$(( $(date +%s) - start ))
cat gpurun_out/bench_ref.json | head -c 1500; echo
tail -3 gpurun_out/bench_ref_err.log
