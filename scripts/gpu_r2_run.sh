timeout 900 compute-sanitizer --tool racecheck --print-limit 20 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "router_kernel and shape0" -p no:cacheprovider > gpurun_out/r2_v10_racecheck.txt 2>&1
tail -15 gpurun_out/r2_v10_racecheck.txt
timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "router_kernel and shape0 or local_step_cfg1" -p no:cacheprovider > gpurun_out/r2_v10_memcheck.txt 2>&1
tail -15 gpurun_out/r2_v10_memcheck.txt
timeout 900 python -m pytest tests/test_dropin.py tests/test_gpu_parity.py -m gpu -q -k "dropin or router_kernel or repeatable" -p no:cacheprovider 2>&1 | tail -5
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r2_v10_cfg5.json 2> gpurun_out/r2_v10_cfg5.err
tail -20 gpurun_out/r2_v10_cfg5.err
