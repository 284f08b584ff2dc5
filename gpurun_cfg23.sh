for c in cfg4 cfg3; do
timeout 600 python bench.py --config $c --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$c.json 2> gpurun_out/bench_${c}_err.log; echo $c rc=$?
head -c 300 gpurun_out/bench_$c.json; echo; tail -2 gpurun_out/bench_${c}_err.log
done
timeout 900 python bench.py --config cfg5 --steps 1 --warmup 3 --H 4 --no-cpu-baseline > gpurun_out/bench_cfg5.json 2> gpurun_out/bench_cfg5_err.log; echo cfg5 rc=$?
head -c 300 gpurun_out/bench_cfg5.json; echo; tail -3 gpurun_out/bench_cfg5_err.log
