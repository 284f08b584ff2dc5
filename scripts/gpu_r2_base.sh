set -x
nproc; free -g; nvidia-smi --query-gpu=name,memory.total --format=csv
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > gpurun_out/r2_base_pytest.txt
timeout 600 python bench.py --config cfg5 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r2_base_cfg5.json 2> gpurun_out/r2_base_cfg5.err
tail -30 gpurun_out/r2_base_cfg5.err
cat gpurun_out/r2_base_pytest.txt
