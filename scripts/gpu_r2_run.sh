timeout 1500 python -m pytest tests -m gpu -q -s -p no:cacheprovider 2>&1 | grep -E "GRADERR|passed|failed|Error|error|^E |PASS|FAIL|sgd|mixed" | tail -80 > gpurun_out/r2_v8_pytest.txt
timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/r2_v8_cfg5.json 2> gpurun_out/r2_v8_cfg5.err
tail -20 gpurun_out/r2_v8_cfg5.err
cat gpurun_out/r2_v8_pytest.txt
