mkdir -p gpurun_out/m30
timeout 900 python -X faulthandler -m pytest tests -m gpu -q -s -p no:cacheprovider > gpurun_out/m30/pytest_full.txt 2>&1
echo "pytest rc=$?"; grep -E "^FAILED|^E  |Fatal" gpurun_out/m30/pytest_full.txt | head -5; tail -1 gpurun_out/m30/pytest_full.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/m30/bench_default.json 2> gpurun_out/m30/bench_default.err; echo "bench rc=$?"
python -c "
import json;d=json.load(open('gpurun_out/m30/bench_default.json'));print(round(d['value']),round(d['ms_per_step'],1),d['e2e']['value'],d['roofline']['frac'],d['roofline']['traffic'],d['clocks']['sm_mhz'],d['gpu_launches'])"
