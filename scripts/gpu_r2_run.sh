for bg in "64,16,0,2" "64,4,1,4" "64,4,2,4" "64,4,2,2" "128,4,1,4" "64,8,4,2"; do
SPES_ADAM_BG=$bg timeout 600 python bench.py --steps 3 --warmup 2 --e2e-steps 1 --prof-rounds 0 --no-cpu-baseline > "gpurun_out/r2_v11_bg$bg.json" 2> "gpurun_out/r2_v11_bg$bg.err"
python -c "
import json;d=json.load(open('gpurun_out/r2_v11_bg$bg.json'));print('$bg',d['value'],d['ms_per_step'],d['clocks'])"
done
