for sms in 148 136 124; do
SPES_GEMM_SMS=$sms timeout 600 python bench.py --steps 3 --warmup 2 --e2e-steps 0 --prof-rounds 0 --no-cpu-baseline > gpurun_out/r2_v18_sms$sms.json 2> gpurun_out/r2_v18_sms$sms.err
python -c "
import json
d=json.load(open('gpurun_out/r2_v18_sms$sms.json'));print('gemm sms $sms',d['value'],d['ms_per_step'],d['clocks'])"
done
SPES_GEMM_SMS=124 SPES_ADAM_BG=128,16,0,2 timeout 600 python bench.py --steps 3 --warmup 2 --e2e-steps 0 --prof-rounds 0 --no-cpu-baseline > gpurun_out/r2_v18_sms124b.json 2> gpurun_out/r2_v18_sms124b.err
python -c "
import json
d=json.load(open('gpurun_out/r2_v18_sms124b.json'));print('gemm sms 124 bg128',d['value'],d['ms_per_step'])"
