# cfg5 sync-interval sweep H = 1..500 at N = 2 and 4 (BASELINE.json configs[4]):
# one warm-up round and two timed rounds per point, no e2e / profiled rounds.
O=gpurun_out/sweep_r2_final
mkdir -p $O
for N in ${NS:-2 4}; do
for H in 1 2 5 10 20 50 100 200 500; do
  S=2; [ $H -ge 200 ] && S=1
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
    --master-port $((29600 + H)) bench.py --gpus $N --config cfg5 --H $H --steps $S --warmup 1 \
    --e2e-steps 0 --prof-rounds 0 --no-cpu-baseline > $O/cfg5_n${N}_H$H.json 2> $O/cfg5_n${N}_H$H.err
  python -c "
import json; d=json.load(open('$O/cfg5_n${N}_H$H.json'))
s=d.get('sync') or {}
print('N=$N H=$H', round(d['value']), 'tok/s', round(d['ms_per_step'],1), 'ms/round', 'sync', round(s.get('ms',0),1), 'ms', round(s.get('frac',0),3))" | tee -a $O/summary.txt
done
done
