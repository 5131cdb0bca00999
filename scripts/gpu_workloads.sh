# BASELINE configs 3, 4 and 5 through bench.py's N>1 leg (run on an N-GPU box):
# gpu_workloads.sh N -> gpurun_out/wl_<workload>_n<N>.json (+ a summary line each)
N=${1:-2}
for wl in ${WORKLOADS:-cfg3 cfg4 cfg5-uniform cfg5-lognormal cfg5-prolong}; do
  CAD_WORKLOAD=$wl timeout ${WL_TIMEOUT:-600} python -m torch.distributed.run --nnodes=1 --nproc-per-node $N \
    --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus $N --steps ${STEPS:-4} --warmup 3 \
    > gpurun_out/wl_${wl}_n$N.json 2> gpurun_out/wl_${wl}_n$N.err
  echo "$wl rc=$?"; python -c "
import json,sys
d=json.loads(open('gpurun_out/wl_${wl}_n$N.json').read().strip().splitlines()[-1])
c=d['comm']
print(round(d['value'],1), round(d['ms_per_step'],2), {k: round(v,4) for k,v in d['imbalance'].items()},
      'hidden', c['hidden_fraction'], 'all', c['hidden_fraction_all_movement'],
      'nccl', c['nccl'] and (round(c['nccl']['ms_pingpong'],1), c['nccl']['hidden_fraction']),
      'compute', round(c['ms_compute_only'],1), 'signal', round(c['ms_signal'],1), 'wire', round(c['ms_wire'],2),
      'e2e', round(d['e2e']['value'],1), d['clocks'].get('sm_mhz'))" || tail -5 gpurun_out/wl_${wl}_n$N.err
done
