# BASELINE configs 4 and 5 through bench.py's N>1 leg (run on an N-GPU box):
# gpu_workloads.sh N -> gpurun_out/wl_<workload>_n<N>.json
N=${1:-2}
for wl in ${WORKLOADS:-cfg4 cfg5-uniform cfg5-lognormal cfg5-prolong}; do
  CAD_WORKLOAD=$wl timeout ${WL_TIMEOUT:-600} python -m torch.distributed.run --nnodes=1 --nproc-per-node $N \
    --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus $N --steps 3 --warmup 3 \
    > gpurun_out/wl_${wl}_n$N.json 2> gpurun_out/wl_${wl}_n$N.err
  echo "$wl rc=$?"; python -c "
import json,sys
d=json.loads(open('gpurun_out/wl_${wl}_n$N.json').read().strip().splitlines()[-1])
print(d['value'], d['ms_per_step'], d['imbalance'], d['comm']['hidden_fraction'], d['clocks'].get('sm_mhz'))" || tail -5 gpurun_out/wl_${wl}_n$N.err
done
