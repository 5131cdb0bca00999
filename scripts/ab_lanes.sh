# A/B of CAD_PUSH_LANES on an N-GPU box (config 3, NCCL line off), interleaved
N=${1:-2}
for rep in 1 2; do
  for lanes in 1 2 4; do
    CAD_PUSH_LANES=$lanes CAD_NCCL_LINE=0 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N \
      --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus $N --steps 4 --warmup 3 > /tmp/lanes.json 2>/dev/null
    python -c "
import json
d=json.loads(open('/tmp/lanes.json').read().strip().splitlines()[-1]); c=d['comm']
print('$rep lanes $lanes', round(d['ms_per_step'],2), 'signal', round(c['ms_signal'],2), 'compute', round(c['ms_compute_only'],2), 'wire', round(c['ms_wire'],2), 'exposed', round(c['exposed_wire_ms'],2), 'probe', c['nvlink_probe_gbs'])"
  done
done
