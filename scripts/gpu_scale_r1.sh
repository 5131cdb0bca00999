# Multi-GPU bench lines on an N-GPU box (N = 2 or 4): bench.py under torchrun at
# N and (if N = 4) at 2, then BASELINE configs 4/5 at N.
N=${1:-4}
for n in $N $([ "$N" = 4 ] && echo 2); do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
    --master-port 29541 bench.py --gpus $n --steps 5 --warmup 3 > gpurun_out/scale_n$n.json 2> gpurun_out/scale_n$n.err
  echo "n=$n rc=$?"; tail -c 300 gpurun_out/scale_n$n.json
done
WORKLOADS="cfg4 cfg5-lognormal cfg5-prolong cfg5-uniform" bash scripts/gpu_workloads.sh $N
