# Round-1 evidence capture (1 GPU). Each command runs once plainly (exit 0)
# before the same command runs under ncu; each ncu process profiles one kernel.
set -e
mkdir -p gpurun_out/r1
python bench.py --steps 2 --warmup 3 --no-cpu > gpurun_out/r1/bench_plain.json 2> gpurun_out/r1/bench_plain.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r1/launches.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu > gpurun_out/r1/ncu_launch.log 2>&1
python scripts/prof_config2.py > gpurun_out/r1/prof_plain.log 2>&1
for k in ca_fwd_pair_kernel ca_bwd_dkdv_pair_kernel ca_bwd_dq_pair_kernel ca_delta_kernel; do
  ncu --set full --clock-control none --import-source on -k regex:$k -c 1 -o gpurun_out/r1/full_$k \
    python scripts/prof_config2.py > gpurun_out/r1/ncu_$k.log 2>&1
done
echo done
