# Round profile capture (run under gpurun, 1 GPU). Plain run first; ncu only
# after it exited 0 with the same arguments. One kernel per ncu process (the
# backward kernels' replays fail when several are captured in one process).
set -e
R=${ROUND:-r2}
CMD="python bench.py --steps 2 --warmup 3 --no-cpu"
$CMD > gpurun_out/prof_bench_plain.json 2> gpurun_out/prof_bench_plain.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${R}_launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1
for k in ca_fwd_pair ca_bwd_dkdv_pair ca_bwd_dq_pair ca_delta; do
  ncu --set full --clock-control none --import-source on -k regex:"$k" -s 1 -c 1 -o gpurun_out/${R}_full_$k $CMD > gpurun_out/ncu_full_$k.log 2>&1 || tail -5 gpurun_out/ncu_full_$k.log
done
echo done
