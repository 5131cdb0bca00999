# Round profile capture (run under gpurun, 1 GPU). Plain run first; ncu only
# after it exited 0 with the same arguments.
set -e
CMD="python bench.py --steps 2 --warmup 3 --no-cpu"
$CMD > gpurun_out/prof_bench_plain.json 2> gpurun_out/prof_bench_plain.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"ca_fwd|ca_bwd_dkdv|ca_bwd_dq" -s 3 -c 3 -o gpurun_out/prof_bench $CMD > gpurun_out/ncu_full.log 2>&1
echo done
