# SM clock / power while the forward runs: pair vs single-CTA forward (50 reps each)
for impl in 1 0; do
  nvidia-smi --query-gpu=clocks.sm,power.draw,clocks_throttle_reasons.active --format=csv,noheader -lms 250 > gpurun_out/pw_$impl.csv &
  pid=$!
  CAD_FWD_PAIR=$impl timeout 200 python scripts/perf_ca.py 60 fwd 2>&1 | head -1
  kill $pid
  echo "pair=$impl"; sort gpurun_out/pw_$impl.csv | uniq -c | sort -rn | head -8
done
