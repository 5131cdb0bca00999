# A/B of the LPT per-unit fixed cost (CAD_SCHED_FIXED for fwd/dQ units,
# CAD_SCHED_KV_FIXED for dK/dV units) on one box, interleaved.
for rep in 1 2; do
  for d in ${DISTS:-pretrain uniform}; do
    for f in ${FIXED:-0 1 3 6}; do
      echo "$rep $d fixed=$f $(CAD_SCHED_FIXED=$f CAD_SCHED_KV_FIXED=$((f * 8)) CAD_PERF_DIST=$d timeout 200 python scripts/perf_ca.py 10 fwd,dkdv,dq 2>&1 | grep -v total | awk '{print $1, $2}' | tr '\n' ' ')"
    done
  done
done
