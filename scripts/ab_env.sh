# A/B of an environment setting on one box, interleaved:
# ab_env.sh PARTS "DISTS" "NAME=VAL ..." (each entry one setting; "-" = none)
PARTS=$1; DISTS=$2; SETS=$3
for rep in 1 2; do
  for d in $DISTS; do
    for e in $SETS; do
      if [ "$e" = "-" ]; then envs=""; else envs="$e"; fi
      echo "$rep $d $e $(env $envs CAD_PERF_DIST=$d timeout 200 python scripts/perf_ca.py 10 $PARTS 2>&1 | grep -v total | awk '{print $1, $2}' | tr '\n' ' ')"
    done
  done
done
