# A/B of variant libraries (scripts/build_variants.sh) on one box, interleaved:
# ab_variants.sh PARTS DIST "v1 v2 ..." (v = default or a variant name)
PARTS=$1; DISTS=$2; VARS=$3
for rep in 1 2; do
  for d in $DISTS; do
    for v in $VARS; do
      if [ $v = default ]; then unset CAD_LIB_PATH; else export CAD_LIB_PATH=paper_2510_18121_b200/lib/variants/libcad_$v.so; fi
      echo "$rep $d $v $(CAD_PERF_DIST=$d timeout 200 python scripts/perf_ca.py 10 $PARTS 2>&1 | grep -v total | tr '\n' ' ')"
    done
  done
done
