# A/B of the fused dK/dV/dQ kernel against the two-pass backward and its
# diagnostic builds (scripts/build_variants.sh), config 2, one box.
[ -z "$NOTEST" ] && CAD_BWD_FUSED=1 timeout 300 python -m pytest tests/test_ca_bwd_gpu.py tests/test_ca_edge_gpu.py -x -q 2>&1 | tail -2
for v in ${VARS:-default nored nodq}; do
  if [ $v = default ]; then unset CAD_LIB_PATH; else export CAD_LIB_PATH=paper_2510_18121_b200/lib/variants/libcad_$v.so; fi
  echo "$v $(CAD_BWD_FUSED=1 timeout 200 python scripts/perf_ca.py 3 dkdv,dq 2>&1 | grep -v total | tr '\n' ' ')"
done
unset CAD_LIB_PATH
echo "two-pass $(timeout 200 python scripts/perf_ca.py 3 dkdv,dq 2>&1 | grep -v total | tr '\n' ' ')"
