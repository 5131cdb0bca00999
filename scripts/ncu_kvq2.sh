# ncu --set full of the fused dK/dV/dQ kernel and of the two-pass dK/dV kernel
# (one kernel per ncu process), config 2, for the stall comparisons.
tag=${1:-kvq2}
CAD_BWD_FUSED=1 timeout 600 ncu --set full --import-source on --clock-control none -k regex:dkdvq -c 1 -o gpurun_out/${tag}_fused python scripts/perf_ca.py 1 dkdv > gpurun_out/${tag}_ncu.log 2>&1
tail -1 gpurun_out/${tag}_ncu.log
if [ -n "$TWO" ]; then
timeout 600 ncu --set full --import-source on --clock-control none -k regex:dkdv_pair -c 1 -o gpurun_out/${tag}_dkdv2 python scripts/perf_ca.py 1 dkdv >> gpurun_out/${tag}_ncu.log 2>&1
tail -1 gpurun_out/${tag}_ncu.log
fi
