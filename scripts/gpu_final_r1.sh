# Round-end evidence on one GPU: the bench line (with CPU baseline), the
# reference arm, then the ncu captures of scripts/gpu_profile_r1.sh.
set -e
mkdir -p gpurun_out/r1
timeout 900 python bench.py > gpurun_out/r1/bench_n1_final.json 2> gpurun_out/r1/bench_n1_final.err
timeout 900 python bench.py --impl reference > gpurun_out/r1/bench_ref_final.json 2> gpurun_out/r1/bench_ref_final.err
bash scripts/gpu_profile_r1.sh
