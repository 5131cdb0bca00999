# Light ncu capture of the three CA kernels in the bench (DRAM/L2 bytes, tensor %).
set -e
CMD="python bench.py --steps 2 --warmup 3 --no-cpu"
$CMD > /dev/null 2>&1
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,sm__ops_path_tensor_op_utchmma_src_bf16_dst_fp32_sparsity_off.avg.pct_of_peak_sustained_elapsed,sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active,sm__cycles_elapsed.avg.per_second,lts__t_bytes.sum,lts__t_sector_hit_rate.pct,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed,smsp__inst_issued.avg.pct_of_peak_sustained_active --clock-control none -k regex:"${1:-ca_fwd|ca_bwd_dkdv|ca_bwd_dq}" -s 3 -c 3 --csv --log-file gpurun_out/traffic.csv $CMD > gpurun_out/ncu_t.log 2>&1
python - <<'PY'
import csv
rows=[r for r in csv.reader(open('gpurun_out/traffic.csv')) if len(r)>10]
h=rows[0]; ik=h.index('Kernel Name'); im=h.index('Metric Name'); iu=h.index('Metric Unit'); iv=h.index('Metric Value')
for r in rows[1:]: print(r[ik].split('(')[0][:24], r[im][:48], r[iu], r[iv])
PY
