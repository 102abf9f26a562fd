timeout 1200 ncu --set full --clock-control none -k regex:"conv2_fwd_tc|conv2_bwd_x_tc|conv2_bwd_w_tc|conv1_fwd_tc|conv1_bwd_w_tc|fc1_tc_kernel|fc1_mat_tc|fc1_agg_tc" -c 40 -o /tmp/r02b_tc python bench.py --steps 1 --warmup 3 --e2e-steps 0 --no-cpu-baseline --profile-steps 1 > gpurun_out/r02b_ncu.log 2>&1; echo ncu_rc=$?
ncu -i /tmp/r02b_tc.ncu-rep --page raw --csv > /tmp/r02b_raw.csv
python - <<'PY'
import csv
rows = list(csv.reader(open('/tmp/r02b_raw.csv')))
hdr = rows[0]
keep = [i for i, h in enumerate(hdr) if h in ('ID', 'Kernel Name', 'Grid Size', 'Block Size') or any(x in h for x in (
    'gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum', 'sm__pipe_tensor_cycles_active_realtime.avg.pct',
    'sm__ops_path_tensor_src_fp16_dst_fp32.sum', 'sm__ops_path_tensor_src_tf32_dst_fp32.sum', 'smsp__sass_inst_executed_op_utcmma.sum',
    'sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed', 'l1tex__throughput.avg.pct_of_peak_sustained_active',
    'sm__throughput.avg.pct_of_peak_sustained_elapsed', 'gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed',
    'launch__registers_per_thread', 'smsp__sass_inst_executed_op_tmem_ldt.sum')) and not h.endswith('per_second')]
with open('gpurun_out/r02b_tc_metrics.csv', 'w', newline='') as f:
    w = csv.writer(f)
    for r in rows:
        w.writerow([r[i] for i in keep])
PY
ls -la gpurun_out/
