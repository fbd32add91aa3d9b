#!/usr/bin/env bash
# ncu counters for the SW-B balancing-threshold sweep (north_star: justify the
# chosen threshold by L2 RED throughput, lts__t_sectors_op_red and FP32 pipe
# utilisation). One uncounted k_backward launch per policy/threshold on view 0
# of the workload; writes gpurun_out/thr_sweep_<policy>_<t>.csv, a summary
# table, and metrics.csv in the reference's experiment layout
# (tools/metrics_csv.py).
set -u
WL=${1:-c3_1m_1080p}
METRICS=gpu__time_duration.sum,lts__t_sectors_op_red.sum,lts__t_requests_op_red.sum,\
smsp__sass_inst_executed_op_global_red.sum,lts__d_atomic_input_cycles_active.avg.pct_of_peak_sustained_elapsed,\
sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_fma.sum,\
sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,\
sm__inst_executed.sum,sm__cycles_elapsed.max,smsp__sass_thread_inst_executed_op_fadd_pred_on.sum,\
smsp__pcsamp_warps_issue_stalled_lg_throttle,smsp__pcsamp_warps_issue_stalled_mio_throttle,\
smsp__pcsamp_warps_issue_stalled_long_scoreboard,smsp__pcsamp_sample_count,\
dram__bytes_read.sum,dram__bytes_write.sum
mkdir -p gpurun_out
for spec in native:0 sw_b:0 sw_b:4 sw_b:8 sw_b:10 sw_b:12 sw_b:16 sw_b:20 sw_b:24 sw_b:28 sw_b:32 sw_s:0 sw_s:16 sw_s:32 cccl:0; do
  pol=${spec%%:*}; t=${spec##*:}
  timeout 300 ncu --metrics "$METRICS" --clock-control none -k regex:k_backward -s 1 -c 1 --csv \
    python tools/profile_backward.py --workload "$WL" --policy "$pol" --threshold "$t" --reps 2 \
    > "gpurun_out/thr_sweep_${pol}_${t}.csv" 2>/dev/null
  echo "$spec rc=$?"
done
python tools/threshold_sweep_summary.py gpurun_out/thr_sweep_*.csv > gpurun_out/thr_sweep_summary.txt
python tools/metrics_csv.py gpurun_out/thr_sweep_*.csv > gpurun_out/metrics.csv
cat gpurun_out/thr_sweep_summary.txt
