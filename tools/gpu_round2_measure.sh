#!/usr/bin/env bash
# One GPU call: the per-threshold ncu counters of the bench workload's view 0
# (tools/profile_sweep.py -> profiles/backward_*.json), then bench.py.
set -u
BENCH_ARGS=("$@")
mkdir -p gpurun_out
M=sm__inst_executed.sum,dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,lts__t_requests_op_red.sum
for spec in "c5_3m_1080p_64views 64 0" "c3_1m_1080p 1 0"; do
  set -- $spec
  timeout 900 ncu --metrics "$M" --clock-control none --print-units base -k regex:k_backward --csv \
    python tools/profile_sweep.py --workload "$1" --views "$2" --view "$3" \
    --specs-out "gpurun_out/specs_$1.json" > "gpurun_out/sweep_$1.csv" 2> "gpurun_out/sweep_$1.err"
  echo "sweep $1 rc=$?"
  python tools/profile_json.py "gpurun_out/specs_$1.json" "gpurun_out/sweep_$1.csv"
done
cp profiles/backward_*.json gpurun_out/ 2>/dev/null
python bench.py "${BENCH_ARGS[@]}" > gpurun_out/bench.json 2> gpurun_out/bench.err
echo "bench rc=$?"
tail -c 2500 gpurun_out/bench.json
