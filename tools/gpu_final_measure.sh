#!/usr/bin/env bash
# End-of-round measurement set (repo root, one B200): bench line, reference
# arm, per-config table, the ncu launch list of a short bench command, and
# ncu full captures of the hot kernel (C5 view 0, the timed chain's
# row-major order) and of the forward blend.
set -u
mkdir -p gpurun_out
timeout 600 python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err
echo "bench rc=$?"
timeout 400 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref_final.json 2>> gpurun_out/bench_final.err
echo "reference rc=$?"
timeout 900 python tools/config_table.py > gpurun_out/config_table.jsonl 2> gpurun_out/config_table.err
echo "config table rc=$?"
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_final.csv python bench.py --steps 3 --warmup 3 --e2e-steps 1 \
  --no-cpu-baseline > gpurun_out/bench_under_ncu.log 2>&1
echo "launch list rc=$?"
python tools/launch_summary.py gpurun_out/launches_final.csv > gpurun_out/launches_final_summary.txt 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_forward -s 0 -c 1 \
  -o gpurun_out/fwd_full_c5 python tools/profile_backward.py --workload c5_3m_1080p_64views \
  --policy sw_b --threshold 16 --reps 0 > gpurun_out/ncu_fwd.log 2>&1
echo "ncu forward rc=$?"
