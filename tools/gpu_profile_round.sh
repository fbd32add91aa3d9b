#!/usr/bin/env bash
# One GPU session's measurement set (run from the repo root on the B200 box):
# threshold-sweep counters, one full ncu capture of the hot kernel, the bench
# line, and the ncu launch list of a short bench command.
set -u
mkdir -p gpurun_out
bash tools/threshold_sweep_ncu.sh c3_1m_1080p > gpurun_out/thr_sweep.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_backward -s 1 -c 1 \
  -o gpurun_out/bwd_full python tools/profile_backward.py --policy sw_b --threshold 10 \
  > gpurun_out/ncu_full.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_forward -s 0 -c 1 \
  -o gpurun_out/fwd_full python tools/profile_backward.py --policy sw_b --threshold 10 --reps 0 \
  >> gpurun_out/ncu_full.log 2>&1
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2>> gpurun_out/bench.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 3 --e2e-steps 1 \
  --no-cpu-baseline > gpurun_out/bench_under_ncu.log 2>&1
python tools/launch_summary.py gpurun_out/launches.csv > gpurun_out/launches_summary.txt 2>&1
