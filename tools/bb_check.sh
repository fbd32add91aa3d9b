#!/usr/bin/env bash
# Block-binning check on the GPU box: list-construction parity tests, the
# forward A/B (block vs the duplicate + tile-sort path) and the C5 kernel list.
set -u
mkdir -p gpurun_out
timeout 600 python -m pytest -x -q tests/test_gpu_raster.py -k "binning_paths or 4k or views_host" > gpurun_out/t_bb.log 2>&1
echo "raster tests rc=$?"; tail -2 gpurun_out/t_bb.log
timeout 300 python -m pytest -x -q tests/test_gpu_parity_full.py -k "small_cases" >> gpurun_out/t_bb.log 2>&1
echo "parity tests rc=$?"; tail -2 gpurun_out/t_bb.log
for wl in c3_1m_1080p c5_3m_1080p_64views; do
  python tools/forward_ab.py --workload $wl --modes block depth-first
done
timeout 200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/fwdbb.csv \
  python tools/forward_ab.py --workload c5_3m_1080p_64views --modes block --reps 1 > /dev/null 2>&1
python tools/ncu_times.py gpurun_out/fwdbb.csv > gpurun_out/fwdbb.txt
tail -14 gpurun_out/fwdbb.txt
