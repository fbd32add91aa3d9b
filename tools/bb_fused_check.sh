#!/usr/bin/env bash
# Fused block-binning level 1 (DW_BB_FUSED, default on): parity tests with it
# on, memcheck/racecheck of the driver, forward A/B against the entry scan +
# radix pass (DW_BB_FUSED=0), and the C5 kernel list.
set -u
mkdir -p gpurun_out
timeout 600 python -m pytest -x -q tests/test_gpu_raster.py -k "binning_paths or 4k or views_host or overflow or concentrated" > gpurun_out/t_bbf.log 2>&1
echo "raster tests rc=$?"; tail -2 gpurun_out/t_bbf.log
timeout 600 python -m pytest -x -q tests/test_gpu_parity_full.py -k "small_cases" >> gpurun_out/t_bbf.log 2>&1
echo "parity tests rc=$?"; tail -2 gpurun_out/t_bbf.log
for tool in memcheck racecheck; do
  timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 20 \
    python tools/sanitize_driver.py > gpurun_out/sanitizer_bbf_$tool.txt 2>&1
  echo "$tool rc=$?"; tail -2 gpurun_out/sanitizer_bbf_$tool.txt
done
for rep in 1 2; do
  for wl in c5_3m_1080p_64views c3_1m_1080p; do
    for f in 0 1; do
      echo -n "fused=$f " >> gpurun_out/bbf_ab.jsonl
      DW_BB_FUSED=$f timeout 300 python tools/forward_ab.py --workload $wl --modes block >> gpurun_out/bbf_ab.jsonl
    done
  done
done
python - <<'PY'
import json
for l in open("gpurun_out/bbf_ab.jsonl"):
    tag, js = l.split(" ", 1)
    d = json.loads(js); b = d["block"]
    print(f'{tag} {d["workload"][:12]:12s} fwd {b["forward_ms"]:.4f} min {b["min_ms"]:.4f} binning {b["stages"]["binning"]:.4f}')
PY
timeout 200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/fwdbbf.csv \
  python tools/forward_ab.py --workload c5_3m_1080p_64views --modes block --reps 1 > /dev/null 2>&1
python tools/ncu_times.py gpurun_out/fwdbbf.csv > gpurun_out/fwdbbf.txt
tail -16 gpurun_out/fwdbbf.txt
