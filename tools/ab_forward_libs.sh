#!/usr/bin/env bash
# Forward A/B across library builds (block binning variants):
#   bash tools/ab_forward_libs.sh OUT.jsonl lib1.so [lib2.so ...]   (libs relative to csrc/)
set -u
out=$1; shift
for rep in 1 2; do
  for wl in c5_3m_1080p_64views c3_1m_1080p; do
    for lib in "$@"; do
      echo -n "$lib " >> "$out"
      DISTWAR_LIB=paper_2401_05345_b200/csrc/$lib timeout 300 python tools/forward_ab.py \
        --workload $wl --modes block >> "$out" 2>> "$out.err"
    done
  done
done
python - "$out" <<'PY'
import json, sys
for l in open(sys.argv[1]):
    lib, js = l.split(" ", 1)
    d = json.loads(js)
    b = d["block"]
    print(f'{lib:28s} {d["workload"][:12]:12s} fwd {b["forward_ms"]:.4f} min {b["min_ms"]:.4f} binning {b["stages"]["binning"]:.4f}')
PY
