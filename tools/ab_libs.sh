#!/usr/bin/env bash
# A/B the in-tree library against alternative builds on the BASELINE scenes.
#   [AB_REPEAT=n] [AB_WORKLOADS="..."] bash tools/ab_libs.sh OUT.jsonl POLICIES lib1.so [lib2.so ...]
#   (libs relative to csrc/; repeats interleave the libs to average out box drift)
set -u
out=$1; pols=$2; shift 2
WLS=${AB_WORKLOADS:-c3_1m_1080p c2_100k_800 c4_200k_contention_1080p}
for rep in $(seq 1 ${AB_REPEAT:-1}); do
for wl in $WLS; do
  for lib in "$@"; do
    DISTWAR_LIB=paper_2401_05345_b200/csrc/$lib timeout 300 python tools/ab_backward.py \
      --workload $wl --policies "$pols" --reps 10 >> "$out" 2>> "$out.err"
  done
done
done
python - "$out" <<'PY'
import json, sys
for l in open(sys.argv[1]):
    d = json.loads(l)
    print(d["lib"].split("csrc/")[-1][:28], d["workload"][:14], round(d["forward_ms"], 4), d["backward_ms"])
PY
