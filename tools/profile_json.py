"""Regenerate profiles/backward_inst.json and profiles/backward_dram_bytes.json
(read by bench.py for its issue roofline and `traffic`) from the per-policy
ncu CSVs of tools/threshold_sweep_ncu.sh.

    python tools/profile_json.py c3_1m_1080p profiles/r01/thr_sweep_csv/*.csv
"""
import json
import os
import re
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from threshold_sweep_summary import load  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main(workload, paths):
    inst, dram = {}, {}
    for p in paths:
        m = re.search(r"thr_sweep_(\w+?)_(\d+)\.csv$", p)
        if not m:
            continue
        d = load(p)
        if not d:
            continue
        key = f"{m.group(1)}:{m.group(2)}"
        if "sm__inst_executed.sum" in d:
            inst[key] = d["sm__inst_executed.sum"]
        if "dram__bytes_read.sum" in d and "dram__bytes_write.sum" in d:
            dram[key] = d["dram__bytes_read.sum"] + d["dram__bytes_write.sum"]
    src = os.path.relpath(os.path.dirname(os.path.abspath(paths[0])), ROOT)
    out_i = {"_source": f"ncu sm__inst_executed.sum (warp instructions) of one backward launch "
                        f"per policy:threshold, {workload} view 0, {src}",
             workload: dict(sorted(inst.items()))}
    json.dump(out_i, open(os.path.join(ROOT, "profiles", "backward_inst.json"), "w"), indent=1)
    # traffic of the SW-B launch nearest the bench's usual threshold (10-12)
    swb = {int(k.split(":")[1]): v for k, v in dram.items() if k.startswith("sw_b:")}
    if swb:
        t = min(swb, key=lambda x: abs(x - 10))
        out_d = {"_source": f"ncu dram__bytes_read.sum + dram__bytes_write.sum of one SW-B "
                            f"backward launch (t = {t}), {workload} view 0, {src}",
                 workload: swb[t], "per_threshold": {f"sw_b:{k}": v for k, v in sorted(swb.items())}}
        json.dump(out_d, open(os.path.join(ROOT, "profiles", "backward_dram_bytes.json"), "w"),
                  indent=1)
    print(f"{len(inst)} instruction counts, {len(dram)} traffic figures")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2:])
