"""Regenerate profiles/backward_inst.json and profiles/backward_dram_bytes.json
(read by bench.py for its issue roofline and roofline `traffic`) from an ncu
CSV of tools/profile_sweep.py (one k_backward launch per spec, in spec order).

    python tools/profile_json.py gpurun_out/specs.json gpurun_out/sweep.csv

Entries are keyed "<workload>@view<k>/<views>" -> {spec: value}; other keys in
the files are kept.
"""
import csv
import io
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def launches(path):
    """[{metric: value}] per kernel launch, in launch order."""
    text = open(path).read()
    start = text.find('"ID"')
    rows = list(csv.DictReader(io.StringIO(text[start:])))
    out, order = {}, []
    for row in rows:
        i = int(row["ID"])
        if i not in out:
            out[i] = {"kernel": row["Kernel Name"]}
            order.append(i)
        v = row["Metric Value"].replace(",", "")
        try:
            out[i][row["Metric Name"]] = float(v)
        except ValueError:
            pass
    return [out[i] for i in order]


def main(specs_path, csv_path):
    sp = json.load(open(specs_path))
    ls = launches(csv_path)
    per = sp.get("launches_per_spec", 1)  # > 1: the spec's LAST launch is the measured one
    if len(ls) != per * len(sp["specs"]):
        raise SystemExit(f"{len(ls)} launches for {len(sp['specs'])} specs x {per}")
    ls = ls[per - 1::per]
    key = f"{sp['workload']}@view{sp['view']}/{sp['views']}"
    src = os.path.relpath(os.path.abspath(csv_path), ROOT)
    files = {"inst": os.path.join(ROOT, "profiles", "backward_inst.json"),
             "dram": os.path.join(ROOT, "profiles", "backward_dram_bytes.json"),
             "time": os.path.join(ROOT, "profiles", "backward_ncu_ms.json")}
    tables = {}
    for name, p in files.items():
        tables[name] = json.load(open(p)) if os.path.exists(p) else {}
    inst, dram, tms = {}, {}, {}
    for spec, l in zip(sp["specs"], ls):
        inst[spec] = l.get("sm__inst_executed.sum")
        if "dram__bytes_read.sum" in l and "dram__bytes_write.sum" in l:
            dram[spec] = l["dram__bytes_read.sum"] + l["dram__bytes_write.sum"]
        if "gpu__time_duration.sum" in l:
            tms[spec] = l["gpu__time_duration.sum"] * 1e-6  # ns -> ms
    tables["inst"]["_source"] = ("ncu sm__inst_executed.sum (warp instructions) of one backward "
                                 "launch per policy:threshold (tools/profile_sweep.py)")
    tables["dram"]["_source"] = ("ncu dram__bytes_read.sum + dram__bytes_write.sum of one "
                                 "backward launch per policy:threshold (tools/profile_sweep.py)")
    tables["time"]["_source"] = "ncu gpu__time_duration.sum (cold, serialised) per launch, ms"
    for name, d in (("inst", inst), ("dram", dram), ("time", tms)):
        tables[name][key] = {"csv": src, "instances": sp["instances"], **d}
        json.dump(tables[name], open(files[name], "w"), indent=1)
    print(key, len(inst), "specs")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
