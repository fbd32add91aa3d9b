"""Tabulate tools/threshold_sweep_ncu.sh output (one ncu --csv file per policy)."""
import csv
import io
import re
import sys

COLS = [("gpu__time_duration.sum", "ms", 1.0),
        ("smsp__sass_inst_executed_op_global_red.sum", "RED inst (M)", 1e-6),
        ("lts__t_requests_op_red.sum", "L2 red req (M)", 1e-6),
        ("lts__t_sectors_op_red.sum", "L2 red sectors (M)", 1e-6),
        ("lts__d_atomic_input_cycles_active.avg.pct_of_peak_sustained_elapsed", "L2 atom busy %", 1.0),
        ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "FMA pipe %", 1.0),
        ("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "ALU pipe %", 1.0),
        ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue %", 1.0),
        ("sm__inst_executed.sum", "inst (M)", 1e-6)]


def load(path):
    text = open(path).read()
    lines = [l for l in text.splitlines() if l.startswith('"')]
    rows = list(csv.reader(io.StringIO("\n".join(lines))))
    if not rows:
        return {}
    h = rows[0]
    mi, vi, ui = h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit")
    out = {}
    for r in rows[1:]:
        v = float(r[vi].replace(",", ""))
        if r[mi] == "gpu__time_duration.sum":
            v *= {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3,
                  "msecond": 1.0, "ms": 1.0}.get(r[ui].strip(), 1.0)
        else:  # byte counters in bytes
            v *= {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(r[ui].strip(), 1.0)
        out[r[mi]] = v
    return out


def main(paths):
    def key(p):
        m = re.search(r"thr_sweep_(\w+?)_(\d+)\.csv", p)
        order = {"native": 0, "sw_b": 1, "sw_s": 2, "cccl": 3}
        return (order.get(m.group(1), 9), int(m.group(2))) if m else (9, 0)

    print("policy:t     " + " | ".join(c[1] for c in COLS))
    for p in sorted(paths, key=key):
        m = re.search(r"thr_sweep_(\w+?)_(\d+)\.csv", p)
        d = load(p)
        if not d:
            print(f"{m.group(1)}:{m.group(2):3s} (no data)")
            continue
        vals = [f"{d.get(k, float('nan')) * s:9.3f}" for k, _, s in COLS]
        print(f"{m.group(1) + ':' + m.group(2):12s} " + " | ".join(vals))


if __name__ == "__main__":
    main(sys.argv[1:])
