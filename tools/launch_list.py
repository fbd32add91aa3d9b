"""Per-launch table (time, DRAM bytes) from an ncu --csv metrics dump.

    python tools/launch_list.py gpurun_out/launches.csv
"""
import csv
import sys


def main(path):
    rows = [r for r in csv.DictReader(l for l in open(path) if l.startswith('"'))]
    cur, order = {}, []
    for r in rows:
        k = (r["ID"], r["Kernel Name"][:60])
        if k not in cur:
            cur[k] = {}
            order.append(k)
        cur[k][r["Metric Name"]] = float(r["Metric Value"].replace(",", ""))
    tot = 0.0
    for k in order:
        m = cur[k]
        us = m.get("gpu__time_duration.sum", 0) / 1e3
        tot += us
        mb = (m.get("dram__bytes_read.sum", 0) + m.get("dram__bytes_write.sum", 0)) / 1e6
        print(f"{k[0]:>4} {k[1]:<60} {us:9.1f} us {mb:8.1f} MB")
    print(f"total {tot:.1f} us")


if __name__ == "__main__":
    main(sys.argv[1])
