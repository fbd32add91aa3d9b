"""ncu driver for the trace-driven kernels on the reference's own C3 trace
(SURVEY §8(d) trace family): one launch of k_reduce_trace per policy, in a
fixed order, for `ncu -k regex:k_reduce_trace --metrics ...`; then
`--summarize CSV` turns the ncu CSV into DRAM bytes / algorithmic bytes /
HBM fraction per policy (profiles/r02/ncu/trace_c3_dram.md).

    ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
        -k regex:k_reduce_trace --csv python tools/profile_trace.py > trace.csv
    python tools/profile_trace.py --summarize trace.csv
"""
import csv
import io
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

TRACE_C3 = dict(num_primitives=1_000_000, params_per_primitive=9, image_width=1920,
                image_height=1080, mean_fragment_span=48.0, fragments_per_pixel_mean=8.0,
                locality=0.99, activity_prob=0.7, seed=1)
ORDER = [("native", 0), ("sw_b", 8), ("sw_s", 8), ("cccl", 0)]


def run():
    from paper_2401_05345_b200 import warpred as wr

    tr = wr.generate(wr.SceneSpec(**TRACE_C3))
    d = wr.DeviceTrace(tr)
    for name, t in ORDER:
        wr.gpu_run(d, wr.Policy(wr.parse_policy_kind(name), t), want_sums=False)
    print(json.dumps({"records": d.records, "params": d.params, "P": d.num_primitives}),
          file=sys.stderr)


def summarize(path):
    text = open(path).read()
    text = text[text.find('"ID"'):]
    per = {}
    names = {}
    for r in csv.DictReader(io.StringIO(text)):
        per.setdefault(int(r["ID"]), {})[r["Metric Name"]] = (
            float(r["Metric Value"].replace(",", "")), r["Metric Unit"])
        names[int(r["ID"])] = r["Kernel Name"]
    peaks = json.load(open(os.path.join(os.path.dirname(os.path.dirname(
        os.path.abspath(__file__))), "MEASURED_PEAKS.json"))) if os.path.exists(
        "MEASURED_PEAKS.json") else {}
    hbm = peaks.get("hbm_gbs") or 6545.3
    R, N, P = 519532, 9, 1_000_000
    alg = R * (132 + 128 * N) + 4 * P * N
    print("| policy | ms (ncu) | DRAM read MB | DRAM write MB | DRAM / algorithmic | algorithmic GB/s | of HBM |")
    print("|---|---|---|---|---|---|---|")
    kinds = {"0": "native", "1": "sw_s", "2": "sw_b", "3": "cccl"}
    for i in sorted(per):
        # k_reduce_trace<N, policy, COUNT>: the timed (COUNT = 0) instantiation
        args = names[i].split("<", 1)[1].split(">", 1)[0].replace(" ", "").split(",")
        if args[2] != "0":
            continue
        name = kinds[args[1]]
        t = dict(ORDER)[name]
        m = per[i]
        ms = m["gpu__time_duration.sum"][0] / 1e6
        rd = m["dram__bytes_read.sum"][0] / 1e6
        wr_ = m["dram__bytes_write.sum"][0] / 1e6
        gbs = alg / (ms * 1e-3) / 1e9
        print(f"| {name}:{t} | {ms:.4f} | {rd:.1f} | {wr_:.1f} | {(rd + wr_) * 1e6 / alg:.3f} | "
              f"{gbs:.0f} | {gbs / hbm:.3f} |")
    print(f"\nalgorithmic bytes per launch = R (132 + 128 N) + 4 P N = {alg / 1e6:.1f} MB "
          f"(R = {R}, N = {N}, P = {P}); HBM peak {hbm} GB/s")


if __name__ == "__main__":
    if len(sys.argv) > 2 and sys.argv[1] == "--summarize":
        summarize(sys.argv[2])
    else:
        run()
