"""A/B of the forward over environment switches read per launch (e.g.
DW_FWD_DB): V views of a workload rendered without host synchronisation, back
to back on one stream and over four streams, settings interleaved; images of
every arm must equal the first arm's bit for bit.

    python tools/ab_forward_env.py --settings "DW_FWD_DB=0;DW_FWD_DB=1"
"""
import argparse
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="c5_3m_1080p_64views")
    ap.add_argument("--views", type=int, default=16)
    ap.add_argument("--rounds", type=int, default=4)
    ap.add_argument("--settings", default="DW_FWD_DB=0;DW_FWD_DB=1")
    a = ap.parse_args()
    import torch

    from paper_2401_05345_b200.rasterizer import GaussianRasterizer
    from paper_2401_05345_b200.scene import CONFIGS, make_scene, orbit_cameras

    P, W, H, hc, nv = CONFIGS[a.workload]
    dev = torch.device("cuda:0")
    sc = {k: torch.from_numpy(v).to(dev) for k, v in make_scene(P, W, H, seed=0, high_contention=hc).items()}
    args = [sc[k] for k in ("means3D", "scales", "rotations", "opacities", "colors")]
    cams = orbit_cameras(W, H, max(nv, a.views))[: a.views]
    rs = []
    for c in cams:
        r = GaussianRasterizer()
        r.render_forward(*args, c)
        r.reserve(P, W, H, r.num_rendered + r.num_rendered // 2 + 4096)
        rs.append(r)
    imgs = [torch.empty((3, H, W), device=dev) for _ in cams]
    rads = [torch.empty(P, dtype=torch.int32, device=dev) for _ in range(4)]
    sts = [torch.cuda.Stream() for _ in range(4)]

    def apply(v):
        for kv in v.split(","):
            k, _, val = kv.partition("=")
            os.environ[k] = val

    def run(ns):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for s in sts[:ns]:
            s.wait_event(e0)
        for k, (r, c) in enumerate(zip(rs, cams)):
            r.render_forward_async(*args, c, imgs[k], rads[k % 4], stream=sts[k % ns])
        for s in sts[:ns]:
            torch.cuda.current_stream().wait_stream(s)
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / len(rs)

    settings = a.settings.split(";")
    res = {f"{v}|{ns}": [] for v in settings for ns in (1, 4)}
    ref = None
    for v in settings:
        apply(v)
        run(1)
        got = torch.stack(imgs).cpu()
        if ref is None:
            ref = got
        assert torch.equal(got, ref), f"images differ: {v}"
    for _ in range(a.rounds):
        for v in settings:
            apply(v)
            for ns in (1, 4):
                res[f"{v}|{ns}"].append(round(run(ns), 4))
    print(json.dumps({"workload": a.workload, "views": a.views,
                      "median_ms_per_view": {k: statistics.median(x) for k, x in res.items()}}))


if __name__ == "__main__":
    main()
