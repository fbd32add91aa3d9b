"""A/B: a rank's chain of backwards (one rasterizer per view, all rendered
beforehand, adding into one gradient) launched (a) as bench.py's timed loop
did -- an event pair around every launch, (b) plain with events only around
the step, (c) chained (dw_render_backward_chained after the first: no
grid-completion wait, launch tails overlap). L2 flushed between steps.

    python tools/ab_bwd_chain.py --views 16 --rounds 5
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
    ap.add_argument("--rounds", type=int, default=5)
    ap.add_argument("--threshold", type=int, default=15)
    ap.add_argument("--modes", default="events,plain,chained")
    ap.add_argument("--grad-stride", type=int, default=9,
                    help="floats per gradient row (12: a -DDW_GRAD_STRIDE=12 A/B build)")
    a = ap.parse_args()
    import torch

    from paper_2401_05345_b200 import warpred as wr
    from paper_2401_05345_b200.rasterizer import GaussianRasterizer, render_backward_views
    from paper_2401_05345_b200.scene import CONFIGS, make_dL_dpixels, make_scene, orbit_cameras

    P, W, H, hc, nviews = CONFIGS[a.workload]
    dev = torch.device("cuda:0")
    sc = {k: torch.from_numpy(v).to(dev) for k, v in make_scene(P, W, H, seed=0, high_contention=hc).items()}
    args = [sc[k] for k in ("means3D", "scales", "rotations", "opacities", "colors")]
    cams = orbit_cameras(W, H, max(nviews, a.views))[: a.views]
    rasts = []
    for c in cams:
        r = GaussianRasterizer()
        r.render_forward(*args, c)
        rasts.append(r)
    dLs = [torch.from_numpy(make_dL_dpixels(W, H, seed=1 + k)).to(dev) for k in range(a.views)]
    grad = torch.zeros((P, a.grad_stride), device=dev)
    pol = wr.Policy(wr.PolicyKind.sw_b, a.threshold)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731

    def step(mode):
        # "chained+DW_BWD_WARPS=2": a mode with environment switches set for it
        mode, *envs = mode.split("+")
        for k in ("DW_BWD_WARPS",):
            os.environ.pop(k, None)
        for kv in envs:
            k, _, v = kv.partition("=")
            os.environ[k] = v
        flush.fill_(1.0)
        torch.cuda.synchronize()
        e0, e1 = ev(), ev()
        e0.record()
        grad.zero_()
        for i, (r, dL) in enumerate(zip(rasts, dLs) if mode != "batch" else ()):
            if mode == "events":
                a0, a1 = ev(), ev()
                a0.record()
                r.render_backward(dL, pol, grad=grad)
                a1.record()
            elif mode != "batch":
                r.render_backward(dL, pol, grad=grad, chained=(mode == "chained" and i > 0))
        if mode == "batch":  # dw_render_backward_views: chain + padded rows + fold
            render_backward_views(rasts, dLs, pol, grad)
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / len(rasts)

    modes = tuple(a.modes.split(","))
    for m in modes:
        step(m)
    res = {m: [] for m in modes}
    for _ in range(a.rounds):
        for m in modes:
            res[m].append(round(step(m), 4))
    step(modes[-1])
    g_last = grad.clone()
    step(modes[0])
    rel = float((grad - g_last).norm() / grad.norm())
    print(json.dumps({"workload": a.workload, "views": a.views, "ms_per_view": res,
                      "median": {m: statistics.median(v) for m, v in res.items()},
                      "lib": os.environ.get("DISTWAR_LIB", "libdistwar.so"),
                      f"grad_rel_diff_{modes[-1]}_vs_{modes[0]}": rel}))


if __name__ == "__main__":
    main()
