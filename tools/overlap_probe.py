"""Would the batched host path gain from running the next wave's forwards
CONCURRENTLY with the current wave's backward chain (forwards on
high-priority streams, the chain on a low-priority one) instead of one phase
after the other? Device-only, C5 scene: views A (rendered) are back-propagated
as one chain while views B are rendered, vs the same work in sequence.

    python tools/overlap_probe.py --views 8
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
    ap.add_argument("--views", type=int, default=8)
    ap.add_argument("--streams", type=int, default=4)
    a = ap.parse_args()
    import torch

    from paper_2401_05345_b200 import warpred as wr
    from paper_2401_05345_b200.rasterizer import GaussianRasterizer, render_backward_views
    from paper_2401_05345_b200.scene import CONFIGS, make_dL_dpixels, make_scene, orbit_cameras

    P, W, H, hc, _ = CONFIGS[a.workload]
    dev = torch.device("cuda:0")
    sc = {k: torch.from_numpy(v).to(dev) for k, v in make_scene(P, W, H, seed=0, high_contention=hc).items()}
    args = [sc[k] for k in ("means3D", "scales", "rotations", "opacities", "colors")]
    n = a.views
    cams = orbit_cameras(W, H, 2 * n)
    A = [GaussianRasterizer() for _ in range(n)]
    B = [GaussianRasterizer() for _ in range(n)]
    for r, c in zip(A + B, cams):
        r.render_forward(*args, c)
        r.reserve(P, W, H, r.num_rendered + r.num_rendered // 2 + 4096)
    for r, c in zip(A + B, cams):
        r.render_forward(*args, c)
    dLs = [torch.from_numpy(make_dL_dpixels(W, H, seed=1 + k)).to(dev) for k in range(n)]
    grad = torch.zeros((P, 9), device=dev)
    pol = wr.Policy(wr.PolicyKind.sw_b, 16)
    lo, hi = torch.cuda.Stream.priority_range() if hasattr(torch.cuda.Stream, "priority_range") else (0, -1)
    fwd_hi = [torch.cuda.Stream(priority=-1) for _ in range(a.streams)]
    fwd_lo = [torch.cuda.Stream(priority=0) for _ in range(a.streams)]
    bwd_lo = torch.cuda.Stream(priority=0)
    imgs = [torch.empty((3, H, W), device=dev) for _ in range(a.streams)]
    rads = [torch.empty(P, dtype=torch.int32, device=dev) for _ in range(a.streams)]

    def run(mode):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fs = fwd_hi if mode == "overlap_prio" else fwd_lo
        for s in fs + [bwd_lo]:
            s.wait_event(e0)
        if mode == "sequential":
            with torch.cuda.stream(bwd_lo):
                render_backward_views(A, dLs, pol, grad, stream=bwd_lo)
            ev = torch.cuda.Event()
            ev.record(bwd_lo)
            for s in fs:
                s.wait_event(ev)
        else:
            render_backward_views(A, dLs, pol, grad, stream=bwd_lo)
        for k, (r, c) in enumerate(zip(B, cams[n:])):
            j = k % a.streams
            r.render_forward_async(*args, c, imgs[j], rads[j], stream=fs[j])
        cur = torch.cuda.current_stream()
        for s in fs + [bwd_lo]:
            cur.wait_stream(s)
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / n

    out = {}
    for m in ("sequential", "overlap", "overlap_prio"):
        run(m)
        out[m] = round(statistics.median(run(m) for _ in range(4)), 4)
    print(json.dumps({"workload": a.workload, "views": n, "ms_per_view_pair": out}))


if __name__ == "__main__":
    main()
