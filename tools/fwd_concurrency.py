"""Do two views' forwards overlap? Times V forwards serially on one stream and
in pairs on two streams (two rasterizers), nosync (device-side counts), and
the same for forward + backward per view, C5 scene.

    python tools/fwd_concurrency.py --views 16
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
    a = ap.parse_args()
    import torch

    from paper_2401_05345_b200 import warpred as wr
    from paper_2401_05345_b200.rasterizer import GaussianRasterizer
    from paper_2401_05345_b200.scene import CONFIGS, make_dL_dpixels, make_scene, orbit_cameras

    P, W, H, hc, _ = CONFIGS[a.workload]
    dev = torch.device("cuda:0")
    sc = {k: torch.from_numpy(v).to(dev) for k, v in make_scene(P, W, H, seed=0).items()}
    args = [sc[k] for k in ("means3D", "scales", "rotations", "opacities", "colors")]
    cams = orbit_cameras(W, H, 64)[: a.views]
    dL = torch.from_numpy(make_dL_dpixels(W, H, seed=1)).to(dev)
    rs = [GaussianRasterizer(), GaussianRasterizer()]
    st = [torch.cuda.Stream(), torch.cuda.Stream()]
    for r in rs:  # size the no-sync reserves
        r.render_forward(*args, cams[0])
        r.reserve(P, W, H, int(r.num_rendered * 1.5) + 4096)
    grad = torch.zeros((P, 9), device=dev)
    imgs = [torch.empty((3, H, W), device=dev) for _ in rs]
    radii = [torch.empty(P, dtype=torch.int32, device=dev) for _ in rs]
    pol = wr.Policy(wr.PolicyKind.sw_b, 16)

    def run(pairs, backward):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for s in st:
            s.wait_event(e0)
        for k, cam in enumerate(cams):
            b = k & 1 if pairs else 0
            rs[b].render_forward_async(*args, cam, imgs[b], radii[b], stream=st[b])
            if backward:
                rs[b].render_backward(dL, pol, grad=grad, stream=st[b])
        cur = torch.cuda.current_stream()
        for s in st:
            cur.wait_stream(s)
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / len(cams)

    def run_grouped():
        """F(k) || F(k+1), then B(k), B(k+1): forwards of a pair overlap each
        other, backwards run alone (each fills the GPU)."""
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for s in st:
            s.wait_event(e0)
        for k in range(0, len(cams), 2):
            done = []
            for b in range(2):
                if k + b < len(cams):
                    rs[b].render_forward_async(*args, cams[k + b], imgs[b], radii[b], stream=st[b])
                    ev = torch.cuda.Event()
                    ev.record(st[b])
                    done.append(ev)
            for ev in done:
                st[0].wait_event(ev)
            for b in range(len(done)):
                rs[b].render_backward(dL, pol, grad=grad, stream=st[0])
            ev = torch.cuda.Event()
            ev.record(st[0])
            st[1].wait_event(ev)  # the next pair's forward reuses state 1
        cur = torch.cuda.current_stream()
        for s in st:
            cur.wait_stream(s)
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / len(cams)

    def run_waves(nstreams):
        """All views' forwards rotating over `nstreams` streams (one state per
        view), then their backwards as one chain -- the batched host path's
        device work without its copies."""
        rs_all = [GaussianRasterizer() for _ in cams]
        sts = [torch.cuda.Stream() for _ in range(nstreams)]
        for r in rs_all:
            r.render_forward(*args, cams[0])
        imgs_all = [torch.empty((3, H, W), device=dev) for _ in cams]
        rad_all = [torch.empty(P, dtype=torch.int32, device=dev) for _ in cams]
        for r in rs_all:
            r.reserve(P, W, H, int(r.num_rendered * 1.5) + 4096)

        def once():
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for s in sts:
                s.wait_event(e0)
            for k, cam in enumerate(cams):
                rs_all[k].render_forward_async(*args, cam, imgs_all[k], rad_all[k],
                                               stream=sts[k % nstreams])
            cur = torch.cuda.current_stream()
            e_f = torch.cuda.Event(enable_timing=True)
            for s in sts:
                cur.wait_stream(s)
            e_f.record()
            for k in range(len(cams)):
                rs_all[k].render_backward(dL, pol, grad=grad, chained=k > 0)
            e1.record()
            torch.cuda.synchronize()
            return e0.elapsed_time(e_f) / len(cams), e0.elapsed_time(e1) / len(cams)

        once()
        runs = [once() for _ in range(3)]
        return (round(statistics.median(r[0] for r in runs), 4),
                round(statistics.median(r[1] for r in runs), 4))

    out = {}
    for ns in (1, 2, 4):
        f, t = run_waves(ns)
        out[f"waves_{ns}streams_fwd"] = f
        out[f"waves_{ns}streams_total"] = t
    run_grouped()
    out["fwd_pair_then_bwd"] = round(statistics.median(run_grouped() for _ in range(3)), 4)
    for name, pairs, bwd in (("fwd_serial", False, False), ("fwd_two_streams", True, False),
                             ("fwd_bwd_serial", False, True), ("fwd_bwd_two_streams", True, True)):
        run(pairs, bwd)
        out[name] = round(statistics.median(run(pairs, bwd) for _ in range(3)), 4)
    print(json.dumps({"workload": a.workload, "views": a.views, "ms_per_view": out}))


if __name__ == "__main__":
    main()
