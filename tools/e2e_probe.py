"""Where does the end-to-end step (dw_render_views_host) spend its time?
Times, on one scene and V views: (a) the host-buffer call with and without
image download, (b) the same forward + backward of every view from device
buffers on one stream (no copies), (c) the pinned copies alone.

    python tools/e2e_probe.py --views 64
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="c3_1m_1080p")
    ap.add_argument("--views", type=int, default=64)
    ap.add_argument("--reps", type=int, default=3)
    a = ap.parse_args()
    import torch

    from paper_2401_05345_b200 import warpred as wr
    from paper_2401_05345_b200.rasterizer import GaussianRasterizer, render_views_host
    from paper_2401_05345_b200.scene import CONFIGS, make_dL_dpixels, orbit_cameras, make_scene

    P, W, H, hc, _ = CONFIGS[a.workload]
    V = a.views
    dev = torch.device("cuda:0")
    sc = make_scene(P, W, H, seed=0, high_contention=hc)
    cams = orbit_cameras(W, H, V)
    dL = make_dL_dpixels(W, H, seed=1)
    pol = wr.Policy(wr.PolicyKind.sw_b, 8)
    pin = {k: torch.from_numpy(v).pin_memory() for k, v in sc.items()}
    dL_h = torch.from_numpy(dL).unsqueeze(0).expand(V, -1, -1, -1).contiguous().pin_memory()
    img_h = torch.empty((V, 3, H, W)).pin_memory()
    grad_h = torch.empty((P, 9)).pin_memory()
    ptrs = [pin[k].data_ptr() for k in ("means3D", "scales", "rotations", "opacities", "colors")]
    r = GaussianRasterizer()
    out = {"views": V}

    def timed(fn):
        fn()
        torch.cuda.synchronize()
        ts = []
        for _ in range(a.reps):
            t0 = time.perf_counter()
            fn()
            torch.cuda.synchronize()
            ts.append(time.perf_counter() - t0)
        return min(ts) * 1e3

    s = torch.cuda.current_stream()
    out["host_call_ms"] = timed(lambda: render_views_host(r, ptrs, P, cams, dL_h.data_ptr(), pol,
                                                          img_h.data_ptr(), grad_h.data_ptr(), s))
    out["host_call_noimg_ms"] = timed(lambda: render_views_host(r, ptrs, P, cams, dL_h.data_ptr(),
                                                                pol, None, grad_h.data_ptr(), s))
    d = {k: v.to(dev) for k, v in pin.items()}
    dLd = dL_h[0].to(dev)
    grad = torch.zeros((P, 9), device=dev)
    r2 = GaussianRasterizer()

    def device_loop():
        for k in range(V):
            r2.render_forward(d["means3D"], d["scales"], d["rotations"], d["opacities"],
                              d["colors"], cams[k])
            r2.render_backward(dLd, pol, grad=grad)

    out["device_loop_ms"] = timed(device_loop)
    dst = torch.empty_like(dL_h, device=dev)
    out["h2d_dL_ms"] = timed(lambda: dst.copy_(dL_h, non_blocking=True))
    out["d2h_img_ms"] = timed(lambda: img_h.copy_(dst, non_blocking=True))
    out["h2d_GBps"] = dL_h.numel() * 4 / out["h2d_dL_ms"] / 1e6
    out["d2h_GBps"] = img_h.numel() * 4 / out["d2h_img_ms"] / 1e6
    print(json.dumps(out))


if __name__ == "__main__":
    main()
