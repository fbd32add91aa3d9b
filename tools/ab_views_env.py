"""A/B of the batched host path (dw_render_views_host, 64 views, images
downloaded) over the values of environment switches it reads per call
(--settings "A=1,B=2;A=3" sets several per arm; a bare value sets --env):
DW_VIEWS_STACK (views per stacked frame, profiles/r02/ab/stacked_views.md);
the PDL record (profiles/r02/ab/pdl_two_streams.md) used a since-removed
DW_VIEWS_PDL. Settings interleave, so box drift averages out.

    python tools/ab_views_env.py --env DW_VIEWS_STACK --settings "1;2;3" --rounds 4
"""
import argparse
import json
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="c5_3m_1080p_64views")
    ap.add_argument("--views", type=int, default=64)
    ap.add_argument("--rounds", type=int, default=4)
    ap.add_argument("--env", default="DW_VIEWS_STACK")
    ap.add_argument("--settings", default="1;2;3")
    a = ap.parse_args()
    import torch

    from paper_2401_05345_b200 import warpred as wr
    from paper_2401_05345_b200.rasterizer import GaussianRasterizer, render_views_host
    from paper_2401_05345_b200.scene import CONFIGS, make_dL_dpixels, make_scene, orbit_cameras

    P, W, H, hc, _ = CONFIGS[a.workload]
    V = a.views
    sc = make_scene(P, W, H, seed=0, high_contention=hc)
    cams = orbit_cameras(W, H, V)
    dL = make_dL_dpixels(W, H, seed=1)
    pol = wr.Policy(wr.PolicyKind.sw_b, 15)
    pin = {k: torch.from_numpy(v).pin_memory() for k, v in sc.items()}
    dL_h = torch.from_numpy(dL).unsqueeze(0).expand(V, -1, -1, -1).contiguous().pin_memory()
    img_h = torch.empty((V, 3, H, W)).pin_memory()
    grad_h = torch.empty((P, 9)).pin_memory()
    ptrs = [pin[k].data_ptr() for k in ("means3D", "scales", "rotations", "opacities", "colors")]
    r = GaussianRasterizer()
    s = torch.cuda.current_stream()
    settings = a.settings.split(";")

    def apply(v):
        for kv in v.split(","):
            k, _, val = kv.rpartition("=")
            os.environ[k or a.env] = val
    res = {v: [] for v in settings}
    for v in settings:  # warm-up each setting (allocations, reserves)
        apply(v)
        render_views_host(r, ptrs, P, cams, dL_h.data_ptr(), pol, img_h.data_ptr(),
                          grad_h.data_ptr(), s)
    torch.cuda.synchronize()
    for _ in range(a.rounds):
        for v in settings:
            apply(v)
            t0 = time.perf_counter()
            render_views_host(r, ptrs, P, cams, dL_h.data_ptr(), pol, img_h.data_ptr(),
                              grad_h.data_ptr(), s)
            torch.cuda.synchronize()
            res[v].append(round((time.perf_counter() - t0) * 1e3, 2))
    print(json.dumps({"workload": a.workload, "views": V, "env": a.env, "ms_per_step": res,
                      "median": {v: statistics.median(x) for v, x in res.items()}}))


if __name__ == "__main__":
    main()
