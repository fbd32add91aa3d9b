"""ncu driver for the backward's per-threshold counters: one forward of a view
of a workload, then ONE render_backward launch per (policy, threshold) spec in
a fixed order (every SW-B threshold 0..32, plus native / SW-S / CCCL), each
synchronised, so `ncu -k regex:k_backward` sees exactly one launch per spec.
The spec order is written to --specs-out for tools/profile_json.py.

    ncu --metrics sm__inst_executed.sum,dram__bytes_read.sum,... --csv \
        -k regex:k_backward python tools/profile_sweep.py --workload c5_3m_1080p_64views \
        --views 64 --view 0 --specs-out gpurun_out/specs.json > gpurun_out/sweep.csv
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

SPECS = ["native:0"] + [f"sw_b:{t}" for t in range(33)] + ["sw_s:0", "sw_s:8", "sw_s:16",
                                                            "sw_s:32", "cccl:0"]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="c3_1m_1080p")
    ap.add_argument("--views", type=int, default=1, help="orbit camera count (1: view 0 camera)")
    ap.add_argument("--view", type=int, default=0)
    ap.add_argument("--specs-out", required=True)
    a = ap.parse_args()
    import torch

    from paper_2401_05345_b200 import warpred as wr
    from paper_2401_05345_b200.rasterizer import GaussianRasterizer, render_backward_views
    from paper_2401_05345_b200.scene import (CONFIGS, make_camera, make_dL_dpixels, make_scene,
                                             orbit_cameras)

    P, W, H, hc, _ = CONFIGS[a.workload]
    dev = torch.device("cuda:0")
    sc = {k: torch.from_numpy(v).to(dev)
          for k, v in make_scene(P, W, H, seed=0, high_contention=hc).items()}
    cam = orbit_cameras(W, H, a.views)[a.view] if a.views > 1 else make_camera(W, H)
    dL = torch.from_numpy(make_dL_dpixels(W, H, seed=1 + a.view)).to(dev)
    r = GaussianRasterizer()
    r.render_forward(sc["means3D"], sc["scales"], sc["rotations"], sc["opacities"], sc["colors"],
                     cam)
    grad = torch.zeros((P, 9), device=dev)
    for spec in SPECS:
        # bench.py's timed path: dw_render_backward_views over a batch -- here
        # the view twice, so the second launch is a chained one (row-major tile
        # order, SW-B / SW-S into the padded [P][12] buffer); profile_json.py
        # keeps each spec's second launch
        k, t = spec.split(":")
        render_backward_views([r, r], [dL, dL], wr.Policy(wr.parse_policy_kind(k), int(t)), grad)
        torch.cuda.synchronize()
    json.dump({"workload": a.workload, "views": a.views, "view": a.view, "specs": SPECS,
               "launches_per_spec": 2, "instances": r.num_rendered}, open(a.specs_out, "w"))


if __name__ == "__main__":
    main()
