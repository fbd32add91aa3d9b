"""Time render_backward (CUDA events, median of reps) for a set of policies on
one view of a BASELINE config with the library DISTWAR_LIB points at.

    DISTWAR_LIB=path/to/lib.so python tools/ab_backward.py --workload c3_1m_1080p
"""
import argparse
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="c3_1m_1080p")
    ap.add_argument("--reps", type=int, default=15)
    ap.add_argument("--policies", default="native:0,sw_b:0,sw_b:4,sw_b:8,sw_b:12,sw_b:16,sw_s:0,sw_s:16,cccl:0")
    a = ap.parse_args()
    import torch

    from paper_2401_05345_b200 import _lib
    from paper_2401_05345_b200 import warpred as wr
    from paper_2401_05345_b200.rasterizer import GaussianRasterizer
    from paper_2401_05345_b200.scene import CONFIGS, make_camera, make_dL_dpixels, make_scene

    P, W, H, hc, _ = CONFIGS[a.workload]
    dev = torch.device("cuda:0")
    sc = {k: torch.from_numpy(v).to(dev) for k, v in make_scene(P, W, H, seed=0,
                                                                   high_contention=hc).items()}
    dL = torch.from_numpy(make_dL_dpixels(W, H, seed=1)).to(dev)
    r = GaussianRasterizer()
    fwd = []
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        r.render_forward(sc["means3D"], sc["scales"], sc["rotations"], sc["opacities"],
                         sc["colors"], make_camera(W, H))
        e1.record()
        torch.cuda.synchronize()
        fwd.append(e0.elapsed_time(e1))
    grad = torch.zeros((P, 9), device=dev)
    _, pairs = r.render_backward(dL, wr.Policy(wr.PolicyKind.native, 0), grad=grad, count_pairs=True)
    out = {"lib": _lib.LIB_PATH, "workload": a.workload, "pairs": pairs,
           "instances": r.num_rendered, "forward_ms": statistics.median(fwd[1:]), "backward_ms": {}}
    flush = torch.empty(64 * 1024 * 1024, device=dev)
    for spec in a.policies.split(","):
        name, t = spec.split(":")
        pol = wr.Policy(wr.parse_policy_kind(name), int(t))
        ms = []
        for i in range(a.reps + 2):
            flush.fill_(float(i))
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            r.render_backward(dL, pol, grad=grad)
            e1.record()
            torch.cuda.synchronize()
            if i >= 2:
                ms.append(e0.elapsed_time(e1))
        out["backward_ms"][spec] = round(statistics.median(ms), 4)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
