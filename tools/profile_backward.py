"""Minimal driver for ncu: one view of a BASELINE config, forward once, then
`--reps` uncounted render_backward launches of one policy (so `-k
regex:k_backward -s 1 -c 1` captures exactly the timed instantiation).

    ncu --set full -k regex:k_backward -s 1 -c 1 -o prof \
        python tools/profile_backward.py --policy sw_b --threshold 12
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="c3_1m_1080p")
    ap.add_argument("--policy", default="sw_b")
    ap.add_argument("--threshold", type=int, default=12)
    ap.add_argument("--reps", type=int, default=3)
    a = ap.parse_args()
    import torch

    from paper_2401_05345_b200 import warpred as wr
    from paper_2401_05345_b200.rasterizer import GaussianRasterizer
    from paper_2401_05345_b200.scene import CONFIGS, make_camera, make_dL_dpixels, make_scene

    P, W, H, hc, _ = CONFIGS[a.workload]
    dev = torch.device("cuda:0")
    sc = {k: torch.from_numpy(v).to(dev) for k, v in make_scene(P, W, H, seed=0,
                                                                   high_contention=hc).items()}
    dL = torch.from_numpy(make_dL_dpixels(W, H, seed=1)).to(dev)
    r = GaussianRasterizer()
    r.render_forward(sc["means3D"], sc["scales"], sc["rotations"], sc["opacities"], sc["colors"],
                     make_camera(W, H))
    grad = torch.zeros((P, 9), device=dev)
    pol = wr.Policy(wr.parse_policy_kind(a.policy), a.threshold)
    for _ in range(a.reps):
        r.render_backward(dL, pol, grad=grad)
    torch.cuda.synchronize()
    print("ok", r.num_rendered)


if __name__ == "__main__":
    main()
