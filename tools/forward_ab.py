"""Forward A/B across list constructions: median event-timed forward of one
view and its per-stage breakdown, per binning mode.

    python tools/forward_ab.py --workload c3_1m_1080p --modes scatter depth-first
"""
import argparse
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))

ENV = {"scatter": {"DW_SCATTER": "1", "DW_DENSE_BINNING": "0", "DW_TILE_FIRST": "0"},
       "depth-first": {"DW_SCATTER": "0", "DW_DENSE_BINNING": "0", "DW_TILE_FIRST": "0",
                       "DW_BLOCK_BINNING": "0"},
       "block": {"DW_SCATTER": "0", "DW_DENSE_BINNING": "0", "DW_TILE_FIRST": "0",
                 "DW_BLOCK_BINNING": "1"},
       "tile-first": {"DW_SCATTER": "0", "DW_DENSE_BINNING": "0", "DW_TILE_FIRST": "1"},
       "dense": {"DW_DENSE_BINNING": "1"}, "auto": {}}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="c3_1m_1080p")
    ap.add_argument("--views", type=int, default=1)
    ap.add_argument("--view", type=int, default=0)
    ap.add_argument("--modes", nargs="+", default=["scatter", "depth-first"])
    ap.add_argument("--reps", type=int, default=10)
    a = ap.parse_args()
    import torch

    from paper_2401_05345_b200.rasterizer import GaussianRasterizer
    from paper_2401_05345_b200.scene import CONFIGS, make_camera, make_scene, orbit_cameras

    P, W, H, hc, _ = CONFIGS[a.workload]
    dev = torch.device("cuda:0")
    t = {k: torch.from_numpy(v).to(dev)
         for k, v in make_scene(P, W, H, seed=0, high_contention=hc).items()}
    cam = orbit_cameras(W, H, a.views)[a.view] if a.views > 1 else make_camera(W, H)
    args = [t[k] for k in ("means3D", "scales", "rotations", "opacities", "colors")]
    out = {"workload": a.workload, "view": f"{a.view}/{a.views}"}
    for mode in a.modes:
        for k in ("DW_SCATTER", "DW_DENSE_BINNING", "DW_TILE_FIRST", "DW_BLOCK_BINNING"):
            os.environ.pop(k, None)
        os.environ.update(ENV[mode])
        r = GaussianRasterizer()
        ms = []
        for i in range(a.reps + 2):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            r.render_forward(*args, cam)
            e1.record()
            torch.cuda.synchronize()
            if i >= 2:
                ms.append(e0.elapsed_time(e1))
        r.stage_timing(True)
        r.render_forward(*args, cam)
        st = r.stage_ms()
        r.render_forward(*args, cam)
        st2 = r.stage_ms()
        out[mode] = {"forward_ms": statistics.median(ms), "min_ms": min(ms),
                     "stages": {k: min(st[k], st2[k]) for k in st}, "instances": r.num_rendered}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
