"""Per-config measurements for every BASELINE config: forward
ms / fps, backward ms for native and tuned SW-B, contributions/s, REDs, and
the fractions of the L2-atomic (measured RED peaks) and HBM rooflines.
One view per config (C5's 64-view batch is bench.py's multi-GPU workload).

    python tools/config_table.py > gpurun_out/config_table.jsonl
"""
import ctypes as C
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch

    from paper_2401_05345_b200 import _lib
    from paper_2401_05345_b200 import warpred as wr
    from paper_2401_05345_b200.rasterizer import GaussianRasterizer, microbench_red
    from paper_2401_05345_b200.scene import CONFIGS, make_camera, make_dL_dpixels, make_scene

    dev = torch.device("cuda:0")
    hbm = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                      "MEASURED_PEAKS.json")))["hbm_gbs"] \
        if os.path.exists("MEASURED_PEAKS.json") else 6650.0
    peaks = {"same": microbench_red(1, 1 << 28), "distwar": microbench_red(3, 1 << 28)}
    flush = torch.empty(64 * 1024 * 1024, device=dev)

    def timed(fn, reps):
        ms = []
        for i in range(reps + 2):
            flush.fill_(float(i))
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            fn()
            e1.record()
            torch.cuda.synchronize()
            if i >= 2:
                ms.append(e0.elapsed_time(e1))
        return statistics.median(ms)

    for name, (P, W, H, hc, views) in CONFIGS.items():
        sc = {k: torch.from_numpy(v).to(dev) for k, v in make_scene(P, W, H, seed=0,
                                                                       high_contention=hc).items()}
        cam = make_camera(W, H)
        dL = torch.from_numpy(make_dL_dpixels(W, H, seed=1)).to(dev)
        r = GaussianRasterizer()
        args = [sc[k] for k in ("means3D", "scales", "rotations", "opacities", "colors")]
        fwd = timed(lambda: r.render_forward(*args, cam), 5)
        grad = torch.zeros((P, 9), device=dev)
        _, pairs = r.render_backward(dL, wr.Policy(wr.PolicyKind.native, 0), grad=grad,
                                     count_pairs=True)
        reps = 3 if hc else 7
        nat = timed(lambda: r.render_backward(dL, wr.Policy(wr.PolicyKind.native, 0), grad=grad),
                    reps)
        sweep = {t: timed(lambda: r.render_backward(dL, wr.Policy(wr.PolicyKind.sw_b, t),
                                                    grad=grad), reps)
                 for t in (0, 4, 8, 12, 16, 20, 24)}
        tb = min(sweep, key=lambda t: (sweep[t], t))
        r.render_backward(dL, wr.Policy(wr.PolicyKind.sw_b, tb), grad=grad, count_pairs=True)
        red = C.c_uint64()
        _lib.check(_lib.lib().dw_rasterizer_last_reds(r.handle, C.byref(red)))
        vis = int((r.buffer("radii") > 0).sum())
        alg = 4 * r.num_rendered + 44 * vis + 20 * W * H + 36 * P
        contrib = 9 * pairs
        row = {
            "config": name, "gaussians": P, "width": W, "height": H, "views_in_config": views,
            "instances": r.num_rendered, "pairs": pairs, "contributions": contrib,
            "forward_ms": fwd, "forward_fps": 1e3 / fwd,
            "native_ms": nat, "native_contrib_per_s": contrib / (nat * 1e-3),
            "native_l2_red_frac": contrib / (nat * 1e-3) / peaks["same"],
            "sw_b_threshold": tb, "sw_b_ms": sweep[tb], "sw_b_sweep_ms": sweep,
            "sw_b_contrib_per_s": contrib / (sweep[tb] * 1e-3),
            "sw_b_reds": red.value, "sw_b_l2_red_frac": red.value / (sweep[tb] * 1e-3) / peaks["distwar"],
            "sw_b_hbm_frac": alg / (sweep[tb] * 1e-3) / (hbm * 1e9),
            "speedup": nat / sweep[tb], "red_peaks_per_s": peaks,
        }
        print(json.dumps(row), flush=True)
        del r, sc, grad
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
