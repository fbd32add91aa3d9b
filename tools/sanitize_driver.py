"""Exercise every libdistwar kernel once on small inputs, for
compute-sanitizer (memcheck / racecheck / synccheck / initcheck):

    compute-sanitizer --tool racecheck python tools/sanitize_driver.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch

    from paper_2401_05345_b200 import warpred as wr
    from paper_2401_05345_b200.rasterizer import (Adam, GaussianRasterizer, render_backward_views,
                                                  render_views_host)
    from paper_2401_05345_b200.scene import make_camera, make_dL_dpixels, make_scene, orbit_cameras

    dev = torch.device("cuda:0")
    # trace-driven kernels: every compiled N and policy, counted and not
    for n in (1, 2, 3, 4, 5, 9, 17):
        tr = wr.generate(wr.SceneSpec(num_primitives=300, params_per_primitive=n, image_width=64,
                                      image_height=32, locality=0.7, activity_prob=0.6, seed=n))
        d = wr.DeviceTrace(tr)
        for kind, t in ((0, 0), (1, 8), (2, 8), (3, 0)):
            wr.gpu_run(d, wr.Policy(wr.PolicyKind(kind), t))
    # rasterizer: odd image size, all policies, tap, preprocess backward, Adam
    P, W, H = 4000, 77, 53
    sc = {k: torch.from_numpy(v).to(dev) for k, v in make_scene(P, W, H, seed=2).items()}
    cam = make_camera(W, H)
    dL = torch.from_numpy(make_dL_dpixels(W, H)).to(dev)
    r = GaussianRasterizer()
    r.render_forward(sc["means3D"], sc["scales"], sc["rotations"], sc["opacities"], sc["colors"], cam)
    for kind, t in ((0, 0), (1, 8), (2, 8), (3, 0)):
        r.render_backward(dL, wr.Policy(wr.PolicyKind(kind), t))
        r.render_backward(dL, wr.Policy(wr.PolicyKind(kind), t), count_pairs=True)
    g2, tr, _ = r.render_backward_tap(dL, threshold=4)
    g3 = r.preprocess_backward(sc["means3D"], sc["scales"], sc["rotations"], g2)
    Adam(sc).step(g3)
    r.buffer("keys")
    # a large-list scene (wide rects -> warp-cooperative duplication, 4096-tiles sort)
    big = {k: torch.from_numpy(v).to(dev) for k, v in
           make_scene(3000, 640, 480, seed=3, high_contention=True).items()}
    cam2 = make_camera(640, 480)
    r.render_forward(big["means3D"], big["scales"], big["rotations"], big["opacities"],
                     big["colors"], cam2)
    r.render_backward(torch.from_numpy(make_dL_dpixels(640, 480)).to(dev),
                      wr.Policy(wr.PolicyKind.sw_b, 8))
    # every list construction on a scene whose block lists take several
    # staging rounds (block binning), plus a no-sync forward over its reserve
    mid = {k: torch.from_numpy(v).to(dev) for k, v in make_scene(60000, 640, 480, seed=4).items()}
    cam3 = make_camera(640, 480)
    margs = [mid[k] for k in ("means3D", "scales", "rotations", "opacities", "colors")]
    dL3 = torch.from_numpy(make_dL_dpixels(640, 480)).to(dev)
    modes = {"block": {"DW_BLOCK_BINNING": "1"}, "depth-first": {"DW_BLOCK_BINNING": "0"},
             "tile-first": {"DW_TILE_FIRST": "1"}, "scatter": {"DW_SCATTER": "1"},
             "dense": {"DW_DENSE_BINNING": "1"}}
    for mode, env in modes.items():
        for k in ("DW_BLOCK_BINNING", "DW_TILE_FIRST", "DW_SCATTER", "DW_DENSE_BINNING"):
            os.environ.pop(k, None)
        os.environ.update(env)
        rm = GaussianRasterizer()
        rm.render_forward(*margs, cam3)
        rm.render_backward(dL3, wr.Policy(wr.PolicyKind.sw_b, 16))
        rm.buffer("keys")
        n = rm.num_rendered
        ra = GaussianRasterizer()  # buffers only grow: a fresh one for the small reserve
        ra.reserve(60000, 640, 480, n // 2)  # too small: the async forward must overflow cleanly
        img3 = torch.empty((3, 480, 640), device=dev)
        rad3 = torch.empty(60000, dtype=torch.int32, device=dev)
        ra.render_forward_async(*margs, cam3, img3, rad3)
        assert ra.instances()[1], mode
        ra.reserve(60000, 640, 480, n + 4096)
        ra.render_forward_async(*margs, cam3, img3, rad3)
        assert not ra.instances()[1], mode
        ra.render_backward(dL3, wr.Policy(wr.PolicyKind.sw_b, 16))
    for k in ("DW_BLOCK_BINNING", "DW_TILE_FIRST", "DW_SCATTER", "DW_DENSE_BINNING"):
        os.environ.pop(k, None)
    # batched host path
    cams = orbit_cameras(W, H, 3)
    pin = {k: v.cpu().pin_memory() for k, v in sc.items()}
    dLh = torch.stack([dL.cpu()] * 3).pin_memory()
    img = torch.empty((3, 3, H, W)).pin_memory()
    grad = torch.empty((P, 9)).pin_memory()
    render_views_host(r, [pin[k].data_ptr() for k in ("means3D", "scales", "rotations",
                                                      "opacities", "colors")],
                      P, cams, dLh.data_ptr(), wr.Policy(wr.PolicyKind.sw_b, 8), img.data_ptr(),
                      grad.data_ptr())
    # the same with stacked frames and more views (waves, no-sync pool states)
    os.environ["DW_VIEWS_STACK"] = "3"
    cams7 = orbit_cameras(W, H, 7)
    dLh7 = torch.stack([dL.cpu()] * 7).pin_memory()
    img7 = torch.empty((7, 3, H, W)).pin_memory()
    render_views_host(r, [pin[k].data_ptr() for k in ("means3D", "scales", "rotations",
                                                      "opacities", "colors")],
                      P, cams7, dLh7.data_ptr(), wr.Policy(wr.PolicyKind.sw_b, 8), img7.data_ptr(),
                      grad.data_ptr())
    os.environ.pop("DW_VIEWS_STACK")
    # stacked forward + its backward; a batch chain (padded rows + fold), chained calls
    rs3 = GaussianRasterizer()
    args = [sc[k] for k in ("means3D", "scales", "rotations", "opacities", "colors")]
    rs3.render_forward_views(*args, orbit_cameras(W, H, 3))
    rs3.render_backward(torch.stack([dL] * 3), wr.Policy(wr.PolicyKind.sw_b, 8))
    views = []
    for c in orbit_cameras(W, H, 3):
        rv = GaussianRasterizer()
        rv.render_forward(*args, c)
        views.append(rv)
    g = torch.zeros((P, 9), device=dev)
    render_backward_views(views, [dL] * 3, wr.Policy(wr.PolicyKind.sw_b, 8), g)
    render_backward_views(views, [dL] * 3, wr.Policy(wr.PolicyKind.native, 0), g)
    for k, rv in enumerate(views):
        rv.render_backward(dL, wr.Policy(wr.PolicyKind.sw_b, 8), grad=g, chained=k > 0)
    torch.cuda.synchronize()
    print("sanitize driver OK")


if __name__ == "__main__":
    main()
