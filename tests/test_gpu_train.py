"""GPU: the steps either side of the hot path -- preprocess
backward to 3D gradients, the fused Adam step, and a short training loop.

Bars: preprocess backward fed the oracle's own screen-space gradients matches
the oracle's float64 3D gradients to relative L2 1e-4 (pure fp32 rounding);
fed the GPU backward's gradients, relative L2 2e-3 (the backward's own
tolerance, tests/test_gpu_raster.py); Adam matches the float64 reference to
1e-5 relative; and 30 steps of render -> DISTWAR backward -> preprocess
backward -> Adam reduce an L2 image loss.
"""
import ctypes as C

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _ocam(cam):
    from oracle.bindings import Camera as OCam

    oc = OCam()
    cc = cam.to_c()
    C.memmove(C.byref(oc), C.byref(cc), C.sizeof(oc))
    return oc


@pytest.mark.parametrize("yaw", [0.0, 9.0])
def test_preprocess_backward_matches_oracle(cuda, orc, yaw):
    import torch

    from oracle.bindings import gs_train_grads
    from paper_2401_05345_b200 import warpred as wr
    from paper_2401_05345_b200.rasterizer import GaussianRasterizer
    from paper_2401_05345_b200.scene import make_camera, make_dL_dpixels, make_scene

    P, W, H = 20_000, 320, 240
    sc = make_scene(P, W, H, seed=12)
    cam = make_camera(W, H, yaw_deg=yaw)
    dL = make_dL_dpixels(W, H, seed=13)
    g2_ref, g3_ref = gs_train_grads(orc, sc, _ocam(cam), dL)
    t = {k: torch.from_numpy(v).to(cuda) for k, v in sc.items()}
    r = GaussianRasterizer()
    r.render_forward(t["means3D"], t["scales"], t["rotations"], t["opacities"], t["colors"], cam)
    # (1) the kernel alone: oracle's grad2d in
    g3 = r.preprocess_backward(t["means3D"], t["scales"], t["rotations"],
                               torch.from_numpy(g2_ref.astype(np.float32)).to(cuda))
    got = g3.cpu().numpy().astype(np.float64)
    rel = np.linalg.norm(got - g3_ref) / np.linalg.norm(g3_ref)
    assert rel < 1e-4, rel
    for sl in (slice(0, 3), slice(3, 6), slice(6, 10), slice(10, 11), slice(11, 14)):
        part = np.linalg.norm(got[:, sl] - g3_ref[:, sl]) / max(np.linalg.norm(g3_ref[:, sl]), 1e-30)
        assert part < 1e-3, (sl, part)
    # (2) the whole GPU chain; accumulation across two calls doubles it
    g2 = r.render_backward(torch.from_numpy(dL).to(cuda), wr.Policy(wr.PolicyKind.sw_b, 8))
    g3b = r.preprocess_backward(t["means3D"], t["scales"], t["rotations"], g2)
    r.preprocess_backward(t["means3D"], t["scales"], t["rotations"], g2, grad3d=g3b)
    got = g3b.cpu().numpy().astype(np.float64) / 2
    rel = np.linalg.norm(got - g3_ref) / np.linalg.norm(g3_ref)
    assert rel < 2e-3, rel


def test_adam_matches_reference(cuda, orc):
    import torch

    from oracle.bindings import gs_adam
    from paper_2401_05345_b200.rasterizer import Adam
    from paper_2401_05345_b200.scene import make_scene

    sc = make_scene(1000, 64, 64, seed=2)
    t = {k: torch.from_numpy(v.copy()).to(cuda) for k, v in sc.items()}
    lr = (1e-3, 2e-3, 3e-3, 4e-3, 5e-3)
    opt = Adam(t, lr=lr, eps=1e-8)
    flat = np.concatenate([sc["means3D"], sc["scales"], sc["rotations"], sc["opacities"][:, None],
                           sc["colors"]], axis=1).astype(np.float64)
    m, v = np.zeros_like(flat), np.zeros_like(flat)
    rng = np.random.default_rng(3)
    lrs = np.repeat(np.array(lr), [3, 3, 4, 1, 3])[None, :]
    for step in range(1, 4):
        g = rng.normal(size=flat.shape)
        opt.step(torch.from_numpy(g.astype(np.float32)).to(cuda))
        for col in range(14):  # per-group lr: run the reference column-wise
            p, gg = flat[:, col].copy(), g[:, col].copy()
            mm, vv = m[:, col].copy(), v[:, col].copy()
            gs_adam(orc, p, gg, mm, vv, float(lrs[0, col]), 0.9, 0.999, 1e-8, step)
            flat[:, col], m[:, col], v[:, col] = p, mm, vv
    got = np.concatenate([t["means3D"].cpu().numpy(), t["scales"].cpu().numpy(),
                          t["rotations"].cpu().numpy(), t["opacities"].cpu().numpy()[:, None],
                          t["colors"].cpu().numpy()], axis=1)
    np.testing.assert_allclose(got, flat, rtol=1e-5, atol=1e-6)


def test_backward_step_is_cuda_graph_capturable(cuda):
    """The per-step hot path -- zero grad, DISTWAR backward over several
    resident views, preprocess backward, Adam -- launches without host syncs or
    allocations, so it captures into one CUDA graph and replays to the same
    result as eager execution."""
    import torch

    from paper_2401_05345_b200 import warpred as wr
    from paper_2401_05345_b200.rasterizer import Adam, GaussianRasterizer
    from paper_2401_05345_b200.scene import make_dL_dpixels, make_scene, orbit_cameras

    P, W, H, V = 20_000, 256, 192, 3
    base = make_scene(P, W, H, seed=21)
    cams = orbit_cameras(W, H, V)
    dLs = [torch.from_numpy(make_dL_dpixels(W, H, seed=30 + k)).to(cuda) for k in range(V)]

    def setup():
        s = {k: torch.from_numpy(v.copy()).to(cuda) for k, v in base.items()}
        rs = [GaussianRasterizer() for _ in range(V)]
        for r, c in zip(rs, cams):
            r.render_forward(s["means3D"], s["scales"], s["rotations"], s["opacities"],
                             s["colors"], c)
        return s, rs, Adam(s)

    pol = wr.Policy(wr.PolicyKind.sw_b, 8)

    def step(s, rs, opt, g2, g3):
        g3.zero_()
        for r, dL in zip(rs, dLs):
            g2.zero_()
            r.render_backward(dL, pol, grad=g2)
            r.preprocess_backward(s["means3D"], s["scales"], s["rotations"], g2, grad3d=g3)
        opt.step(g3)

    s_e, rs_e, opt_e = setup()
    g2e = torch.zeros((P, 9), device=cuda)
    g3e = torch.zeros((P, 14), device=cuda)
    step(s_e, rs_e, opt_e, g2e, g3e)
    torch.cuda.synchronize()

    s_g, rs_g, opt_g = setup()
    g2g = torch.zeros((P, 9), device=cuda)
    g3g = torch.zeros((P, 14), device=cuda)
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    graph = torch.cuda.CUDAGraph()
    opt_g.t = 0  # Adam's step counter is a host argument: captured as 1
    with torch.cuda.stream(side):
        with torch.cuda.graph(graph, stream=side):
            step(s_g, rs_g, opt_g, g2g, g3g)
    torch.cuda.synchronize()
    # capture did not execute; replay once == one eager step
    for k in ("means3D", "scales", "rotations", "opacities", "colors"):
        assert torch.equal(s_g[k], torch.from_numpy(base[k]).to(cuda))
    graph.replay()
    torch.cuda.synchronize()
    rel = (g3g - g3e).norm() / g3e.norm()
    assert rel < 1e-4, float(rel)
    # Adam's first step is lr * sign(g): atomic-order noise can flip the sign
    # of a near-zero gradient element, so bound the fraction that differ
    for k in ("means3D", "colors"):
        off = ~torch.isclose(s_g[k], s_e[k], rtol=1e-5, atol=1e-6)
        assert off.float().mean() < 1e-3, (k, float(off.float().mean()))


def test_training_loop_reduces_loss(cuda):
    import torch

    from paper_2401_05345_b200 import warpred as wr
    from paper_2401_05345_b200.rasterizer import Adam, GaussianRasterizer
    from paper_2401_05345_b200.scene import make_camera, make_scene

    P, W, H = 3000, 128, 96
    cam = make_camera(W, H)
    target_scene = {k: torch.from_numpy(v).to(cuda) for k, v in make_scene(P, W, H, seed=5).items()}
    r = GaussianRasterizer()
    target, _, _ = r.render_forward(*[target_scene[k] for k in ("means3D", "scales", "rotations",
                                                               "opacities", "colors")], cam)
    target = target.clone()
    init = make_scene(P, W, H, seed=5)
    rng = np.random.default_rng(6)
    init["colors"] = np.clip(init["colors"] + rng.normal(0, 0.2, init["colors"].shape), 0, 1
                             ).astype(np.float32)
    init["means3D"] = (init["means3D"] * (1 + rng.normal(0, 0.01, init["means3D"].shape))
                       ).astype(np.float32)
    s = {k: torch.from_numpy(v).to(cuda) for k, v in init.items()}
    opt = Adam(s, lr=(1e-3, 1e-4, 1e-3, 1e-3, 1e-2), eps=1e-15)
    losses = []
    for _ in range(30):
        img, _, _ = r.render_forward(s["means3D"], s["scales"], s["rotations"], s["opacities"],
                                     s["colors"], cam)
        diff = img - target
        losses.append(float((diff * diff).mean()))
        g2 = r.render_backward((2.0 / diff.numel()) * diff, wr.Policy(wr.PolicyKind.sw_b, 8))
        g3 = r.preprocess_backward(s["means3D"], s["scales"], s["rotations"], g2)
        opt.step(g3)
    assert losses[-1] < 0.5 * losses[0], losses


def _scene_t(cuda, sc):
    import torch

    return {k: torch.from_numpy(v.copy()).to(cuda) for k, v in sc.items()}


_KEYS = ("means3D", "scales", "rotations", "opacities", "colors")


@pytest.mark.parametrize("binning", ["scatter", "depth-first", "dense", "block"])
@pytest.mark.parametrize("yaw", [0.0, 23.0])
def test_forward_async_matches_sync(cuda, yaw, binning, monkeypatch):
    """The no-host-sync forward (device-side instance count over a reserved
    capacity) bins and blends exactly like the synchronising forward -- with
    either list construction, including the over-capacity frame."""
    import torch

    from parity import set_binning

    set_binning(monkeypatch, binning)

    from paper_2401_05345_b200.rasterizer import GaussianRasterizer
    from paper_2401_05345_b200.scene import make_camera, make_scene

    P, W, H = 30_000, 320, 240
    s = _scene_t(cuda, make_scene(P, W, H, seed=41))
    cam = make_camera(W, H, yaw_deg=yaw)
    a = GaussianRasterizer()
    img_a, rad_a, nr = a.render_forward(*[s[k] for k in _KEYS], cam)
    img_a, rad_a = img_a.clone(), rad_a.clone()
    b = GaussianRasterizer()
    b.reserve(P, W, H, 2 * nr + 1000)
    img_b = torch.full((3, H, W), float("nan"), device=cuda)
    rad_b = torch.full((P,), -7, dtype=torch.int32, device=cuda)
    b.render_forward_async(*[s[k] for k in _KEYS], cam, img_b, rad_b)
    assert b.instances() == (nr, False)
    assert torch.equal(img_a, img_b)
    assert torch.equal(rad_a, rad_b)
    for name in ("ranges", "values", "n_contrib", "final_T"):
        assert np.array_equal(a.buffer(name), b.buffer(name)), name
    # over capacity: nothing binned, the frame is the background, flag raised
    c = GaussianRasterizer()
    c.reserve(P, W, H, nr // 2)
    img_c = torch.empty((3, H, W), device=cuda)
    rad_c = torch.empty((P,), dtype=torch.int32, device=cuda)
    c.render_forward_async(*[s[k] for k in _KEYS], cam, img_c, rad_c)
    n_c, ovf = c.instances()
    assert ovf and n_c == 0
    bg = torch.tensor(cam.bg, device=cuda).view(3, 1, 1).expand(3, H, W)
    assert torch.equal(img_c, bg.contiguous())
    # and the next in-capacity forward clears the flag
    c.reserve(P, W, H, nr)
    c.render_forward_async(*[s[k] for k in _KEYS], cam, img_c, rad_c)
    assert c.instances() == (nr, False)
    assert torch.equal(img_c, img_a)


def test_forward_async_requires_reserve(cuda):
    import torch

    from paper_2401_05345_b200._lib import InvalidArgument
    from paper_2401_05345_b200.rasterizer import GaussianRasterizer
    from paper_2401_05345_b200.scene import make_camera, make_scene

    s = _scene_t(cuda, make_scene(100, 64, 64, seed=1))
    r = GaussianRasterizer()
    with pytest.raises(InvalidArgument):
        r.render_forward_async(*[s[k] for k in _KEYS], make_camera(64, 64),
                               torch.empty((3, 64, 64), device=cuda),
                               torch.empty((100,), dtype=torch.int32, device=cuda))
    with pytest.raises(InvalidArgument):
        r.reserve(-1, 64, 64, 10)


def test_whole_training_step_is_cuda_graph_capturable(cuda):
    """forward (no host sync) -> L2 image loss -> DISTWAR backward ->
    preprocess backward -> Adam: one CUDA graph per training step. One replay
    matches one eager step; repeated replays train the scene."""
    import torch

    from paper_2401_05345_b200 import warpred as wr
    from paper_2401_05345_b200.rasterizer import Adam, GaussianRasterizer
    from paper_2401_05345_b200.scene import make_camera, make_scene

    P, W, H = 6000, 192, 128
    cam = make_camera(W, H)
    tgt = _scene_t(cuda, make_scene(P, W, H, seed=51))
    r0 = GaussianRasterizer()
    target, _, nr = r0.render_forward(*[tgt[k] for k in _KEYS], cam)
    target = target.clone()
    init = make_scene(P, W, H, seed=51)
    rng = np.random.default_rng(52)
    init["colors"] = np.clip(init["colors"] + rng.normal(0, 0.2, init["colors"].shape), 0, 1
                             ).astype(np.float32)
    pol = wr.Policy(wr.PolicyKind.sw_b, 8)
    lr = (1e-4, 1e-4, 1e-3, 1e-3, 1e-2)

    def setup():
        s = _scene_t(cuda, init)
        r = GaussianRasterizer()
        r.reserve(P, W, H, 4 * nr)
        bufs = dict(img=torch.empty((3, H, W), device=cuda),
                    radii=torch.empty((P,), dtype=torch.int32, device=cuda),
                    g2=torch.zeros((P, 9), device=cuda), g3=torch.zeros((P, 14), device=cuda),
                    loss=torch.zeros((), device=cuda))
        return s, r, Adam(s, lr=lr, eps=1e-15), bufs

    def step(s, r, opt, b):
        r.render_forward_async(*[s[k] for k in _KEYS], cam, b["img"], b["radii"])
        diff = b["img"] - target
        b["loss"].copy_((diff * diff).mean())
        b["g2"].zero_()
        r.render_backward((2.0 / diff.numel()) * diff, pol, grad=b["g2"])
        b["g3"].zero_()
        r.preprocess_backward(s["means3D"], s["scales"], s["rotations"], b["g2"], grad3d=b["g3"])
        opt.step(b["g3"])

    s_e, r_e, opt_e, b_e = setup()
    step(s_e, r_e, opt_e, b_e)
    torch.cuda.synchronize()

    s_g, r_g, opt_g, b_g = setup()
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    graph = torch.cuda.CUDAGraph()
    opt_g.t = 0
    with torch.cuda.stream(side):
        with torch.cuda.graph(graph, stream=side):
            step(s_g, r_g, opt_g, b_g)
    torch.cuda.synchronize()
    assert torch.equal(s_g["colors"], torch.from_numpy(init["colors"]).to(cuda))
    graph.replay()
    torch.cuda.synchronize()
    assert torch.equal(b_g["img"], b_e["img"])
    assert float(b_g["loss"]) == float(b_e["loss"])
    rel = (b_g["g3"] - b_e["g3"]).norm() / b_e["g3"].norm()
    assert rel < 1e-4, float(rel)
    losses = [float(b_g["loss"])]
    for _ in range(40):
        graph.replay()
        torch.cuda.synchronize()
        losses.append(float(b_g["loss"]))
        assert r_g.instances()[1] is False
    assert losses[-1] < 0.6 * losses[0], losses


def test_view_parallel_train_step_matches_oracle(cuda, orc):
    """dist.view_parallel_train_step with the GPU pieces (render forward, DISTWAR
    backward, per-view preprocess backward into one [P, 14] buffer, fused Adam)
    sums the views' 3D gradients as the CPU oracle does, and the update moves
    the replica by the Adam step of that sum (one process: the all-reduce is a
    no-op here; tests/test_dist_gloo.py runs the two-rank step)."""
    import torch

    from oracle.bindings import gs_train_grads
    from paper_2401_05345_b200 import warpred as wr
    from paper_2401_05345_b200.dist import view_parallel_train_step
    from paper_2401_05345_b200.rasterizer import Adam, GaussianRasterizer
    from paper_2401_05345_b200.scene import make_dL_dpixels, make_scene, orbit_cameras

    P, W, H, V = 20_000, 320, 240, 3
    sc = make_scene(P, W, H, seed=21)
    cams = orbit_cameras(W, H, V)
    dLs = {id(c): make_dL_dpixels(W, H, seed=30 + k) for k, c in enumerate(cams)}
    want = sum(gs_train_grads(orc, sc, _ocam(c), dLs[id(c)])[1] for c in cams)
    t = {k: torch.from_numpy(v.copy()).to(cuda) for k, v in sc.items()}
    before = {k: v.clone() for k, v in t.items()}
    r = GaussianRasterizer()
    grad2d = torch.zeros((P, 9), device=cuda)

    def grads_view(cam, grad3d):
        r.render_forward(t["means3D"], t["scales"], t["rotations"], t["opacities"], t["colors"],
                         cam)
        grad2d.zero_()
        r.render_backward(torch.from_numpy(dLs[id(cam)]).to(cuda),
                          wr.Policy(wr.PolicyKind.sw_b, 16), grad=grad2d)
        r.preprocess_backward(t["means3D"], t["scales"], t["rotations"], grad2d, grad3d=grad3d)

    opt = Adam(t)
    grad3d = torch.zeros((P, 14), device=cuda)
    view_parallel_train_step(grads_view, cams, grad3d, opt.step)
    torch.cuda.synchronize()
    got = grad3d.cpu().numpy().astype(np.float64)
    assert np.linalg.norm(got - want) / np.linalg.norm(want) < 2e-3
    # the first Adam step moves every parameter with a nonzero gradient by ~lr
    moved = (t["means3D"] - before["means3D"]).abs().cpu().numpy()
    nz = np.abs(got[:, 0:3]) > 1e-6
    assert np.all(moved[nz] > 0)
