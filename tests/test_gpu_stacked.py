"""Batched views: stacked frames (dw_render_forward_views: several views of
one scene share every launch of the forward and one backward launch), chained
backwards (dw_render_backward_chained) and the batched host path built on
them.
The bar is the single-view path itself: per-tile lists, images, final_T and
n_contrib bit for bit (view v's ids offset by v*P in the frame), gradients
equal to the per-view sum up to fp32 reassociation of the RED order -- and
through tests/test_gpu_raster.py's views-host tests (the default host path:
waves of forwards, chained backwards) the oracle's per-view bounds.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

SCENE_KEYS = ("means3D", "scales", "rotations", "opacities", "colors")


def _scene(cuda, P, W, H, seed, **kw):
    import torch

    from paper_2401_05345_b200.scene import make_scene

    return {k: torch.from_numpy(v).to(cuda) for k, v in make_scene(P, W, H, seed=seed, **kw).items()}


def _grad_close(got, want):
    # two orders of fp32 RED accumulation of the same addends
    err = np.linalg.norm(got - want) / max(np.linalg.norm(want), 1e-30)
    assert err < 1e-5, err


@pytest.mark.parametrize("nv", [2, 3])
def test_stacked_forward_equals_single_views(cuda, nv):
    import torch

    from paper_2401_05345_b200 import warpred as wr
    from paper_2401_05345_b200.rasterizer import GaussianRasterizer, max_stacked_views
    from paper_2401_05345_b200.scene import make_dL_dpixels, orbit_cameras

    P, W, H = 20000, 256, 200  # 13 tile rows per view: the last row is partial
    assert max_stacked_views(W, H) >= nv
    sc = _scene(cuda, P, W, H, seed=71)
    args = [sc[k] for k in SCENE_KEYS]
    cams = orbit_cameras(W, H, 5)[1:1 + nv]
    dL = torch.from_numpy(np.stack([make_dL_dpixels(W, H, seed=80 + v) for v in range(nv)])).to(cuda)
    pol = wr.Policy(wr.PolicyKind.sw_b, 12)
    singles, want = [], torch.zeros((P, 9), dtype=torch.float32, device=cuda)
    for v, cam in enumerate(cams):
        r = GaussianRasterizer()
        img, _, nr = r.render_forward(*args, cam)
        r.render_backward(dL[v], pol, grad=want)
        singles.append(dict(img=img.cpu().numpy(), nr=nr, ranges=r.buffer("ranges"),
                            values=r.buffer("values"), T=r.buffer("final_T"),
                            nc=r.buffer("n_contrib")))
    rs = GaussianRasterizer()
    imgs, nr = rs.render_forward_views(*args, cams)
    assert nr == sum(s["nr"] for s in singles)
    ranges, values = rs.buffer("ranges"), rs.buffer("values")
    T, nc = rs.buffer("final_T"), rs.buffer("n_contrib")
    ntv = singles[0]["ranges"].shape[0]
    assert ranges.shape[0] == nv * ntv
    for v, s in enumerate(singles):
        assert np.array_equal(imgs[v].cpu().numpy(), s["img"])
        assert np.array_equal(T[v * H * W:(v + 1) * H * W], s["T"])
        assert np.array_equal(nc[v * H * W:(v + 1) * H * W], s["nc"])
        rv = ranges[v * ntv:(v + 1) * ntv]
        assert np.array_equal(rv[:, 1] - rv[:, 0], s["ranges"][:, 1] - s["ranges"][:, 0])
        lists = np.concatenate([values[a:b] for a, b in rv])
        assert np.array_equal(lists, s["values"] + v * P)
    grad = torch.zeros((P, 9), dtype=torch.float32, device=cuda)
    rs.render_backward(dL, pol, grad=grad)
    _grad_close(grad.cpu().numpy().astype(np.float64), want.cpu().numpy().astype(np.float64))
    # every policy reads the frame the same way (native: the one-pixel kernel)
    for kind, t in ((wr.PolicyKind.native, 0), (wr.PolicyKind.sw_s, 20), (wr.PolicyKind.cccl, 0)):
        g = torch.zeros((P, 9), dtype=torch.float32, device=cuda)
        rs.render_backward(dL, wr.Policy(kind, t), grad=g)
        _grad_close(g.cpu().numpy().astype(np.float64), want.cpu().numpy().astype(np.float64))


def test_stacked_forward_rejects_bad_stacks(cuda):
    from paper_2401_05345_b200 import _lib
    from paper_2401_05345_b200.rasterizer import GaussianRasterizer, max_stacked_views
    from paper_2401_05345_b200.scene import make_camera

    assert max_stacked_views(1920, 1080) == 3  # 68 tile rows per view, <= 255 in a frame
    assert max_stacked_views(1920, 4320) == 1  # 270 rows: block binning's packing does not fit
    P, W, H = 1000, 64, 64
    sc = _scene(cuda, P, W, H, seed=3)
    args = [sc[k] for k in SCENE_KEYS]
    r = GaussianRasterizer()
    with pytest.raises(_lib.InvalidArgument):
        r.render_forward_views(*args, [make_camera(W, H)] * 4)  # more than 3 views
    with pytest.raises(_lib.InvalidArgument):
        r.render_forward_views(*args, [make_camera(W, H), make_camera(W, H + 16)])
    with pytest.raises(_lib.InvalidArgument):
        r.render_forward_views(*args, [make_camera(W, H), make_camera(W, H, bg=(0, 0, 0))])


def _views_host(monkeypatch, stack, sc_np, cams, dL, wave=None, fstreams=None):
    import torch

    from paper_2401_05345_b200 import warpred as wr
    from paper_2401_05345_b200.rasterizer import GaussianRasterizer, render_views_host

    monkeypatch.setenv("DW_VIEWS_STACK", str(stack))
    for name, val in (("DW_VIEWS_WAVE", wave), ("DW_VIEWS_FSTREAMS", fstreams)):
        if val is None:
            monkeypatch.delenv(name, raising=False)
        else:
            monkeypatch.setenv(name, str(val))
    P = sc_np["means3D"].shape[0]
    V, _, H, W = dL.shape
    pin = {k: torch.from_numpy(v).pin_memory() for k, v in sc_np.items()}
    dL_h = torch.from_numpy(dL).pin_memory()
    img = torch.empty((V, 3, H, W), dtype=torch.float32).pin_memory()
    grad = torch.empty((P, 9), dtype=torch.float32).pin_memory()
    r = GaussianRasterizer()
    ptrs = [pin[k].data_ptr() for k in SCENE_KEYS]
    out = []
    for _ in range(2):  # the second call reuses the states (stacked reserves)
        render_views_host(r, ptrs, P, cams, dL_h.data_ptr(), wr.Policy(wr.PolicyKind.sw_b, 12),
                          img.data_ptr(), grad.data_ptr())
        out.append((img.numpy().copy(), grad.numpy().astype(np.float64)))
    return out


@pytest.mark.parametrize("scene", ["plain", "contention"])
def test_views_host_stack_sizes_agree(cuda, monkeypatch, scene):
    """7 views (frames of 2 or 3 views and a partial last frame; no-sync
    reserves from stacked first frames) == one view per frame: images bit for
    bit, gradients up to the RED order. The contention scene's single views
    take dense binning, so a stacked first frame restarts the batch with one
    view per frame."""
    from paper_2401_05345_b200.scene import make_dL_dpixels, make_scene, orbit_cameras

    hc = scene == "contention"
    P, W, H, V = (3000 if hc else 8000), 192, 144, 7
    sc = make_scene(P, W, H, seed=91, high_contention=hc)
    cams = orbit_cameras(W, H, V)
    dL = np.stack([make_dL_dpixels(W, H, seed=100 + k) for k in range(V)]).astype(np.float32)
    ref = _views_host(monkeypatch, 1, sc, cams, dL)
    for stack in (2, 3):
        got = _views_host(monkeypatch, stack, sc, cams, dL)
        for (gi, gg), (ri, rg) in zip(got, ref):
            assert np.array_equal(gi, ri)
            _grad_close(gg, rg)


def test_views_host_stacked_overflow_redo(cuda, monkeypatch):
    """Frames of two views: frame 0 (two zoomed-out views, few instances)
    sizes the no-sync reserves of the pool states; frame 1 (normal views)
    outgrows its reserve, raises the sticky flag and the batch is redone with
    host-read counts -- the result equals one view per frame."""
    from paper_2401_05345_b200.scene import make_camera, make_dL_dpixels, make_scene

    P, W, H = 4000, 160, 128
    sc = make_scene(P, W, H, seed=33)
    cams = [make_camera(W, H, fov_x_deg=150.0)] * 2 + [make_camera(W, H, yaw_deg=d)
                                                       for d in (0.0, 2.0, 4.0, 6.0, 8.0)]
    V = len(cams)
    dL = np.stack([make_dL_dpixels(W, H, seed=60 + k) for k in range(V)]).astype(np.float32)
    ref = _views_host(monkeypatch, 1, sc, cams, dL)
    got = _views_host(monkeypatch, 2, sc, cams, dL)
    for (gi, gg), (ri, rg) in zip(got, ref):
        assert np.array_equal(gi, ri)
        _grad_close(gg, rg)


def test_chained_backwards_equal_plain(cuda):
    """A chain of independent views' backwards (the first plain, the rest
    dw_render_backward_chained -- no wait for the previous grid) adds the same
    gradients as plain launches; a chained call right after its own forward
    (tile order not yet computed) falls back to a plain launch."""
    import torch

    from paper_2401_05345_b200 import warpred as wr
    from paper_2401_05345_b200.rasterizer import GaussianRasterizer
    from paper_2401_05345_b200.scene import make_dL_dpixels, orbit_cameras

    P, W, H = 30000, 320, 240
    sc = _scene(cuda, P, W, H, seed=12)
    args = [sc[k] for k in SCENE_KEYS]
    cams = orbit_cameras(W, H, 4)
    dLs = [torch.from_numpy(make_dL_dpixels(W, H, seed=20 + k)).to(cuda) for k in range(4)]
    pol = wr.Policy(wr.PolicyKind.sw_b, 14)
    rs = []
    for c in cams:
        r = GaussianRasterizer()
        r.render_forward(*args, c)
        rs.append(r)
    # first backward of each state right after its forward, chained: the tile
    # order is computed first and the launch waits for it
    g0 = torch.zeros((P, 9), dtype=torch.float32, device=cuda)
    for k, (r, dL) in enumerate(zip(rs, dLs)):
        r.render_backward(dL, pol, grad=g0, chained=k > 0)
    plain = torch.zeros((P, 9), dtype=torch.float32, device=cuda)
    for r, dL in zip(rs, dLs):
        r.render_backward(dL, pol, grad=plain)
    chain = torch.zeros((P, 9), dtype=torch.float32, device=cuda)
    for rep in range(3):  # back-to-back chains: launches overlap their neighbours
        for k, (r, dL) in enumerate(zip(rs, dLs)):
            r.render_backward(dL, pol, grad=chain, chained=k > 0 or rep > 0)
    want = plain.cpu().numpy().astype(np.float64)
    _grad_close(g0.cpu().numpy().astype(np.float64), want)
    _grad_close(chain.cpu().numpy().astype(np.float64) / 3.0, want)
    with pytest.raises(ValueError):
        rs[0].render_backward(dLs[0], pol, chained=True)  # needs a given gradient


@pytest.mark.parametrize("policy", ["sw_b", "sw_s", "native", "cccl"])
def test_backward_views_batch_equals_plain(cuda, policy):
    """dw_render_backward_views (one chain; SW-B / SW-S through the padded
    [P][12] accumulation folded into grad) == plain per-view launches, and it
    ADDS into grad like render_backward."""
    import torch

    from paper_2401_05345_b200 import warpred as wr
    from paper_2401_05345_b200.rasterizer import GaussianRasterizer, render_backward_views
    from paper_2401_05345_b200.scene import make_dL_dpixels, orbit_cameras

    P, W, H = 25000, 288, 200
    sc = _scene(cuda, P, W, H, seed=44)
    args = [sc[k] for k in SCENE_KEYS]
    cams = orbit_cameras(W, H, 3)
    dLs = [torch.from_numpy(make_dL_dpixels(W, H, seed=50 + k)).to(cuda) for k in range(3)]
    pol = wr.Policy(wr.parse_policy_kind(policy), 12 if policy in ("sw_b", "sw_s") else 0)
    rs = []
    for c in cams:
        r = GaussianRasterizer()
        r.render_forward(*args, c)
        rs.append(r)
    plain = torch.zeros((P, 9), dtype=torch.float32, device=cuda)
    for r, dL in zip(rs, dLs):
        r.render_backward(dL, pol, grad=plain)
    batch = torch.full((P, 9), 0.5, dtype=torch.float32, device=cuda)
    for _ in range(2):  # the padded buffer is left zeroed for the next batch
        render_backward_views(rs, dLs, pol, batch)
    want = 2 * plain.cpu().numpy().astype(np.float64) + 0.5
    _grad_close(batch.cpu().numpy().astype(np.float64), want)


def test_backward_views_batch_full_size_c5(cuda):
    """BASELINE configs[4] at full size (3M Gaussians, 1080p): bench.py's timed
    call -- the batch of views as one dw_render_backward_views chain into the
    padded rows -- equals plain per-view launches (here three orbit views)."""
    import torch

    from paper_2401_05345_b200 import warpred as wr
    from paper_2401_05345_b200.rasterizer import GaussianRasterizer, render_backward_views
    from paper_2401_05345_b200.scene import CONFIGS, make_dL_dpixels, orbit_cameras

    P, W, H, _, V = CONFIGS["c5_3m_1080p_64views"]
    sc = _scene(cuda, P, W, H, seed=0)
    args = [sc[k] for k in SCENE_KEYS]
    cams = [orbit_cameras(W, H, V)[k] for k in (0, 21, 63)]
    dLs = [torch.from_numpy(make_dL_dpixels(W, H, seed=1 + k)).to(cuda) for k in range(3)]
    pol = wr.Policy(wr.PolicyKind.sw_b, 16)
    rs = []
    for c in cams:
        r = GaussianRasterizer()
        r.render_forward(*args, c)
        rs.append(r)
    plain = torch.zeros((P, 9), dtype=torch.float32, device=cuda)
    for r, dL in zip(rs, dLs):
        r.render_backward(dL, pol, grad=plain)
    batch = torch.zeros((P, 9), dtype=torch.float32, device=cuda)
    render_backward_views(rs, dLs, pol, batch)
    _grad_close(batch.cpu().numpy().astype(np.float64), plain.cpu().numpy().astype(np.float64))


@pytest.mark.parametrize("wave,fstreams,stack", [(2, 4, 1), (3, 1, 1), (1, 2, 2), (2, 3, 3)])
def test_views_host_multi_wave(cuda, monkeypatch, wave, fstreams, stack):
    """Batches longer than one wave: the pool states are reused wave after
    wave (a wave's forwards wait for the previous wave's chain and image
    downloads), over 1-4 forward streams, with and without stacked frames --
    images bit for bit and gradients equal to the default (one wave)."""
    from paper_2401_05345_b200.scene import make_dL_dpixels, make_scene, orbit_cameras

    P, W, H, V = 9000, 176, 128, 9
    sc = make_scene(P, W, H, seed=17)
    cams = orbit_cameras(W, H, V)
    dL = np.stack([make_dL_dpixels(W, H, seed=300 + k) for k in range(V)]).astype(np.float32)
    ref = _views_host(monkeypatch, 1, sc, cams, dL)
    got = _views_host(monkeypatch, stack, sc, cams, dL, wave=wave, fstreams=fstreams)
    for (gi, gg), (ri, rg) in zip(got, ref):
        assert np.array_equal(gi, ri)
        _grad_close(gg, rg)


def test_backward_views_batch_in_cuda_graph(cuda):
    """The batch call (one chain of programmatic-dependent launches, padded
    rows, fold) enqueues no host sync or allocation after its first call, so
    it captures into a CUDA graph; two replays add twice the eager batch."""
    import torch

    from paper_2401_05345_b200 import warpred as wr
    from paper_2401_05345_b200.rasterizer import GaussianRasterizer, render_backward_views
    from paper_2401_05345_b200.scene import make_dL_dpixels, orbit_cameras

    P, W, H = 20000, 256, 192
    sc = _scene(cuda, P, W, H, seed=61)
    args = [sc[k] for k in SCENE_KEYS]
    cams = orbit_cameras(W, H, 4)
    dLs = [torch.from_numpy(make_dL_dpixels(W, H, seed=70 + k)).to(cuda) for k in range(4)]
    pol = wr.Policy(wr.PolicyKind.sw_b, 12)
    rs = []
    for c in cams:
        r = GaussianRasterizer()
        r.render_forward(*args, c)
        rs.append(r)
    eager = torch.zeros((P, 9), dtype=torch.float32, device=cuda)
    render_backward_views(rs, dLs, pol, eager)  # also sizes the padded buffer
    torch.cuda.synchronize()
    g = torch.zeros((P, 9), dtype=torch.float32, device=cuda)
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.stream(side):
        with torch.cuda.graph(graph, stream=side):
            render_backward_views(rs, dLs, pol, g, stream=side)
    torch.cuda.synchronize()
    assert float(g.abs().sum()) == 0.0  # capture did not run
    graph.replay()
    graph.replay()
    torch.cuda.synchronize()
    _grad_close(g.cpu().numpy().astype(np.float64), 2 * eager.cpu().numpy().astype(np.float64))
