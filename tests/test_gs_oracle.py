"""CPU: pin the Gaussian-splatting oracle (oracle/gs_oracle.c) independently.

The reference has no rasterizer, so this oracle is not reference-pinned; it is
instead checked against independent float64 numpy restatements:
  * projection (means2D, depth, 2D covariance -> conic, radius) in float64;
  * binning invariants (sorted keys, ranges, instance <-> rect coverage);
  * the blended image against a brute-force per-Gaussian numpy blend;
  * its analytic backward against central finite differences of that numpy
    blend w.r.t. the 2D parameters (3DGS conventions: mean2D gradients are
    w.r.t. NDC (x 0.5 W), the conic off-diagonal gradient is half of d/db).
"""
import ctypes as C
import math

import numpy as np
import pytest

from oracle.bindings import Camera as OCam


def ocam(cam):
    oc = OCam()
    cc = cam.to_c()
    C.memmove(C.byref(oc), C.byref(cc), C.sizeof(oc))
    return oc


def project64(sc, cam):
    """float64 projection of every Gaussian (independent of the C code)."""
    V = np.asarray(cam.viewmatrix, np.float64)
    Pm = np.asarray(cam.projmatrix, np.float64)
    m = sc["means3D"].astype(np.float64)
    mh = np.concatenate([m, np.ones((len(m), 1))], 1)
    tv = mh @ V.T
    ph = mh @ Pm.T
    ndc = ph[:, :3] / (ph[:, 3:4] + 1e-7)
    W, H = cam.width, cam.height
    pix = np.stack([((ndc[:, 0] + 1) * W - 1) / 2, ((ndc[:, 1] + 1) * H - 1) / 2], 1)
    q = sc["rotations"].astype(np.float64)
    q = q / np.linalg.norm(q, axis=1, keepdims=True)
    r, x, y, z = q.T
    R = np.stack([np.stack([1 - 2 * (y * y + z * z), 2 * (x * y - r * z), 2 * (x * z + r * y)], -1),
                  np.stack([2 * (x * y + r * z), 1 - 2 * (x * x + z * z), 2 * (y * z - r * x)], -1),
                  np.stack([2 * (x * z - r * y), 2 * (y * z + r * x), 1 - 2 * (x * x + y * y)], -1)],
                 1)
    S = sc["scales"].astype(np.float64) * cam.scale_modifier
    Sig = R @ (S[:, :, None] ** 2 * np.transpose(R, (0, 2, 1)))
    fx = W / (2 * cam.tan_fovx)
    fy = H / (2 * cam.tan_fovy)
    tz = tv[:, 2]
    tx = np.clip(tv[:, 0] / tz, -1.3 * cam.tan_fovx, 1.3 * cam.tan_fovx) * tz
    ty = np.clip(tv[:, 1] / tz, -1.3 * cam.tan_fovy, 1.3 * cam.tan_fovy) * tz
    J = np.zeros((len(m), 2, 3))
    J[:, 0, 0] = fx / tz
    J[:, 0, 2] = -fx * tx / tz ** 2
    J[:, 1, 1] = fy / tz
    J[:, 1, 2] = -fy * ty / tz ** 2
    T = J @ V[:3, :3]
    cov = T @ Sig @ np.transpose(T, (0, 2, 1)) + 0.3 * np.eye(2)
    a, b, c = cov[:, 0, 0], cov[:, 0, 1], cov[:, 1, 1]
    det = a * c - b * b
    conic = np.stack([c / det, -b / det, a / det], 1)
    mid = 0.5 * (a + c)
    lam = mid + np.sqrt(np.maximum(0.1, mid * mid - det))
    radius = np.ceil(3 * np.sqrt(lam))
    return pix, tz, conic, radius


@pytest.fixture(scope="module")
def small(orc):
    from paper_2401_05345_b200.scene import make_camera, make_dL_dpixels, make_scene

    sc = make_scene(400, 96, 64, seed=21)
    cam = make_camera(96, 64, yaw_deg=7.0)
    dL = make_dL_dpixels(96, 64, seed=22)
    return sc, cam, dL, orc.gs_render(sc, ocam(cam), dL)


def test_projection_matches_float64(small):
    sc, cam, _, ref = small
    pix, depth, conic, radius = project64(sc, cam)
    vis = ref["radii"] > 0
    assert vis.sum() > 300
    np.testing.assert_allclose(ref["means2D"][vis], pix[vis], rtol=0, atol=2e-3)
    np.testing.assert_allclose(ref["depths"][vis], depth[vis], rtol=1e-6)
    np.testing.assert_allclose(ref["conic_opacity"][vis, :3], conic[vis], rtol=2e-3,
                               atol=1e-6 * np.abs(conic[vis]).max())
    assert np.mean(ref["radii"][vis] == radius[vis]) > 0.98  # ceil() boundary cases aside
    np.testing.assert_array_equal(ref["conic_opacity"][vis, 3], sc["opacities"][vis])


def test_binning_invariants(small):
    sc, cam, _, ref = small
    keys, vals, ranges = ref["keys"], ref["values"], ref["ranges"]
    assert ref["num_rendered"] == int(ref["tiles_touched"].sum()) == len(keys)
    assert np.all(keys[1:] >= keys[:-1])
    tiles_x = (cam.width + 15) // 16
    tile = (keys >> np.uint64(32)).astype(np.int64)
    depth_bits = (keys & np.uint64(0xFFFFFFFF)).astype(np.uint32)
    np.testing.assert_array_equal(depth_bits.view(np.float32), ref["depths"][vals])
    for t in range(len(ranges)):
        s, e = ranges[t]
        assert np.all(tile[s:e] == t)
    # every instance lies inside its Gaussian's rect, and rect areas match
    for i in np.flatnonzero(ref["radii"] > 0)[:50]:
        ts = tile[vals == i]
        assert len(ts) == ref["tiles_touched"][i]
        x, y = ref["means2D"][i]
        rr = ref["radii"][i]
        tx, ty = ts % tiles_x, ts // tiles_x
        assert np.all(tx >= max(0, int((x - rr) / 16))) and np.all(ty >= max(0, int((y - rr) / 16)))
    # stable sort: equal keys keep ascending Gaussian order
    eq = keys[1:] == keys[:-1]
    assert np.all(vals[1:][eq] > vals[:-1][eq])


def blend64(order, tiles_of, xy, conic, opac, col, W, H, bg, need_state=False):
    """Brute-force float64 front-to-back blend, vectorised over pixels."""
    py, px = np.mgrid[0:H, 0:W].astype(np.float64)
    ptile = (py // 16).astype(int) * ((W + 15) // 16) + (px // 16).astype(int)
    T = np.ones((H, W))
    C_ = np.zeros((3, H, W))
    done = np.zeros((H, W), bool)
    for g in order:
        m = np.isin(ptile, tiles_of[g]) & ~done
        dx, dy = xy[g, 0] - px, xy[g, 1] - py
        power = -0.5 * (conic[g, 0] * dx * dx + conic[g, 2] * dy * dy) - conic[g, 1] * dx * dy
        alpha = np.minimum(0.99, opac[g] * np.exp(power))
        ok = m & (power <= 0) & (alpha >= 1 / 255)
        test_T = T * (1 - alpha)
        stop = ok & (test_T < 1e-4)
        done |= stop
        ok &= ~stop
        C_ += np.where(ok, col[g][:, None, None] * alpha * T, 0)
        T = np.where(ok, test_T, T)
    return C_ + T * np.asarray(bg)[:, None, None]


def _tiles_and_order(ref):
    keys, vals = ref["keys"], ref["values"]
    tile = (keys >> np.uint64(32)).astype(np.int64)
    tiles_of = {}
    for t, v in zip(tile, vals):
        tiles_of.setdefault(int(v), []).append(int(t))
    vis = np.flatnonzero(ref["radii"] > 0)
    order = vis[np.lexsort((vis, ref["depths"][vis]))]
    return tiles_of, order


def test_forward_matches_bruteforce(small):
    sc, cam, _, ref = small
    tiles_of, order = _tiles_and_order(ref)
    img = blend64(order, tiles_of, ref["means2D"].astype(np.float64),
                  ref["conic_opacity"][:, :3].astype(np.float64),
                  ref["conic_opacity"][:, 3].astype(np.float64), sc["colors"].astype(np.float64),
                  cam.width, cam.height, cam.bg)
    err = np.abs(img - ref["image"])
    assert err.max() < 2e-2 and np.mean(err > 1e-4) < 2e-3


def test_backward_matches_finite_differences(orc):
    from paper_2401_05345_b200.scene import make_camera, make_dL_dpixels, make_scene

    W, H = 40, 32
    sc = make_scene(24, W, H, seed=5)
    cam = make_camera(W, H)
    dL = make_dL_dpixels(W, H, seed=6).astype(np.float64)
    ref = orc.gs_render(sc, ocam(cam), dL.astype(np.float32))
    tiles_of, order = _tiles_and_order(ref)
    xy = ref["means2D"].astype(np.float64)
    con = ref["conic_opacity"][:, :3].astype(np.float64)
    op = ref["conic_opacity"][:, 3].astype(np.float64)
    col = sc["colors"].astype(np.float64)

    def loss(xy_, con_, op_, col_):
        return float((dL * blend64(order, tiles_of, xy_, con_, op_, col_, W, H, cam.bg)).sum())

    rng = np.random.default_rng(0)
    checked = 0
    for g in rng.permutation(order)[:12]:
        want = ref["grad"][g]
        if np.abs(want).max() == 0:
            continue
        fd = np.zeros(9)
        for p in range(9):
            h = 1e-5 if p in (0, 1) else (1e-7 if p in (2, 3, 4) else 1e-6)
            args = [xy.copy(), con.copy(), op.copy(), col.copy()]
            tgt = {0: (0, 0), 1: (0, 1), 2: (1, 0), 3: (1, 1), 4: (1, 2), 5: (2, None),
                   6: (3, 0), 7: (3, 1), 8: (3, 2)}[p]
            vals = []
            for s in (+1, -1):
                a = [x.copy() for x in args]
                if tgt[1] is None:
                    a[tgt[0]][g] += s * h
                else:
                    a[tgt[0]][g, tgt[1]] += s * h
                vals.append(loss(*a))
            fd[p] = (vals[0] - vals[1]) / (2 * h)
        fd[0] *= 0.5 * W  # d/d ndc.x
        fd[1] *= 0.5 * H
        fd[3] *= 0.5      # symmetric off-diagonal convention
        scale = np.abs(fd).max()
        np.testing.assert_allclose(want, fd, rtol=2e-3, atol=2e-3 * scale)
        checked += 1
    assert checked >= 8


def test_tap_records_reproduce_gradients(orc, small):
    """The per-warp WarpRecords the backward emits sum (oracle_sum) to the
    backward's own per-address gradients, and every record is warp-uniform."""
    sc, cam, dL, _ = small
    ref = orc.gs_render(sc, ocam(cam), dL, tap=True)
    tap = ref["tap"]
    P = sc["means3D"].shape[0]
    sums, _ = orc.oracle_sum(tap, P)
    np.testing.assert_allclose(sums.reshape(P, 9), ref["grad"], rtol=1e-12, atol=1e-12)
    assert np.all(tap.prim == tap.prim[:, :1])
    assert tap.contributions() == 9 * ref["pairs"]
    hist = np.bincount(np.unpackbits(tap.active.view(np.uint8).reshape(-1, 4), axis=1).sum(1),
                       minlength=33)
    assert hist[0] == 0  # only records with an active lane are emitted


def test_multithreaded_backward_equals_single(orc, small):
    sc, cam, dL, ref1 = small
    ref8 = orc.gs_render(sc, ocam(cam), dL, threads=8)
    np.testing.assert_allclose(ref8["grad"], ref1["grad"], rtol=1e-12, atol=1e-12)
    assert ref8["pairs"] == ref1["pairs"]
    np.testing.assert_array_equal(ref8["image"], ref1["image"])


def test_preprocess_backward_matches_finite_differences(orc):
    """3D gradients (means, scales, quaternion, opacity, colour) of the oracle
    vs central differences of the float64 projection + blend chain."""
    from oracle.bindings import gs_train_grads
    from paper_2401_05345_b200.scene import make_camera, make_dL_dpixels, make_scene

    W, H = 40, 32
    sc = make_scene(16, W, H, seed=8)
    cam = make_camera(W, H, yaw_deg=6.0)
    dL = make_dL_dpixels(W, H, seed=9).astype(np.float64)
    ref = orc.gs_render(sc, ocam(cam), dL.astype(np.float32))
    tiles_of, order = _tiles_and_order(ref)
    _, g3 = gs_train_grads(orc, sc, ocam(cam), dL.astype(np.float32), threads=1)

    def loss(s):
        pix, _, conic, _ = project64(s, cam)
        return float((dL * blend64(order, tiles_of, pix, conic,
                                   s["opacities"].astype(np.float64),
                                   s["colors"].astype(np.float64), W, H, cam.bg)).sum())

    base = {k: v.astype(np.float64) for k, v in sc.items()}
    checked = 0
    rng = np.random.default_rng(1)
    for g in rng.permutation(order)[:8]:
        want = g3[g]
        fd = np.zeros(14)
        slots = [("means3D", 0), ("means3D", 1), ("means3D", 2), ("scales", 0), ("scales", 1),
                 ("scales", 2), ("rotations", 0), ("rotations", 1), ("rotations", 2),
                 ("rotations", 3), ("opacities", None), ("colors", 0), ("colors", 1),
                 ("colors", 2)]
        for p, (key, col) in enumerate(slots):
            h = 1e-6 * max(1.0, abs(base[key][g] if col is None else base[key][g, col]))
            vals = []
            for sgn in (+1, -1):
                s = {k: v.copy() for k, v in base.items()}
                if col is None:
                    s[key][g] += sgn * h
                else:
                    s[key][g, col] += sgn * h
                vals.append(loss(s))
            fd[p] = (vals[0] - vals[1]) / (2 * h)
        scale = np.abs(fd).max()
        if scale == 0:
            continue
        np.testing.assert_allclose(want, fd, rtol=5e-3, atol=5e-3 * scale)
        checked += 1
    assert checked >= 6


def test_adam_reference_step(orc):
    from oracle.bindings import gs_adam

    rng = np.random.default_rng(0)
    p, g = rng.normal(size=50), rng.normal(size=50)
    m, v = np.zeros(50), np.zeros(50)
    p0 = p.copy()
    gs_adam(orc, p, g, m, v, 1e-3, 0.9, 0.999, 1e-8, 1)
    # first step of Adam: m_hat = g, v_hat = g^2 -> update lr * sign(g)
    np.testing.assert_allclose(p0 - p, 1e-3 * g / (np.abs(g) + 1e-8), rtol=1e-9)
