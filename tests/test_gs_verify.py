"""CPU: the decision-matched verification oracle (oracle/gs_verify.c), the
checker of tests/test_gpu_parity_full.py, pinned on its own:

* its lists (gs_forward_lists: depth-ordered bucketing) equal gs_forward's
  stable (tile | depth) radix sort, keys included, on every scene family;
* its float64 blend + backward equal gs_oracle.c's (itself checked against a
  brute-force numpy blend and finite differences in test_gs_oracle.py) up to
  fp32 rounding, and its gradients match central finite differences of a
  float64 blend directly;
* world matching: the oracle's own outputs match their default world with
  no flips, and a corrupted pixel (image or n_contrib) is reported as a
  mismatch -- the detection the GPU parity tests rely on;
* the bounds dominate the legacy fp32 oracle's deviation.
"""
import numpy as np
import pytest

from parity import U, grad_tol, ocam

SCENES = [("tiny", 300, 61, 47, False, 0), ("c1", 10_000, 256, 256, False, 0),
          ("contention", 2_000, 320, 200, True, 5), ("orbit", 5_000, 200, 144, False, 31)]


@pytest.fixture(scope="module", params=SCENES, ids=[s[0] for s in SCENES])
def case(request, orc):
    from paper_2401_05345_b200.scene import make_camera, make_dL_dpixels, make_scene

    name, P, W, H, hc, seed = request.param
    sc = make_scene(P, W, H, seed=seed, high_contention=hc)
    cam = make_camera(W, H, yaw_deg=7.0 if name == "orbit" else 0.0)
    dL = make_dL_dpixels(W, H, seed=seed + 1)
    ref = orc.gs_render(sc, ocam(cam), dL, threads=8)
    view = orc.gs_view(sc, ocam(cam), threads=8)
    return sc, cam, dL, ref, view


def test_lists_equal_radix_sort(case):
    _, _, _, ref, view = case
    got = view.lists()
    assert got["num_rendered"] == ref["num_rendered"]
    for k in ("means2D", "radii", "depths", "conic_opacity", "tiles_touched", "keys", "values",
              "ranges"):
        assert np.array_equal(got[k], ref[k]), k


def test_values_match_legacy_oracle(case):
    """Same algorithm, float64 vs fp32 arithmetic (and the exp form of the
    alpha test): images within 1e-4, gradients inside the verify bounds
    wherever the two agree on the contributor set."""
    _, _, dL, ref, view = case
    o, rep, _ = view.verify(dL)
    assert rep["pix_nomatch"] == 0 and rep["pix_world_cap"] == 0
    same = o["n_contrib"] == ref["n_contrib"]
    assert same.mean() > 0.999
    assert np.abs(o["image"] - ref["image"])[:, same].max() < 1e-4
    if same.all():
        assert abs(rep["pairs"] - ref["pairs"]) == 0
        rel = np.linalg.norm(o["grad"] - ref["grad"]) / np.linalg.norm(ref["grad"])
        assert rel < 2e-5, rel
        # the legacy oracle is itself an fp32 computation of the same terms
        assert np.all(np.abs(o["grad"] - ref["grad"]) <= grad_tol(o) + o["grad_abs"] * 1e-4)


def test_self_match_no_flips(case):
    """Fed its own outputs as the 'GPU' ones, every pixel matches the default
    world and nothing is flipped; grad and image are unchanged."""
    _, _, dL, _, view = case
    o, _, _ = view.verify(dL)
    gpu = (o["n_contrib"], o["final_T"].astype(np.float32), o["image"].astype(np.float32))
    o2, rep, flips = view.verify(dL, gpu=gpu)
    assert rep["pix_nomatch"] == 0 and rep["pix_flipped"] == 0 and not flips
    assert np.array_equal(o2["grad"], o["grad"])
    assert np.array_equal(o2["n_contrib"], o["n_contrib"])


def test_corrupted_pixel_is_a_mismatch(case):
    _, cam, dL, _, view = case
    o, _, _ = view.verify(dL)
    nc = o["n_contrib"].copy()
    T = o["final_T"].astype(np.float32)
    img = o["image"].astype(np.float32)
    y, x = cam.height // 2, cam.width // 3
    img_bad = img.copy()
    img_bad[1, y, x] += 1e-3
    o2, rep, _ = view.verify(dL, gpu=(nc, T, img_bad))
    assert rep["pix_nomatch"] == 1 and o2["status"][y, x] == 4
    nc_bad = nc.copy()
    nc_bad[y, x] += 1
    _, rep, _ = view.verify(dL, gpu=(nc_bad, T, img))
    assert rep["pix_nomatch"] == 1


def _blend64(view, lists, sc, W, H, bg, xy, con, op, col):
    """float64 front-to-back blend over the oracle's lists (tiny scenes)."""
    ranges, values = lists["ranges"], lists["values"]
    tiles_x = (W + 15) // 16
    img = np.zeros((3, H, W))
    for py in range(H):
        for px in range(W):
            t = (py // 16) * tiles_x + px // 16
            T, Cc = 1.0, np.zeros(3)
            for g in values[ranges[t, 0]:ranges[t, 1]]:
                dx, dy = xy[g, 0] - px, xy[g, 1] - py
                power = -0.5 * (con[g, 0] * dx * dx + con[g, 2] * dy * dy) - con[g, 1] * dx * dy
                if power > 0:
                    continue
                alpha = min(0.99, op[g] * np.exp(power))
                if alpha < 1 / 255:
                    continue
                tt = T * (1 - alpha)
                if tt < 1e-4:
                    break
                Cc += col[g] * alpha * T
                T = tt
            img[:, py, px] = Cc + T * np.asarray(bg)
    return img


def test_gradients_match_finite_differences(orc):
    from paper_2401_05345_b200.scene import make_camera, make_dL_dpixels, make_scene

    W, H = 40, 32
    sc = make_scene(24, W, H, seed=5)
    cam = make_camera(W, H)
    dL = make_dL_dpixels(W, H, seed=6)
    view = orc.gs_view(sc, ocam(cam), threads=2)
    lists = view.lists()
    o, rep, _ = view.verify(dL)
    assert rep["pix_ambiguous"] == 0
    xy = lists["means2D"].astype(np.float64)
    con = lists["conic_opacity"][:, :3].astype(np.float64)
    op = lists["conic_opacity"][:, 3].astype(np.float64)
    col = sc["colors"].astype(np.float64)
    d64 = dL.astype(np.float64)

    def loss(a):
        return float((d64 * _blend64(view, lists, sc, W, H, cam.bg, *a)).sum())

    img = _blend64(view, lists, sc, W, H, cam.bg, xy, con, op, col)
    assert np.abs(img - o["image"]).max() < 1e-5
    checked = 0
    for g in np.flatnonzero(o["npix"] > 0)[:10]:
        fd = np.zeros(9)
        for p in range(9):
            h = 1e-5 if p in (0, 1) else (1e-7 if p in (2, 3, 4) else 1e-6)
            tgt = {0: (0, 0), 1: (0, 1), 2: (1, 0), 3: (1, 1), 4: (1, 2), 5: (2, None),
                   6: (3, 0), 7: (3, 1), 8: (3, 2)}[p]
            vals = []
            for s in (+1, -1):
                a = [xy.copy(), con.copy(), op.copy(), col.copy()]
                if tgt[1] is None:
                    a[tgt[0]][g] += s * h
                else:
                    a[tgt[0]][g, tgt[1]] += s * h
                vals.append(loss(a))
            fd[p] = (vals[0] - vals[1]) / (2 * h)
        fd[0] *= 0.5 * W
        fd[1] *= 0.5 * H
        fd[3] *= 0.5
        np.testing.assert_allclose(o["grad"][g], fd, rtol=2e-3, atol=2e-3 * np.abs(fd).max())
        checked += 1
    assert checked >= 8


def test_bound_units():
    assert U == 2.0 ** -24
