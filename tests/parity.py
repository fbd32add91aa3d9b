"""Decision-matched parity of the GPU rasterizer against the verification
oracle (oracle/gs_verify.c) -- shared by the GPU parity tests.

The bars, all stated here and none fractional:

* lists: means2D / radii / tiles_touched / (tile | depth) keys / sorted
  values / tile ranges BIT-EXACT (keys skipped only where 64-bit keys of
  0.9 G instances would not fit the test's memory budget; values + ranges
  determine them);
* decisions: every pixel's (n_contrib, final_T, image) must be explained by
  one "world" of the oracle -- its own decisions with some subset of the
  AMBIGUOUS ones flipped (those whose operand lies inside the ex2.approx /
  transmittance error band, gs_verify.c). A pixel no world explains fails
  the test; the flipped decisions are enumerated and their number is
  bounded by FLIPS_PER_MPAIR per million blended pairs (and reported);
* n_contrib equal to the matched world's, exactly; the backward's
  contributing-pair count equal to the matched worlds' pair count, exactly;
* image per pixel and channel |gpu - oracle| <= KAPPA u E_pix |image|_mag
  (u = 2^-24, E_pix and the magnitude from the oracle);
* gradients per element |gpu - oracle| <= KAPPA u bound + (npix + 16) u |terms|
  + slack (gs_verify.c header: the running transmittance error bound per
  pixel times the absolute-valued term, plus fp32 summation of npix terms in
  any order; slack is the world spread of pixels whose outputs fit two
  worlds, normally zero) -- for EVERY element, no fraction excused;
* and the relative L2 error of the whole gradient below GRAD_REL_L2 (the
  naive-atomic policy on C4 excepted, whose ~6,600 fp32 atomic additions per
  address are a summation error of their own: 4e-5, stated in its test).
"""
from __future__ import annotations

import ctypes as C
import json
import os

import numpy as np

U = 2.0 ** -24
KAPPA = 1.0
FLIPS_PER_MPAIR = 1.0
GRAD_REL_L2 = 1e-5
THREADS = os.cpu_count() or 8
# DW_PARITY_MEASURE=1: log the ratios without asserting the numeric bars (the
# structural ones -- lists, world matching, pair counts -- still assert)
MEASURE = os.environ.get("DW_PARITY_MEASURE") == "1"


BINNING_ENV = {  # list constructions of the forward (raster.cu): env overrides
    "auto": {},
    "scatter": {"DW_SCATTER": "1", "DW_DENSE_BINNING": "0", "DW_TILE_FIRST": "0"},
    # depth sort, then duplicate + stable tile sort (the classic construction)
    "depth-first": {"DW_SCATTER": "0", "DW_DENSE_BINNING": "0", "DW_TILE_FIRST": "0",
                    "DW_BLOCK_BINNING": "0"},
    # depth sort, then coarse-block entries + per-tile appends (the default)
    "block": {"DW_SCATTER": "0", "DW_DENSE_BINNING": "0", "DW_TILE_FIRST": "0",
              "DW_BLOCK_BINNING": "1", "DW_BB_FUSED": "0"},
    # the same with the opt-in fused level 1 (per-tile histogram + emit)
    "block-fused": {"DW_SCATTER": "0", "DW_DENSE_BINNING": "0", "DW_TILE_FIRST": "0",
                    "DW_BLOCK_BINNING": "1", "DW_BB_FUSED": "1"},
    "tile-first": {"DW_SCATTER": "0", "DW_DENSE_BINNING": "0", "DW_TILE_FIRST": "1"},
    "dense": {"DW_DENSE_BINNING": "1"},
}


def set_binning(monkeypatch, mode: str) -> None:
    for k in ("DW_SCATTER", "DW_DENSE_BINNING", "DW_TILE_FIRST", "DW_BLOCK_BINNING"):
        monkeypatch.delenv(k, raising=False)
    for k, v in BINNING_ENV[mode].items():
        monkeypatch.setenv(k, v)


def ocam(cam):
    from oracle.bindings import Camera as OCam

    oc = OCam()
    cc = cam.to_c()
    C.memmove(C.byref(oc), C.byref(cc), C.sizeof(oc))
    return oc


def log_stats(rec: dict) -> None:
    path = os.environ.get("DW_PARITY_LOG")
    if path:
        with open(path, "a") as f:
            f.write(json.dumps(rec) + "\n")


def gpu_forward(cuda, sc, cam):
    import torch

    from paper_2401_05345_b200.rasterizer import GaussianRasterizer

    r = GaussianRasterizer()
    t = {k: torch.from_numpy(v).to(cuda) for k, v in sc.items()}
    img, radii, nr = r.render_forward(t["means3D"], t["scales"], t["rotations"],
                                      t["opacities"], t["colors"], cam)
    torch.cuda.synchronize()
    return r, img.cpu().numpy(), radii.cpu().numpy(), nr


def check_lists(r, radii, nr, lists, keys: bool):
    assert nr == lists["num_rendered"], (nr, lists["num_rendered"])
    assert np.array_equal(radii, lists["radii"])
    assert np.array_equal(r.buffer("means2D"), lists["means2D"])
    assert np.array_equal(r.buffer("tiles_touched"), lists["tiles_touched"])
    vis = lists["radii"] > 0
    assert np.array_equal(r.buffer("depths")[vis], lists["depths"][vis])
    assert np.array_equal(r.buffer("conic_opacity")[vis], lists["conic_opacity"][vis])
    assert np.array_equal(r.buffer("ranges"), lists["ranges"])
    assert np.array_equal(r.buffer("values"), lists["values"])
    if keys:
        assert np.array_equal(r.buffer("keys"), lists["keys"])


def check_forward(name, r, img, view, dL):
    """Match worlds; returns the oracle's outputs and report."""
    H, W = view.H, view.W
    nc = r.buffer("n_contrib").reshape(H, W)
    fT = r.buffer("final_T").reshape(H, W)
    # measure mode matches worlds under a wide tolerance so the ratios of a
    # failing case are still reported
    o, rep, flips = view.verify(dL, gpu=(nc, fT, img), kappa=64.0 if MEASURE else KAPPA)
    assert rep["pix_world_cap"] == 0, rep
    bad = np.argwhere(o["status"] == 4)
    assert rep["pix_nomatch"] == 0, (name, rep, bad[:8].tolist())
    assert np.array_equal(nc, o["n_contrib"])
    tol = KAPPA * U * o["epix"][None] * o["image_mag"] + 1e-30
    err = np.abs(img.astype(np.float64) - o["image"])
    ratio_img = float((err / tol).max()) if err.size else 0.0
    assert MEASURE or ratio_img <= 1.0, (name, ratio_img)
    assert MEASURE or rep["flips"] <= FLIPS_PER_MPAIR * rep["pairs"] / 1e6 + 2, (name, rep)
    return o, rep, flips, ratio_img


def grad_tol(o):
    """Per-element gradient bound of an oracle verify output (module doc)."""
    return (KAPPA * U * o["grad_bound"] + (o["npix"][:, None] + 16.0) * U * o["grad_abs"]
            + o["grad_slack"] + 1e-30)


def check_backward(name, r, dL_dev, policy, o, rep, rel_l2=GRAD_REL_L2):
    g, pairs = r.render_backward(dL_dev, policy, count_pairs=True)
    g = g.double().cpu().numpy()
    assert pairs == rep["pairs"], (name, policy, pairs, rep["pairs"])
    want = o["grad"]
    tol = grad_tol(o)
    err = np.abs(g - want)
    ratio = err / tol
    worst = np.unravel_index(int(np.argmax(ratio)), ratio.shape) if ratio.size else (0, 0)
    rmax = float(ratio[worst]) if ratio.size else 0.0
    rel = float(np.linalg.norm(g - want) / max(np.linalg.norm(want), 1e-30))
    assert MEASURE or rmax <= 1.0, (name, policy, rmax, worst, g[worst[0]].tolist(),
                         want[worst[0]].tolist(), tol[worst[0]].tolist())
    assert MEASURE or rel < rel_l2, (name, policy, rel)
    return rmax, rel


def verify_case(cuda, orc, name, sc, cam, dL, policies, keys=True, rel_l2=None):
    """Forward lists + decisions + image, then every policy's backward.
    Returns a stats dict (also appended to $DW_PARITY_LOG)."""
    import torch

    r, img, radii, nr = gpu_forward(cuda, sc, cam)
    view = orc.gs_view(sc, ocam(cam), threads=THREADS, with_keys=keys)
    check_lists(r, radii, nr, view.lists(), keys)
    o, rep, flips, ratio_img = check_forward(name, r, img, view, dL)
    dL_dev = torch.from_numpy(dL).to(cuda)
    stats = {"case": name, "instances": int(nr), "report": rep, "image_ratio_max": ratio_img,
             "flips": flips[:16], "policies": {}}
    for pol in policies:
        bar = (rel_l2 or {}).get(pol.kind.name, GRAD_REL_L2)
        rmax, rel = check_backward(name, r, dL_dev, pol, o, rep, bar)
        stats["policies"][f"{pol.kind.name}:{pol.threshold}"] = {"ratio_max": rmax,
                                                                 "rel_l2": rel}
    log_stats(stats)
    return stats


def oracle_views(orc, sc, cams, dLs):
    """Default-world oracle outputs of several views, for GPU paths that do
    not expose per-view decisions (render_views_host): the spread of every
    other world of an ambiguous pixel is added to the bounds (slack).
    Returns (images, image bounds, summed grad, summed per-element bound)."""
    imgs, ibounds, grad, bound = [], [], None, None
    for cam, dL in zip(cams, dLs):
        v = orc.gs_view(sc, ocam(cam), threads=THREADS)
        o, rep, _ = v.verify(dL)
        assert rep["pix_world_cap"] == 0, rep
        imgs.append(o["image"])
        ibounds.append(KAPPA * U * o["epix"][None] * o["image_mag"] + o["image_slack"] + 1e-30)
        t = grad_tol(o)
        grad = o["grad"] if grad is None else grad + o["grad"]
        bound = t if bound is None else bound + t
    return imgs, ibounds, grad, bound
