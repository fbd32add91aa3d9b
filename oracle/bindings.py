"""TEST INFRASTRUCTURE ONLY: ctypes bindings to the CPU oracles.

* ``Oracle`` -> ``oracle/liboracle.so``: the plain-C restatement of the
  reference's reduction stage (warpred_oracle.c) and the Gaussian-splatting
  CPU rasterizer (gs_oracle.c).
* ``Ref`` -> ``oracle/_ref/libwarpred_ref.so``: the UNMODIFIED reference
  sources compiled by ``oracle/Makefile`` plus ``ref_driver.cpp``.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline /
``--impl reference`` legs may import this module; the product package never
does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libwarpred_ref.so")

NATIVE, SW_S, SW_B, CCCL, HW_ATOMRED = 0, 1, 2, 3, 4
NPARAM = 9


class SceneSpec(C.Structure):
    """Layout of wr_scene_spec (reference include/warpred.h:42-53)."""

    _fields_ = [
        ("num_primitives", C.c_int32),
        ("params_per_primitive", C.c_int32),
        ("image_width", C.c_int32),
        ("image_height", C.c_int32),
        ("mean_fragment_span", C.c_double),
        ("fragments_per_pixel_mean", C.c_double),
        ("activity_prob", C.c_double),
        ("locality", C.c_double),
        ("seed", C.c_uint64),
        ("quantized_values", C.c_int32),
    ]


def scene(**kw) -> SceneSpec:
    """SceneSpec with the reference defaults (workload.hpp:16-36)."""
    s = SceneSpec(1024, 3, 64, 32, 64.0, 1.0, 1.0, 1.0, 0, 1)
    for k, v in kw.items():
        setattr(s, k, v)
    return s


class _OrTrace(C.Structure):
    _fields_ = [
        ("scene", SceneSpec),
        ("num_records", C.c_int64),
        ("capacity", C.c_int64),
        ("warp_id", C.POINTER(C.c_int32)),
        ("iteration", C.POINTER(C.c_int32)),
        ("active", C.POINTER(C.c_uint32)),
        ("prim", C.POINTER(C.c_int32)),
        ("grads", C.POINTER(C.c_double)),
    ]


class Camera(C.Structure):
    _fields_ = [
        ("width", C.c_int32),
        ("height", C.c_int32),
        ("viewmatrix", C.c_float * 16),
        ("projmatrix", C.c_float * 16),
        ("tan_fovx", C.c_float),
        ("tan_fovy", C.c_float),
        ("bg", C.c_float * 3),
        ("scale_modifier", C.c_float),
    ]


class _GsState(C.Structure):
    _fields_ = [
        ("P", C.c_int32), ("W", C.c_int32), ("H", C.c_int32),
        ("tiles_x", C.c_int32), ("tiles_y", C.c_int32),
        ("means2D", C.POINTER(C.c_float)),
        ("depths", C.POINTER(C.c_float)),
        ("radii", C.POINTER(C.c_int32)),
        ("conic_opacity", C.POINTER(C.c_float)),
        ("rgb", C.POINTER(C.c_float)),
        ("tiles_touched", C.POINTER(C.c_uint32)),
        ("num_rendered", C.c_int64),
        ("keys", C.POINTER(C.c_uint64)),
        ("values", C.POINTER(C.c_uint32)),
        ("ranges", C.POINTER(C.c_uint32)),
        ("out_color", C.POINTER(C.c_float)),
        ("final_T", C.POINTER(C.c_float)),
        ("n_contrib", C.POINTER(C.c_uint32)),
        ("tap_count", C.c_int64), ("tap_cap", C.c_int64),
        ("tap_warp", C.POINTER(C.c_int32)),
        ("tap_iter", C.POINTER(C.c_int32)),
        ("tap_active", C.POINTER(C.c_uint32)),
        ("tap_prim", C.POINTER(C.c_int32)),
        ("tap_grads", C.POINTER(C.c_double)),
        ("tap_ppt", C.c_int32),
    ]


class GsFlip(C.Structure):
    _fields_ = [("pixel", C.c_int32), ("position", C.c_uint32), ("gaussian", C.c_int32),
                ("kind", C.c_int32)]


class GsVerifyReport(C.Structure):
    _fields_ = [(k, C.c_int64) for k in (
        "pairs", "pairs_default", "amb_alpha", "amb_term", "pix_ambiguous", "pix_flipped",
        "flips", "pix_unresolved", "pix_nomatch", "pix_world_cap")] + [
        ("max_worlds", C.c_int32), ("nflip_rec", C.c_int32)]

    def as_dict(self):
        return {k: int(getattr(self, k)) for k, _ in self._fields_}


class GsVerifyOut(C.Structure):
    _fields_ = [("grad", C.c_void_p), ("grad_bound", C.c_void_p), ("grad_abs", C.c_void_p),
                ("grad_slack", C.c_void_p), ("npix", C.c_void_p), ("image", C.c_void_p),
                ("image_mag", C.c_void_p), ("image_slack", C.c_void_p), ("final_T", C.c_void_p), ("epix", C.c_void_p),
                ("n_contrib", C.c_void_p), ("status", C.c_void_p), ("flips", C.c_void_p),
                ("flip_cap", C.c_int32), ("nflip_rec", C.c_int32)]


U_F32 = 2.0 ** -24


def _arr(ptr, n, dtype):
    if n == 0:
        return np.zeros(0, dtype=dtype)
    return np.ctypeslib.as_array(ptr, shape=(n,)).astype(dtype, copy=True)


def build(ref: bool = False) -> None:
    subprocess.run(["make", "-s", "-C", HERE], check=True)
    if ref and os.path.isdir("/root/reference/proj"):
        subprocess.run(["make", "-s", "-C", HERE, "ref"], check=True)


class Trace:
    """Flat numpy view of a WarpRecord trace (lane-major f64 grads)."""

    def __init__(self, spec, warp_id, iteration, active, prim, grads):
        self.spec = spec
        self.warp_id = warp_id
        self.iteration = iteration
        self.active = active
        self.prim = prim.reshape(-1, 32)
        n = spec.params_per_primitive
        self.grads = grads.reshape(-1, 32, n)

    @property
    def num_records(self):
        return int(self.active.shape[0])

    @property
    def n(self):
        return int(self.spec.params_per_primitive)

    def contributions(self) -> int:
        pc = np.unpackbits(self.active.view(np.uint8)).sum()
        return int(pc) * self.n


class Oracle:
    """The C restatement (liboracle.so)."""

    def __init__(self, path: str = ORACLE_SO):
        if not os.path.exists(path):
            build()
        L = self.L = C.CDLL(path)
        L.or_last_error.restype = C.c_char_p
        L.or_generate.argtypes = [C.POINTER(SceneSpec), C.POINTER(C.POINTER(_OrTrace))]
        L.or_trace_free.argtypes = [C.POINTER(_OrTrace)]
        L.or_trace_new.argtypes = [C.POINTER(SceneSpec)]
        L.or_trace_new.restype = C.POINTER(_OrTrace)
        L.or_record_policy.argtypes = [
            C.c_uint32, C.c_void_p, C.c_void_p, C.c_int32, C.c_int, C.c_int,
            C.c_void_p, C.c_void_p, C.c_void_p, C.POINTER(C.c_int64),
            C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)]
        L.or_apply_policy.argtypes = [C.POINTER(_OrTrace), C.c_int, C.c_int, C.c_int32,
                                      C.c_void_p, C.c_void_p]
        L.or_oracle_sum.argtypes = [C.POINTER(_OrTrace), C.c_int32, C.c_void_p, C.c_void_p]
        L.or_histograms.argtypes = [C.POINTER(_OrTrace), C.c_void_p, C.c_void_p]
        L.or_save_binary.argtypes = [C.POINTER(_OrTrace), C.c_char_p]
        L.or_load_binary.argtypes = [C.c_char_p, C.POINTER(C.POINTER(_OrTrace))]
        L.gs_last_error.restype = C.c_char_p
        L.gs_state_new.restype = C.POINTER(_GsState)
        L.gs_state_free.argtypes = [C.POINTER(_GsState)]
        L.gs_forward.argtypes = [C.POINTER(_GsState), C.c_int32] + [C.c_void_p] * 5 + [
            C.POINTER(Camera), C.c_int]
        L.gs_backward.argtypes = [C.POINTER(_GsState), C.POINTER(Camera), C.c_void_p,
                                  C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.c_int,
                                  C.POINTER(C.c_int64)]

        L.gs_forward_lists.argtypes = [C.POINTER(_GsState), C.c_int32] + [C.c_void_p] * 5 + [
            C.POINTER(Camera), C.c_int, C.c_int]
        L.gs_verify_last_error.restype = C.c_char_p
        L.gs_verify.argtypes = [C.POINTER(_GsState), C.POINTER(Camera), C.c_void_p, C.c_void_p,
                                C.c_void_p, C.c_void_p, C.c_double, C.POINTER(GsVerifyOut),
                                C.POINTER(GsVerifyReport), C.c_int]

    def _check(self, rc):
        if rc != 0:
            raise RuntimeError(self.L.or_last_error().decode())

    # -- decision-matched verification (gs_verify.c) ---------------------
    def gs_view(self, scene, cam: "Camera", threads=8, with_keys=True) -> "GsView":
        """Projection + per-tile lists (gs_forward_lists), no blend."""
        return GsView(self, scene, cam, threads, with_keys)

    # -- traces ---------------------------------------------------------
    def _to_numpy(self, tp) -> Trace:
        t = tp.contents
        r, n = t.num_records, t.scene.params_per_primitive
        spec = SceneSpec()
        C.pointer(spec)[0] = t.scene
        return Trace(spec, _arr(t.warp_id, r, np.int32), _arr(t.iteration, r, np.int32),
                     _arr(t.active, r, np.uint32), _arr(t.prim, r * 32, np.int32),
                     _arr(t.grads, r * 32 * n, np.float64))

    def _from_numpy(self, tr: Trace):
        tp = self.L.or_trace_new(C.byref(tr.spec))
        t = tp.contents
        r = tr.num_records
        keep = [np.ascontiguousarray(tr.warp_id, np.int32),
                np.ascontiguousarray(tr.iteration, np.int32),
                np.ascontiguousarray(tr.active, np.uint32),
                np.ascontiguousarray(tr.prim, np.int32),
                np.ascontiguousarray(tr.grads, np.float64)]
        t.num_records = r
        t.capacity = 0  # arrays are borrowed; detached before free
        t.warp_id = keep[0].ctypes.data_as(C.POINTER(C.c_int32))
        t.iteration = keep[1].ctypes.data_as(C.POINTER(C.c_int32))
        t.active = keep[2].ctypes.data_as(C.POINTER(C.c_uint32))
        t.prim = keep[3].ctypes.data_as(C.POINTER(C.c_int32))
        t.grads = keep[4].ctypes.data_as(C.POINTER(C.c_double))
        return tp, keep

    def _release(self, tp):
        t = tp.contents
        t.warp_id = t.iteration = t.prim = None
        t.active = None
        t.grads = None
        self.L.or_trace_free(tp)

    def generate(self, spec: SceneSpec) -> Trace:
        tp = C.POINTER(_OrTrace)()
        self._check(self.L.or_generate(C.byref(spec), C.byref(tp)))
        try:
            return self._to_numpy(tp)
        finally:
            self.L.or_trace_free(tp)

    def load_binary(self, path: str) -> Trace:
        tp = C.POINTER(_OrTrace)()
        self._check(self.L.or_load_binary(path.encode(), C.byref(tp)))
        try:
            return self._to_numpy(tp)
        finally:
            self.L.or_trace_free(tp)

    def save_binary(self, tr: Trace, path: str) -> None:
        tp, keep = self._from_numpy(tr)
        try:
            self._check(self.L.or_save_binary(tp, path.encode()))
        finally:
            self._release(tp)

    def oracle_sum(self, tr: Trace, num_prims: int):
        tp, keep = self._from_numpy(tr)
        sums = np.zeros(num_prims * tr.n, np.float64)
        touched = np.zeros(num_prims * tr.n, np.uint8)
        try:
            self._check(self.L.or_oracle_sum(tp, num_prims, sums.ctypes.data,
                                             touched.ctypes.data))
        finally:
            self._release(tp)
        return sums, touched.astype(bool)

    def apply_policy(self, tr: Trace, kind: int, threshold: int, num_prims: int):
        tp, keep = self._from_numpy(tr)
        sums = np.zeros(num_prims * tr.n, np.float64)
        counts = np.zeros(3, np.uint64)
        try:
            self._check(self.L.or_apply_policy(tp, kind, threshold, num_prims,
                                               sums.ctypes.data, counts.ctypes.data))
        finally:
            self._release(tp)
        return sums, {"requests": int(counts[0]), "instructions": int(counts[1]),
                      "fp_adds": int(counts[2])}

    def histograms(self, tr: Trace):
        tp, keep = self._from_numpy(tr)
        d = np.zeros(33, np.uint64)
        a = np.zeros(33, np.uint64)
        try:
            self._check(self.L.or_histograms(tp, d.ctypes.data, a.ctypes.data))
        finally:
            self._release(tp)
        return d, a

    def record_policy(self, active, prim, grads, kind, threshold):
        prim = np.ascontiguousarray(prim, np.int32)
        grads = np.ascontiguousarray(grads, np.float64)
        n = grads.size // 32
        op = np.zeros(32 * n, np.int32)
        oq = np.zeros(32 * n, np.int32)
        ov = np.zeros(32 * n, np.float64)
        cnt, ins, fp = C.c_int64(), C.c_uint64(), C.c_uint64()
        self._check(self.L.or_record_policy(int(active), prim.ctypes.data, grads.ctypes.data,
                                            n, kind, threshold, op.ctypes.data,
                                            oq.ctypes.data, ov.ctypes.data, C.byref(cnt),
                                            C.byref(ins), C.byref(fp)))
        c = cnt.value
        return (list(zip(op[:c].tolist(), oq[:c].tolist(), ov[:c].tolist())),
                ins.value, fp.value)

    # -- Gaussian rasterizer ---------------------------------------------
    def gs_render(self, scene, cam: Camera, dL_dpixels=None, threads=1, tile_stride=1,
                  tap=False, backward=True, tap_ppt=1):
        """Forward (+ backward) on the CPU oracle. Returns a dict of arrays.
        tap_ppt selects the record layout of the tap: 1 = one pixel per lane
        (8x4 per warp), 2 = the GPU reduction kernel's two pixels per lane."""
        L = self.L
        st = L.gs_state_new()
        P = int(scene["means3D"].shape[0])
        ins = [np.ascontiguousarray(scene[k], np.float32)
               for k in ("means3D", "scales", "rotations", "opacities", "colors")]
        try:
            rc = L.gs_forward(st, P, *[a.ctypes.data for a in ins], C.byref(cam), threads)
            if rc:
                raise RuntimeError(L.gs_last_error().decode())
            s = st.contents
            W, H = s.W, s.H
            ntiles = s.tiles_x * s.tiles_y
            nr = s.num_rendered
            out = {
                "means2D": _arr(s.means2D, 2 * P, np.float32).reshape(P, 2),
                "depths": _arr(s.depths, P, np.float32),
                "radii": _arr(s.radii, P, np.int32),
                "conic_opacity": _arr(s.conic_opacity, 4 * P, np.float32).reshape(P, 4),
                "tiles_touched": _arr(s.tiles_touched, P, np.uint32),
                "num_rendered": int(nr),
                "keys": _arr(s.keys, nr, np.uint64),
                "values": _arr(s.values, nr, np.uint32),
                "ranges": _arr(s.ranges, 2 * ntiles, np.uint32).reshape(ntiles, 2),
                "image": _arr(s.out_color, 3 * H * W, np.float32).reshape(3, H, W),
                "final_T": _arr(s.final_T, H * W, np.float32).reshape(H, W),
                "n_contrib": _arr(s.n_contrib, H * W, np.uint32).reshape(H, W),
            }
            if backward and dL_dpixels is not None:
                dL = np.ascontiguousarray(dL_dpixels, np.float32)
                grad = np.zeros(P * NPARAM, np.float64)
                gabs = np.zeros(P * NPARAM, np.float64)
                pairs = C.c_int64()
                st.contents.tap_ppt = tap_ppt
                rc = L.gs_backward(st, C.byref(cam), dL.ctypes.data, grad.ctypes.data,
                                   gabs.ctypes.data, threads, tile_stride, 1 if tap else 0,
                                   C.byref(pairs))
                if rc:
                    raise RuntimeError(L.gs_last_error().decode())
                out["grad"] = grad.reshape(P, NPARAM)
                out["grad_abs"] = gabs.reshape(P, NPARAM)
                out["pairs"] = int(pairs.value)
                if tap:
                    r = s.tap_count
                    out["tap"] = Trace(
                        scene_spec_for(P, NPARAM), _arr(s.tap_warp, r, np.int32),
                        _arr(s.tap_iter, r, np.int32), _arr(s.tap_active, r, np.uint32),
                        _arr(s.tap_prim, 32 * r, np.int32),
                        _arr(s.tap_grads, 32 * NPARAM * r, np.float64))
            return out
        finally:
            L.gs_state_free(st)

    def gs_prepare(self, scene, cam, threads):
        """CPU forward; returns an opaque state for gs_backward_timed."""
        L = self.L
        st = L.gs_state_new()
        P = int(scene["means3D"].shape[0])
        ins = [np.ascontiguousarray(scene[k], np.float32)
               for k in ("means3D", "scales", "rotations", "opacities", "colors")]
        if L.gs_forward(st, P, *[a.ctypes.data for a in ins], C.byref(cam), threads):
            L.gs_state_free(st)
            raise RuntimeError(L.gs_last_error().decode())
        return st

    def gs_free(self, st):
        self.L.gs_state_free(st)

    def gs_backward_timed(self, st, cam, dL_dpixels, threads, tile_stride, tap=0):
        """(seconds, pairs, tapped Trace or None) of the CPU backward over a
        strided tile sample. tap=0 accumulates gradients (the port's whole
        backward); tap=2 only emits the per-warp WarpRecords (gradient math
        without accumulation, for the reference's reducers to consume)."""
        import time
        L = self.L
        P = st.contents.P
        dL = np.ascontiguousarray(dL_dpixels, np.float32)
        grad = np.zeros(P * NPARAM, np.float64)
        pairs = C.c_int64()
        st.contents.tap_ppt = 2  # records in the GPU reduction kernel's lane layout
        t0 = time.perf_counter()
        if L.gs_backward(st, C.byref(cam), dL.ctypes.data, grad.ctypes.data, None,
                         threads, tile_stride, tap, C.byref(pairs)):
            raise RuntimeError(L.gs_last_error().decode())
        dt = time.perf_counter() - t0
        tr = None
        if tap:
            s = st.contents
            r = s.tap_count
            tr = Trace(scene_spec_for(P, NPARAM), _arr(s.tap_warp, r, np.int32),
                       _arr(s.tap_iter, r, np.int32), _arr(s.tap_active, r, np.uint32),
                       _arr(s.tap_prim, 32 * r, np.int32),
                       _arr(s.tap_grads, 32 * NPARAM * r, np.float64))
        return dt, int(pairs.value), tr


class GsView:
    """One view's oracle state built by gs_forward_lists; verify() runs the
    decision-matched blend + backward (gs_verify.c)."""

    def __init__(self, orc: Oracle, scene, cam: Camera, threads: int, with_keys: bool):
        self.orc, self.cam, self.threads = orc, cam, threads
        L = orc.L
        self.st = L.gs_state_new()
        self.P = int(scene["means3D"].shape[0])
        ins = [np.ascontiguousarray(scene[k], np.float32)
               for k in ("means3D", "scales", "rotations", "opacities", "colors")]
        if L.gs_forward_lists(self.st, self.P, *[a.ctypes.data for a in ins], C.byref(cam),
                              threads, 1 if with_keys else 0):
            msg = L.gs_verify_last_error().decode()
            L.gs_state_free(self.st)
            self.st = None
            raise RuntimeError(msg)
        s = self.st.contents
        self.W, self.H = s.W, s.H
        self.num_rendered = int(s.num_rendered)
        self.with_keys = with_keys

    def __del__(self):
        if getattr(self, "st", None) is not None:
            self.orc.L.gs_state_free(self.st)
            self.st = None

    def lists(self):
        s = self.st.contents
        P, nr, ntiles = self.P, self.num_rendered, s.tiles_x * s.tiles_y
        out = {
            "means2D": _arr(s.means2D, 2 * P, np.float32).reshape(P, 2),
            "depths": _arr(s.depths, P, np.float32),
            "radii": _arr(s.radii, P, np.int32),
            "conic_opacity": _arr(s.conic_opacity, 4 * P, np.float32).reshape(P, 4),
            "tiles_touched": _arr(s.tiles_touched, P, np.uint32),
            "num_rendered": nr,
            "values": _arr(s.values, nr, np.uint32),
            "ranges": _arr(s.ranges, 2 * ntiles, np.uint32).reshape(ntiles, 2),
        }
        if self.with_keys:
            out["keys"] = _arr(s.keys, nr, np.uint64)
        return out

    def verify(self, dL_dpixels=None, gpu=None, kappa=1.0, flip_cap=4096):
        """gpu: None or (n_contrib [H*W] u32, final_T [H*W] f32, image [3,H,W] f32).
        Returns (dict of arrays, report dict, flips list)."""
        P, W, H = self.P, self.W, self.H
        HW = W * H
        o = {
            "grad": np.zeros(P * NPARAM), "grad_bound": np.zeros(P * NPARAM),
            "grad_abs": np.zeros(P * NPARAM), "grad_slack": np.zeros(P * NPARAM),
            "npix": np.zeros(P, np.int32), "image": np.zeros(3 * HW),
            "image_mag": np.zeros(3 * HW), "image_slack": np.zeros(3 * HW), "final_T": np.zeros(HW), "epix": np.zeros(HW),
            "n_contrib": np.zeros(HW, np.uint32), "status": np.zeros(HW, np.uint8),
        }
        flips = (GsFlip * max(flip_cap, 1))()
        out = GsVerifyOut(**{k: v.ctypes.data for k, v in o.items()}, flips=C.addressof(flips),
                          flip_cap=flip_cap, nflip_rec=0)
        rep = GsVerifyReport()
        keep = []
        dl = None
        if dL_dpixels is not None:
            dl = np.ascontiguousarray(dL_dpixels, np.float32)
            keep.append(dl)
        g = [None, None, None]
        if gpu is not None:
            g = [np.ascontiguousarray(gpu[0], np.uint32).reshape(-1),
                 np.ascontiguousarray(gpu[1], np.float32).reshape(-1),
                 np.ascontiguousarray(gpu[2], np.float32).reshape(-1)]
            assert g[0].size == HW and g[1].size == HW and g[2].size == 3 * HW
        L = self.orc.L
        rc = L.gs_verify(self.st, C.byref(self.cam), dl.ctypes.data if dl is not None else None,
                         *[a.ctypes.data if a is not None else None for a in g], float(kappa),
                         C.byref(out), C.byref(rep), self.threads)
        if rc:
            raise RuntimeError(L.gs_verify_last_error().decode())
        o["grad"] = o["grad"].reshape(P, NPARAM)
        for k in ("grad_bound", "grad_abs", "grad_slack"):
            o[k] = o[k].reshape(P, NPARAM)
        o["image"] = o["image"].reshape(3, H, W)
        o["image_mag"] = o["image_mag"].reshape(3, H, W)
        o["image_slack"] = o["image_slack"].reshape(3, H, W)
        for k in ("final_T", "epix", "n_contrib", "status"):
            o[k] = o[k].reshape(H, W)
        fl = [(f.pixel, f.position, f.gaussian, f.kind) for f in flips[:out.nflip_rec]]
        return o, rep.as_dict(), fl


def scene_spec_for(num_prims: int, n: int) -> SceneSpec:
    return scene(num_primitives=num_prims, params_per_primitive=n, quantized_values=0)


class Ref:
    """The reference itself (oracle/_ref/libwarpred_ref.so)."""

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(path)
        L = self.L = C.CDLL(path)
        L.ref_last_error.restype = C.c_char_p
        L.ref_generate.argtypes = [C.POINTER(SceneSpec), C.POINTER(C.c_void_p)]
        L.ref_load_binary.argtypes = [C.c_char_p, C.POINTER(C.c_void_p)]
        L.ref_save_binary.argtypes = [C.c_void_p, C.c_char_p]
        L.ref_from_arrays.argtypes = [C.c_int64, C.c_int32, C.c_int32] + [C.c_void_p] * 5 + [
            C.POINTER(C.c_void_p)]
        L.ref_free.argtypes = [C.c_void_p]
        L.ref_record_count.argtypes = [C.c_void_p]
        L.ref_record_count.restype = C.c_int64
        L.ref_params.argtypes = [C.c_void_p]
        L.ref_params.restype = C.c_int32
        L.ref_num_primitives.argtypes = [C.c_void_p]
        L.ref_num_primitives.restype = C.c_int32
        L.ref_export.argtypes = [C.c_void_p] + [C.c_void_p] * 5
        L.ref_criterion1_draws.argtypes = [C.c_int32, C.c_void_p, C.c_void_p]
        L.ref_read_metrics_csv.argtypes = [C.c_char_p, C.c_int32, C.POINTER(C.c_int64),
                                           C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
        L.ref_oracle_sum.argtypes = [C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p]
        L.ref_apply_policy.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int32, C.c_void_p,
                                       C.c_void_p]
        L.ref_record_policy.argtypes = [C.c_uint32, C.c_void_p, C.c_void_p, C.c_int32, C.c_int,
                                        C.c_int, C.c_void_p, C.c_void_p, C.c_void_p,
                                        C.POINTER(C.c_int64), C.POINTER(C.c_uint64),
                                        C.POINTER(C.c_uint64)]
        L.ref_time_policy.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int32, C.c_int,
                                      C.c_int64, C.POINTER(C.c_double), C.POINTER(C.c_uint64),
                                      C.POINTER(C.c_uint64)]

    def _check(self, rc):
        if rc != 0:
            raise RuntimeError(self.L.ref_last_error().decode())

    def generate(self, spec):
        h = C.c_void_p()
        self._check(self.L.ref_generate(C.byref(spec), C.byref(h)))
        return h

    def load_binary(self, path):
        h = C.c_void_p()
        self._check(self.L.ref_load_binary(path.encode(), C.byref(h)))
        return h

    def from_trace(self, tr: Trace):
        h = C.c_void_p()
        keep = [np.ascontiguousarray(tr.warp_id, np.int32),
                np.ascontiguousarray(tr.iteration, np.int32),
                np.ascontiguousarray(tr.active, np.uint32),
                np.ascontiguousarray(tr.prim, np.int32),
                np.ascontiguousarray(tr.grads, np.float64)]
        self._check(self.L.ref_from_arrays(tr.num_records, tr.n, tr.spec.num_primitives,
                                           *[k.ctypes.data for k in keep], C.byref(h)))
        return h

    def free(self, h):
        self.L.ref_free(h)

    def save_binary(self, h, path):
        self._check(self.L.ref_save_binary(h, path.encode()))

    def to_numpy(self, h, spec=None) -> Trace:
        r = self.L.ref_record_count(h)
        n = self.L.ref_params(h)
        w = np.zeros(r, np.int32)
        it = np.zeros(r, np.int32)
        a = np.zeros(r, np.uint32)
        p = np.zeros(r * 32, np.int32)
        g = np.zeros(r * 32 * n, np.float64)
        self.L.ref_export(h, w.ctypes.data, it.ctypes.data, a.ctypes.data, p.ctypes.data,
                          g.ctypes.data)
        if spec is None:
            spec = scene(params_per_primitive=n,
                         num_primitives=self.L.ref_num_primitives(h))
        return Trace(spec, w, it, a, p, g)

    def oracle_sum(self, h, num_prims):
        n = self.L.ref_params(h)
        sums = np.zeros(num_prims * n, np.float64)
        touched = np.zeros(num_prims * n, np.uint8)
        self._check(self.L.ref_oracle_sum(h, num_prims, sums.ctypes.data, touched.ctypes.data))
        return sums, touched.astype(bool)

    def read_metrics_csv(self, path: str, max_rows: int = 4096):
        """The reference's experiment::read_metrics_csv on a file: list of
        (policy kind, threshold or None, 7 integer RunMetrics, energy_proxy,
        grad_speedup, end_to_end_speedup)."""
        n = C.c_int64()
        pol = np.zeros(max_rows, np.int32)
        thr = np.zeros(max_rows, np.int32)
        ints = np.zeros(7 * max_rows, np.uint64)
        dbl = np.zeros(3 * max_rows, np.float64)
        self._check(self.L.ref_read_metrics_csv(path.encode(), max_rows, C.byref(n),
                                                pol.ctypes.data, thr.ctypes.data,
                                                ints.ctypes.data, dbl.ctypes.data))
        k = min(n.value, max_rows)
        return [(int(pol[i]), None if thr[i] < 0 else int(thr[i]),
                 ints[7 * i:7 * i + 7].tolist(), *dbl[3 * i:3 * i + 3].tolist())
                for i in range(k)]

    def criterion1_draws(self, ntraces: int):
        """The (SceneSpec, thresholds) sequence of the reference's acceptance
        criterion 1 (tests/acceptance.cpp:93-146); thresholds[p] = (sw_s, sw_b)
        of preset p."""
        specs = (SceneSpec * ntraces)()
        thr = np.zeros(ntraces * 6, np.int32)
        self._check(self.L.ref_criterion1_draws(ntraces, C.addressof(specs), thr.ctypes.data))
        out = []
        for i in range(ntraces):
            d = {k: getattr(specs[i], k) for k, _ in SceneSpec._fields_}
            out.append((d, thr[6 * i:6 * i + 6].reshape(3, 2).tolist()))
        return out

    def apply_policy(self, h, kind, threshold, num_prims):
        n = self.L.ref_params(h)
        sums = np.zeros(num_prims * n, np.float64)
        counts = np.zeros(3, np.uint64)
        self._check(self.L.ref_apply_policy(h, kind, threshold, num_prims, sums.ctypes.data,
                                            counts.ctypes.data))
        return sums, {"requests": int(counts[0]), "instructions": int(counts[1]),
                      "fp_adds": int(counts[2])}

    def record_policy(self, active, prim, grads, kind, threshold):
        prim = np.ascontiguousarray(prim, np.int32)
        grads = np.ascontiguousarray(grads, np.float64)
        n = grads.size // 32
        op = np.zeros(32 * n, np.int32)
        oq = np.zeros(32 * n, np.int32)
        ov = np.zeros(32 * n, np.float64)
        cnt, ins, fp = C.c_int64(), C.c_uint64(), C.c_uint64()
        self._check(self.L.ref_record_policy(int(active), prim.ctypes.data, grads.ctypes.data,
                                             n, kind, threshold, op.ctypes.data, oq.ctypes.data,
                                             ov.ctypes.data, C.byref(cnt), C.byref(ins),
                                             C.byref(fp)))
        c = cnt.value
        return (list(zip(op[:c].tolist(), oq[:c].tolist(), ov[:c].tolist())),
                ins.value, fp.value)

    def time_policy(self, h, kind, threshold, num_prims, threads, max_records=0):
        s, c, q = C.c_double(), C.c_uint64(), C.c_uint64()
        self._check(self.L.ref_time_policy(h, kind, threshold, num_prims, threads, max_records,
                                           C.byref(s), C.byref(c), C.byref(q)))
        return s.value, c.value, q.value


def _gs_pb_setup(L):
    L.gs_preprocess_backward.argtypes = [C.POINTER(_GsState), C.c_int32, C.c_void_p, C.c_void_p,
                                         C.c_void_p, C.POINTER(Camera), C.c_void_p, C.c_void_p]
    L.gs_adam.argtypes = [C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_double,
                          C.c_double, C.c_double, C.c_double, C.c_int]


def gs_train_grads(orc: "Oracle", scene, cam: Camera, dL_dpixels, threads=8):
    """CPU oracle of one view's full backward: (grad2d [P,9], grad3d [P,14])."""
    L = orc.L
    _gs_pb_setup(L)
    P = int(scene["means3D"].shape[0])
    ins = [np.ascontiguousarray(scene[k], np.float32)
           for k in ("means3D", "scales", "rotations", "opacities", "colors")]
    st = orc.gs_prepare(scene, cam, threads)
    try:
        dL = np.ascontiguousarray(dL_dpixels, np.float32)
        g2 = np.zeros(P * NPARAM, np.float64)
        pairs = C.c_int64()
        if L.gs_backward(st, C.byref(cam), dL.ctypes.data, g2.ctypes.data, None, threads, 1, 0,
                         C.byref(pairs)):
            raise RuntimeError(L.gs_last_error().decode())
        g3 = np.zeros(P * 14, np.float64)
        if L.gs_preprocess_backward(st, P, ins[0].ctypes.data, ins[1].ctypes.data,
                                    ins[2].ctypes.data, C.byref(cam), g2.ctypes.data,
                                    g3.ctypes.data):
            raise RuntimeError(L.gs_last_error().decode())
        return g2.reshape(P, NPARAM), g3.reshape(P, 14)
    finally:
        orc.gs_free(st)


def gs_adam(orc: "Oracle", param, grad, m, v, lr, beta1, beta2, eps, step):
    """In-place float64 Adam step on contiguous float64 arrays."""
    _gs_pb_setup(orc.L)
    orc.L.gs_adam(param.size, param.ctypes.data, grad.ctypes.data, m.ctypes.data, v.ctypes.data,
                  lr, beta1, beta2, eps, step)
