"""render_forward / render_backward over the C ABI (torch tensors as HBM).

Mirrors the operator shape of a tile-based 3DGS rasterizer: one forward that
projects, bins, sorts and blends a view, and one backward that scatters the
per-pixel gradients into per-Gaussian gradients -- with the scatter done by a
DISTWAR policy (``warpred.Policy``). torch is only the device-memory and
stream plumbing: every tensor crosses the boundary as a raw pointer.

Gradient buffer layout: float32 [P, 9] in Address order (reducers.hpp:19-23),
params (mean2D.x, mean2D.y, conic.x, conic.y, conic.z, opacity, r, g, b).
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib
from ._lib import check, lib
from .warpred import Policy, PolicyKind

NPARAM = 9
NPARAM3D = 14
GRAD_NAMES = ("mean2D.x", "mean2D.y", "conic.x", "conic.y", "conic.z", "opacity", "r", "g", "b")
GRAD3D_NAMES = ("mean.x", "mean.y", "mean.z", "scale.x", "scale.y", "scale.z", "rot.r", "rot.x",
                "rot.y", "rot.z", "opacity", "r", "g", "b")


class Adam:
    """Fused Adam over a scene dict of CUDA tensors (dw_adam_step); moments
    are [P, 14] in the grad3d layout. lr per group: means, scales,
    rotations, opacities, colors."""

    def __init__(self, scene: dict, lr=(1.6e-4, 5e-3, 1e-3, 5e-2, 2.5e-3), betas=(0.9, 0.999),
                 eps=1e-15):
        import torch

        self.scene = scene
        P = int(scene["means3D"].shape[0])
        dev = scene["means3D"].device
        self.exp_avg = torch.zeros((P, NPARAM3D), dtype=torch.float32, device=dev)
        self.exp_avg_sq = torch.zeros((P, NPARAM3D), dtype=torch.float32, device=dev)
        self.cfg = _lib.AdamConfigC((C.c_float * 5)(*lr), betas[0], betas[1], eps)
        self.t = 0

    def step(self, grad3d, stream=None):
        import torch

        self.t += 1
        s = self.scene
        f32 = torch.float32
        P, sp = _scene_ptrs(s["means3D"], s["scales"], s["rotations"], s["opacities"],
                            s["colors"])
        check(lib().dw_adam_step(
            P, *sp, _ptr(grad3d, "grad3d", f32, min_numel=NPARAM3D * P),
            _ptr(self.exp_avg, "exp_avg", f32, NPARAM3D * P),
            _ptr(self.exp_avg_sq, "exp_avg_sq", f32, NPARAM3D * P), C.byref(self.cfg), self.t,
            _stream(stream)))

# dw_rasterizer_buffer ids
BUFFERS = {"means2D": (0, np.float32, 2), "depths": (1, np.float32, 1),
           "radii": (2, np.int32, 1), "conic_opacity": (3, np.float32, 4),
           "tiles_touched": (4, np.uint32, 1), "keys": (5, np.uint64, 1),
           "values": (6, np.uint32, 1), "ranges": (7, np.uint32, 2),
           "final_T": (8, np.float32, 1), "n_contrib": (9, np.uint32, 1)}


def _ptr(t, name, dtype=None, numel=None, min_numel=None):
    """Raw device pointer of a tensor the C side will trust blindly: type,
    device (the current one), contiguity, dtype and element count are
    checked here, so a wrong-shaped buffer raises instead of corrupting HBM."""
    import torch

    if not isinstance(t, torch.Tensor):
        raise TypeError(f"{name} must be a torch.Tensor")
    if not t.is_cuda:
        raise ValueError(f"{name} must be a CUDA tensor")
    if t.device.index != torch.cuda.current_device():
        raise ValueError(f"{name} is on {t.device}, the current device is "
                         f"cuda:{torch.cuda.current_device()}")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")
    if dtype is not None and t.dtype != dtype:
        raise ValueError(f"{name} must be {dtype}")
    if numel is not None and t.numel() != numel:
        raise ValueError(f"{name} must have {numel} elements, has {t.numel()}")
    if min_numel is not None and t.numel() < min_numel:
        raise ValueError(f"{name} must have at least {min_numel} elements, has {t.numel()}")
    return t.data_ptr()


def _scene_ptrs(means3D, scales, rotations, opacities, colors):
    import torch

    f32 = torch.float32
    P = int(means3D.shape[0])
    return P, (_ptr(means3D, "means3D", f32, 3 * P), _ptr(scales, "scales", f32, 3 * P),
               _ptr(rotations, "rotations", f32, 4 * P), _ptr(opacities, "opacities", f32, P),
               _ptr(colors, "colors", f32, 3 * P))


def _stream(stream):
    import torch

    if stream is None:
        return C.c_void_p(torch.cuda.current_stream().cuda_stream)
    if isinstance(stream, int):
        return C.c_void_p(stream)
    return C.c_void_p(stream.cuda_stream)


class GaussianRasterizer:
    """Owns one view's device state (``dw_rasterizer``)."""

    def __init__(self):
        h = C.c_void_p()
        check(lib().dw_rasterizer_create(C.byref(h)))
        self._h = h
        self.P = 0
        self.num_rendered = 0
        self.camera = None

    def __del__(self):
        h = getattr(self, "_h", None)
        if h and h.value and _lib._lib is not None:
            _lib._lib.dw_rasterizer_free(h)
            self._h = None

    @property
    def handle(self):
        return self._h

    def render_forward(self, means3D, scales, rotations, opacities, colors, camera,
                       out_color=None, radii=None, stream=None):
        """Returns (out_color [3,H,W], radii [P], num_rendered)."""
        import torch

        f32 = torch.float32
        P, sp = _scene_ptrs(means3D, scales, rotations, opacities, colors)
        if out_color is None:
            out_color = torch.empty((3, camera.height, camera.width), dtype=f32,
                                    device=means3D.device)
        if radii is None:
            radii = torch.empty((P,), dtype=torch.int32, device=means3D.device)
        nr = C.c_int64()
        cam = camera.to_c()
        check(lib().dw_render_forward(
            self._h, P, *sp, C.byref(cam),
            _ptr(out_color, "out_color", f32, 3 * camera.height * camera.width),
            _ptr(radii, "radii", torch.int32, P), C.byref(nr), _stream(stream)))
        self.P, self.num_rendered, self.camera, self.views = P, nr.value, camera, 1
        return out_color, radii, nr.value

    def render_forward_views(self, means3D, scales, rotations, opacities, colors, cameras,
                             out_images=None, stream=None):
        """dw_render_forward_views: len(cameras) views of one scene stacked into
        one frame (every forward launch covers all of them); the next
        render_backward takes dL_dpixels [V, 3, H, W]. Returns
        (out_images [V, 3, H, W], num_rendered of the frame)."""
        import torch

        f32 = torch.float32
        V = len(cameras)
        if V < 1:
            raise ValueError("need at least one camera")
        H, W = cameras[0].height, cameras[0].width
        P, sp = _scene_ptrs(means3D, scales, rotations, opacities, colors)
        if out_images is None:
            out_images = torch.empty((V, 3, H, W), dtype=f32, device=means3D.device)
        arr = (_lib.CameraC * V)(*[c.to_c() for c in cameras])
        nr = C.c_int64()
        check(lib().dw_render_forward_views(
            self._h, P, *sp, arr, V, _ptr(out_images, "out_images", f32, V * 3 * H * W),
            C.byref(nr), _stream(stream)))
        self.P, self.num_rendered, self.camera, self.views = P, nr.value, cameras[0], V
        return out_images, nr.value

    def reserve(self, P: int, width: int, height: int, max_instances: int):
        """Pre-size every buffer (dw_rasterizer_reserve) so that a forward /
        backward within these sizes allocates nothing -- required before
        render_forward_async and before capturing a CUDA graph."""
        check(lib().dw_rasterizer_reserve(self._h, int(P), int(width), int(height),
                                          int(max_instances)))

    def render_forward_async(self, means3D, scales, rotations, opacities, colors, camera,
                             out_color, radii, stream=None):
        """render_forward with no host synchronisation (graph-capturable): the
        instance count stays on the device; read it with instances()."""
        import torch

        f32 = torch.float32
        P, sp = _scene_ptrs(means3D, scales, rotations, opacities, colors)
        cam = camera.to_c()
        check(lib().dw_render_forward_async(
            self._h, P, *sp, C.byref(cam),
            _ptr(out_color, "out_color", f32, 3 * camera.height * camera.width),
            _ptr(radii, "radii", torch.int32, P), _stream(stream)))
        self.P, self.num_rendered, self.camera, self.views = P, None, camera, 1
        return out_color, radii

    def instances(self):
        """(num_rendered, overflowed) of the last forward; synchronises."""
        n, ovf = C.c_int64(), C.c_int()
        check(lib().dw_rasterizer_num_rendered(self._h, C.byref(n), C.byref(ovf)))
        self.num_rendered = n.value
        return n.value, bool(ovf.value)

    def render_backward(self, dL_dpixels, policy: Policy = Policy(PolicyKind.sw_b, 0),
                        grad=None, count_pairs: bool = False, stream=None,
                        chained: bool = False):
        """Adds into grad [P, 9] (allocated zeroed if None). Returns grad, or
        (grad, pairs) when count_pairs (a separate counting instantiation).
        chained: dw_render_backward_chained -- the previous kernel on the
        stream writes nothing this backward reads (see include/distwar.h)."""
        import torch

        if chained:
            if grad is None or count_pairs:
                raise ValueError("a chained backward adds into a given grad, uncounted")
            check(lib().dw_render_backward_chained(
                self._h, _ptr(dL_dpixels, "dL_dpixels", torch.float32, self._npix3()),
                int(policy.kind), policy.threshold,
                _ptr(grad, "grad", torch.float32, min_numel=NPARAM * self.P), _stream(stream)))
            return grad
        alloc = grad is None
        if alloc:  # >= 1 row: an empty scene still passes a non-null buffer
            grad = torch.zeros((max(self.P, 1), NPARAM), dtype=torch.float32,
                               device=dL_dpixels.device)
        pairs = C.c_uint64()
        check(lib().dw_render_backward(
            self._h, _ptr(dL_dpixels, "dL_dpixels", torch.float32, self._npix3()),
            int(policy.kind), policy.threshold,
            _ptr(grad, "grad", torch.float32, min_numel=NPARAM * self.P),
            C.byref(pairs) if count_pairs else None, _stream(stream)))
        grad = grad[:self.P] if alloc else grad
        return (grad, pairs.value) if count_pairs else grad

    def render_backward_tap(self, dL_dpixels, threshold: int = 0, grad=None,
                            max_records: int = 1 << 22, stream=None):
        """SW-B backward that also returns the per-warp WarpRecords it
        reduced, as a warpred.Trace (save with .save_binary -> WRTRACEB).
        Returns (grad, trace, total_records)."""
        import torch

        from .warpred import Trace

        alloc = grad is None
        if alloc:  # >= 1 row: an empty scene still passes a non-null buffer
            grad = torch.zeros((max(self.P, 1), NPARAM), dtype=torch.float32,
                               device=dL_dpixels.device)
        h, total = C.c_void_p(), C.c_int64()
        check(lib().dw_render_backward_tap(
            self._h, _ptr(dL_dpixels, "dL_dpixels", torch.float32, self._npix3()), threshold,
            _ptr(grad, "grad", torch.float32, min_numel=NPARAM * self.P), max_records,
            C.byref(h), C.byref(total),
            _stream(stream)))
        grad = grad[:self.P] if alloc else grad
        return grad, Trace(h.value), total.value

    def preprocess_backward(self, means3D, scales, rotations, grad2d, grad3d=None, stream=None):
        """Adds this view's 3D gradients (from grad2d [P, 9]) into grad3d
        [P, 14] (means3D xyz, scales xyz, rotation rxyz, opacity, rgb)."""
        import torch

        if grad3d is None:
            grad3d = torch.zeros((self.P, NPARAM3D), dtype=torch.float32, device=grad2d.device)
        f32 = torch.float32
        P = self.P
        check(lib().dw_preprocess_backward(
            self._h, _ptr(means3D, "means3D", f32, 3 * P), _ptr(scales, "scales", f32, 3 * P),
            _ptr(rotations, "rotations", f32, 4 * P),
            _ptr(grad2d, "grad2d", f32, min_numel=NPARAM * P),
            _ptr(grad3d, "grad3d", f32, min_numel=NPARAM3D * P), _stream(stream)))
        return grad3d

    STAGES = ("preprocess", "depth_sort", "offsets", "binning", "ranges", "blend")

    def stage_timing(self, enable: bool = True):
        """Record CUDA events between the stages of later forwards (diagnostic)."""
        check(lib().dw_rasterizer_stage_timing(self._h, 1 if enable else 0))

    def stage_ms(self) -> dict:
        """Per-stage ms of the last stage-timed forward (synchronises)."""
        out = (C.c_double * 6)()
        n = C.c_int32()
        check(lib().dw_rasterizer_stage_ms(self._h, out, C.byref(n)))
        return {self.STAGES[i]: out[i] for i in range(n.value)}

    def _npix3(self) -> int:
        if self.camera is None:
            raise _lib.InvalidArgument(1, "render_backward before render_forward")
        return 3 * self.camera.height * self.camera.width * getattr(self, "views", 1)

    def buffer(self, name: str) -> np.ndarray:
        """Host copy of an intermediate buffer (parity tests)."""
        which, dtype, width = BUFFERS[name]
        p, n = C.c_void_p(), C.c_int64()
        check(lib().dw_rasterizer_buffer(self._h, which, C.byref(p), C.byref(n)))
        out = np.zeros(n.value, dtype)
        check(lib().dw_copy_to_host(out.ctypes.data, p, out.nbytes))
        return out.reshape(-1, width) if width > 1 else out

    def render_host(self, scene: dict, camera, dL_dpixels: np.ndarray,
                    policy: Policy = Policy(PolicyKind.sw_b, 0)):
        """End-to-end from host buffers (``dw_render_host``): returns
        (image [3,H,W], grad [P,9]) as numpy."""
        P = int(scene["means3D"].shape[0])
        arrs = [np.ascontiguousarray(scene[k], np.float32)
                for k in ("means3D", "scales", "rotations", "opacities", "colors")]
        for a, k, w in zip(arrs, ("means3D", "scales", "rotations", "opacities", "colors"),
                           (3, 3, 4, 1, 3)):
            if a.size != w * P:
                raise ValueError(f"{k} must have {w * P} elements, has {a.size}")
        dL = np.ascontiguousarray(dL_dpixels, np.float32)
        if dL.size != 3 * camera.height * camera.width:
            raise ValueError(f"dL_dpixels must have {3 * camera.height * camera.width} elements")
        img = np.zeros((3, camera.height, camera.width), np.float32)
        grad = np.zeros((P, NPARAM), np.float32)
        cam = camera.to_c()
        check(lib().dw_render_host(self._h, P, *[a.ctypes.data for a in arrs], C.byref(cam),
                                   dL.ctypes.data, int(policy.kind), policy.threshold,
                                   img.ctypes.data, grad.ctypes.data, None))
        return img, grad


class ThresholdTuner:
    """Online balancing-threshold selection for a training loop (SURVEY
    §8(f4), tuner.hpp:15): on the first iteration and then
    every `period` iterations, time one backward per threshold 0..32 on the
    current view and keep the argmin, ties to the lowest t (tuner.cpp:46-49).
    `timer(threshold) -> ms` may be injected; the default times
    render_backward on a scratch gradient with CUDA events."""

    def __init__(self, period: int = 2000, kind: PolicyKind = PolicyKind.sw_b, reps: int = 1,
                 timer=None):
        if period < 1:
            raise ValueError("period must be >= 1")
        if kind not in (PolicyKind.sw_s, PolicyKind.sw_b):
            raise ValueError("only sw_s / sw_b take a threshold")
        self.period, self.kind, self.reps, self.timer = period, kind, reps, timer
        self.iteration = 0
        self.chosen = None
        self.history = []  # (iteration, chosen, {t: ms})

    def _cuda_timer(self, rast, dL):
        import torch

        scratch = torch.zeros((rast.P, NPARAM), dtype=torch.float32, device=dL.device)

        def time_t(t):
            best = None
            for _ in range(self.reps):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                rast.render_backward(dL, Policy(self.kind, t), grad=scratch)
                e1.record()
                e1.synchronize()
                ms = e0.elapsed_time(e1)
                best = ms if best is None else min(best, ms)
            return best

        return time_t

    def policy(self, rast=None, dL=None) -> Policy:
        """The policy for this iteration (re-tunes when due); call once per
        iteration after render_forward of the view about to be back-propagated."""
        if self.chosen is None or self.iteration % self.period == 0:
            timer = self.timer or self._cuda_timer(rast, dL)
            sweep = {t: timer(t) for t in range(33)}
            best = 0
            for t in range(1, 33):
                if sweep[t] < sweep[best]:
                    best = t
            self.chosen = best
            self.history.append((self.iteration, best, sweep))
        self.iteration += 1
        return Policy(self.kind, self.chosen)


def render_backward_views(rasts, dLs, policy: Policy, grad, stream=None):
    """dw_render_backward_views: the backwards of rendered views of one scene
    (rasts[k] with dLs[k]) added into grad [P, 9] as one chain."""
    import torch

    n = len(rasts)
    if n < 1 or len(dLs) != n:
        raise ValueError("one dL/dpixel per rasterizer, at least one")
    P = rasts[0].P
    hs = (C.c_void_p * n)(*[r.handle for r in rasts])
    ds = (C.c_void_p * n)(*[_ptr(d, "dL_dpixels", torch.float32, r._npix3())
                            for r, d in zip(rasts, dLs)])
    check(lib().dw_render_backward_views(hs, ds, n, int(policy.kind), policy.threshold,
                                         _ptr(grad, "grad", torch.float32, min_numel=NPARAM * P),
                                         _stream(stream)))
    return grad


def max_stacked_views(width: int, height: int) -> int:
    """dw_rasterizer_max_stacked_views: views of this size one stacked frame holds."""
    out = C.c_int32()
    check(lib().dw_rasterizer_max_stacked_views(int(width), int(height), C.byref(out)))
    return out.value


def render_views_host(rast: "GaussianRasterizer", scene_ptrs, P: int, cams, dL_ptr: int,
                      policy: Policy, images_ptr, grad_ptr: int, stream=None) -> None:
    """dw_render_views_host over raw host pointers (pinned for overlap):
    scene_ptrs = (means3D, scales, rotations, opacities, colors)."""
    arr = (_lib.CameraC * len(cams))(*[c.to_c() for c in cams])
    check(lib().dw_render_views_host(rast.handle, P, *scene_ptrs, arr, len(cams), dL_ptr,
                                     int(policy.kind), policy.threshold, images_ptr, grad_ptr,
                                     None if stream is None else _stream(stream)))


def render_views(rast: "GaussianRasterizer", scene_ptrs, P: int, cams, dL_ptr: int,
                 policy: Policy, images_ptr, grad, stream=None):
    """dw_render_views: render_views_host with the gradient left on the
    device in `grad` (a CUDA tensor of P*9 fp32, overwritten) -- the multi-GPU
    path all-reduces it over NCCL before one device-to-host copy."""
    import torch

    arr = (_lib.CameraC * len(cams))(*[c.to_c() for c in cams])
    check(lib().dw_render_views(rast.handle, P, *scene_ptrs, arr, len(cams), dL_ptr,
                                int(policy.kind), policy.threshold, images_ptr,
                                _ptr(grad, "grad", torch.float32, NPARAM * P),
                                None if stream is None else _stream(stream)))
    return grad


def nccl_comm_ptr(group=None) -> int:
    """The ncclComm_t of a torch.distributed NCCL process group (default: the
    world), for the C ABI's communicator-aware calls. The communicator is
    created lazily by torch: one barrier makes sure it exists."""
    import torch
    import torch.distributed as dist

    group = group if group is not None else dist.group.WORLD
    dist.barrier(group=group, device_ids=[torch.cuda.current_device()])
    backend = group._get_backend(torch.device("cuda"))
    return int(backend._comm_ptr())


def allreduce_grads(grad, comm: int, stream=None):
    """dw_allreduce_grads: sum a CUDA fp32 gradient tensor in place across the
    ranks of an NCCL communicator (nccl_comm_ptr) on `stream`."""
    import torch

    check(lib().dw_allreduce_grads(C.c_void_p(comm), _ptr(grad, "grad", torch.float32),
                                   grad.numel(), _stream(stream)))
    return grad


def render_views_allreduce(rast: "GaussianRasterizer", scene_ptrs, P: int, cams, dL_ptr: int,
                           policy: Policy, images_ptr, grad_ptr: int, comm: int, stream=None):
    """dw_render_views_allreduce: one rank's whole view-parallel step through
    the C ABI from host buffers -- its views forward + backward into a device
    gradient, the NCCL all-reduce across `comm`, one D2H into grad_ptr (host,
    P*9 fp32)."""
    arr = (_lib.CameraC * len(cams))(*[c.to_c() for c in cams])
    check(lib().dw_render_views_allreduce(rast.handle, P, *scene_ptrs, arr, len(cams), dL_ptr,
                                          int(policy.kind), policy.threshold, images_ptr, None,
                                          grad_ptr, C.c_void_p(comm),
                                          None if stream is None else _stream(stream)))


def microbench_red(pattern: int, ops: int = 1 << 28, stream=None) -> float:
    """Measured REDs/s: 0 distinct, 1 same-address warp, 2 v4, 3 DISTWAR 9-lane."""
    out = C.c_double()
    check(lib().dw_microbench_red(pattern, ops, C.byref(out),
                                  None if stream is None else _stream(stream)))
    return out.value
