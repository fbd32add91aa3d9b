"""Host-side mirror of the reference's reduction-stage interface, over the C ABI.

Reference names are kept so code written against warpred reads the same:

* ``SceneSpec`` / ``generate``          workload.hpp:16-36, workload.cpp:99-153
* ``PolicyKind`` / ``Policy``           reducers.hpp:94-104 (same enum values)
* ``Trace.save_binary/load_binary``     trace_io.hpp:382-386 (WRTRACEB)
* ``histogram_distinct_primitives`` /
  ``histogram_active_lanes``           workload.hpp:88-94
* ``apply_policy`` (whole trace, GPU)   reducers.cpp:222-237 + the summation
                                        idiom of test_reducers.cpp:304-308
* ``simulate`` -> ``gpu_run``           hwsim::simulate replaced by the real B200
* ``tune``                              tuner.cpp:29-52 on measured time

Errors keep the reference's mapping: invalid arguments raise ``ValueError``
(``InvalidArgument``), I/O ``OSError``, everything else ``RuntimeError``.
"""
from __future__ import annotations

import ctypes as C
import enum
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from ._lib import check, lib

MIN_BALANCE_THRESHOLD = 0   # reducers.hpp:65
MAX_BALANCE_THRESHOLD = 33  # reducers.hpp:66
DEFAULT_REPROFILE_PERIOD = 2000  # tuner.hpp:15


class PolicyKind(enum.IntEnum):
    native = 0
    sw_s = 1
    sw_b = 2
    cccl = 3
    hw_atomred = 4


class PolicyFamily(enum.IntEnum):
    sw_s = 0
    sw_b = 1


def policy_uses_threshold(kind: PolicyKind) -> bool:  # reducers.cpp:239-241
    return kind in (PolicyKind.sw_s, PolicyKind.sw_b)


def policy_kind_name(kind: PolicyKind) -> str:  # reducers.cpp:243-252
    return PolicyKind(kind).name


def parse_policy_kind(name: str) -> PolicyKind:  # reducers.cpp:254-261
    try:
        return PolicyKind[name]
    except KeyError:
        raise ValueError(f"unknown policy: {name}") from None


@dataclass
class Policy:
    kind: PolicyKind = PolicyKind.native
    threshold: int = 0


@dataclass
class SceneSpec:
    """workload::SceneSpec with the reference defaults (workload.hpp:16-36)."""

    num_primitives: int = 1024
    params_per_primitive: int = 3
    image_width: int = 64
    image_height: int = 32
    mean_fragment_span: float = 64.0
    fragments_per_pixel_mean: float = 1.0
    activity_prob: float = 1.0
    locality: float = 1.0
    seed: int = 0
    quantized_values: bool = True

    def to_c(self) -> _lib.SceneSpecC:
        return _lib.SceneSpecC(self.num_primitives, self.params_per_primitive, self.image_width,
                               self.image_height, self.mean_fragment_span,
                               self.fragments_per_pixel_mean, self.activity_prob, self.locality,
                               self.seed, 1 if self.quantized_values else 0)

    @classmethod
    def from_c(cls, s: _lib.SceneSpecC) -> "SceneSpec":
        return cls(s.num_primitives, s.params_per_primitive, s.image_width, s.image_height,
                   s.mean_fragment_span, s.fragments_per_pixel_mean, s.activity_prob, s.locality,
                   s.seed, bool(s.quantized_values))


class Trace:
    """Host WarpRecord trace owned by libdistwar (``dw_trace``)."""

    def __init__(self, handle: int):
        if not handle:
            raise ValueError("null trace handle")
        self._h = C.c_void_p(handle)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h and h.value and _lib._lib is not None:
            _lib._lib.dw_trace_free(h)
            self._h = None

    @property
    def handle(self):
        return self._h

    def record_count(self) -> int:
        return int(lib().dw_trace_record_count(self._h))

    __len__ = record_count

    def scene(self) -> SceneSpec:
        s = _lib.SceneSpecC()
        check(lib().dw_trace_arrays(self._h, None, None, None, C.byref(s)))
        return SceneSpec.from_c(s)

    def arrays(self):
        """(active u32[R], prim i32[R,32], grads f64[R,32,N]) copies."""
        a, p, g = C.c_void_p(), C.c_void_p(), C.c_void_p()
        s = _lib.SceneSpecC()
        check(lib().dw_trace_arrays(self._h, C.byref(a), C.byref(p), C.byref(g), C.byref(s)))
        r, n = self.record_count(), s.params_per_primitive

        def view(ptr, ctype, count, dtype):
            if count == 0:
                return np.zeros(0, dtype)
            return np.ctypeslib.as_array(C.cast(ptr, C.POINTER(ctype)), (count,)).astype(dtype)

        return (view(a, C.c_uint32, r, np.uint32),
                view(p, C.c_int32, r * 32, np.int32).reshape(r, 32),
                view(g, C.c_double, r * 32 * n, np.float64).reshape(r, 32, n))

    def contributions(self) -> int:
        a, _, _ = self.arrays()
        return int(np.unpackbits(a.view(np.uint8)).sum()) * self.scene().params_per_primitive

    def save_binary(self, path: str) -> None:
        check(lib().dw_trace_save(self._h, path.encode(), 1))

    @classmethod
    def load_binary(cls, path: str) -> "Trace":
        h = C.c_void_p()
        check(lib().dw_trace_load(path.encode(), 1, C.byref(h)))
        return cls(h.value)

    @classmethod
    def from_arrays(cls, active, prim, grads, num_primitives: int, warp_id=None,
                    iteration=None) -> "Trace":
        active = np.ascontiguousarray(active, np.uint32)
        prim = np.ascontiguousarray(prim, np.int32)
        grads = np.ascontiguousarray(grads, np.float64)
        r = active.shape[0]
        n = grads.size // max(r * 32, 1) if r else int(grads.shape[-1])
        w = None if warp_id is None else np.ascontiguousarray(warp_id, np.int32)
        it = None if iteration is None else np.ascontiguousarray(iteration, np.int32)
        h = C.c_void_p()
        check(lib().dw_trace_from_arrays(r, n, num_primitives,
                                         None if w is None else w.ctypes.data,
                                         None if it is None else it.ctypes.data,
                                         active.ctypes.data, prim.ctypes.data, grads.ctypes.data,
                                         C.byref(h)))
        return cls(h.value)


def generate(scene: SceneSpec) -> Trace:
    h = C.c_void_p()
    check(lib().dw_trace_generate(C.byref(scene.to_c()), C.byref(h)))
    return Trace(h.value)


def histogram_distinct_primitives(trace: Trace) -> dict:
    out = np.zeros(33, np.uint64)
    check(lib().dw_trace_histogram_distinct(trace.handle, out.ctypes.data))
    return {k: int(v) for k, v in enumerate(out) if v}


def histogram_active_lanes(trace: Trace) -> dict:
    out = np.zeros(33, np.uint64)
    check(lib().dw_trace_histogram_active(trace.handle, out.ctypes.data))
    return {k: int(v) for k, v in enumerate(out) if v}


class DeviceTrace:
    """SoA fp32 copy of a trace in HBM (``dw_device_trace``)."""

    def __init__(self, trace: Trace, stream: int = 0):
        h = C.c_void_p()
        check(lib().dw_trace_upload(trace.handle, C.c_void_p(stream), C.byref(h)))
        self._h = h
        a, p, v = C.c_void_p(), C.c_void_p(), C.c_void_p()
        r, n, P = C.c_int64(), C.c_int32(), C.c_int32()
        check(lib().dw_device_trace_view(h, C.byref(a), C.byref(p), C.byref(v), C.byref(r),
                                         C.byref(n), C.byref(P)))
        self.d_active, self.d_prim, self.d_vals = a.value, p.value, v.value
        self.records, self.params, self.num_primitives = r.value, n.value, P.value

    def __del__(self):
        h = getattr(self, "_h", None)
        if h and h.value and _lib._lib is not None:
            _lib._lib.dw_device_trace_free(h)
            self._h = None

    @property
    def handle(self):
        return self._h


def reduce_records(d_active: int, d_prim: int, d_vals: int, num_records: int, params: int,
                   num_primitives: int, policy: Policy, d_grad: int, d_red_count: int = 0,
                   stream: int = 0) -> None:
    """The hot path over raw device pointers (``dw_reduce_records``)."""
    check(lib().dw_reduce_records(d_active, d_prim, d_vals, num_records, params, num_primitives,
                                  int(policy.kind), policy.threshold, d_grad,
                                  d_red_count or None, C.c_void_p(stream)))


@dataclass
class GpuMetrics:
    kernel_ms: float
    atomic_requests_to_l2: int
    contributions: int
    records: int


def gpu_run(dtrace: DeviceTrace, policy: Policy, want_sums: bool = True):
    """Replacement of hwsim::simulate: run `policy` on the B200 and return
    (sums f32[P*N] or None, GpuMetrics)."""
    m = _lib.GpuMetricsC()
    out = np.zeros(dtrace.num_primitives * dtrace.params, np.float32) if want_sums else None
    check(lib().dw_gpu_run(dtrace.handle, int(policy.kind), policy.threshold,
                           None if out is None else out.ctypes.data, C.byref(m)))
    return out, GpuMetrics(m.kernel_ms, m.atomic_requests_to_l2, m.contributions, m.records)


@dataclass
class TuneReport:
    us_by_threshold: dict = field(default_factory=dict)
    chosen: int = 0
    profile_iteration: int = 0
    reprofile_period: int = DEFAULT_REPROFILE_PERIOD


def tune(trace: Trace, family: PolicyFamily, iteration: int = -1, reps: int = 5) -> TuneReport:
    """tuner::tune (tuner.cpp:29-52) on measured kernel time."""
    r = _lib.TuneReportC()
    check(lib().dw_tune(trace.handle, int(family), iteration, reps, C.byref(r)))
    return TuneReport({t: r.us_by_threshold[t] for t in range(33)}, r.chosen,
                      r.profile_iteration, r.reprofile_period)
