"""ctypes binding of ``libdistwar.so`` (the C ABI declared in include/distwar.h).

There is no fallback: if the shared library is missing or a call fails, an
exception is raised. The library is built in-tree by ``__graft_entry__.build()``
(``make -C paper_2401_05345_b200/csrc``).
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
# DISTWAR_LIB selects an alternative in-tree build (A/B experiments); default
# is the one __graft_entry__.build() produces.
LIB_PATH = os.environ.get("DISTWAR_LIB") or os.path.join(HERE, "csrc", "libdistwar.so")

DW_OK, DW_ERR_INVALID_ARGUMENT, DW_ERR_IO, DW_ERR_RUNTIME = 0, 1, 2, 3


class DistwarError(RuntimeError):
    """A non-OK dw_status; ``code`` is the status, the message dw_last_error()."""

    def __init__(self, code: int, message: str):
        super().__init__(message)
        self.code = code


class InvalidArgument(DistwarError, ValueError):
    pass


class IOFailure(DistwarError, OSError):
    pass


class SceneSpecC(C.Structure):
    """dw_scene_spec == wr_scene_spec (reference include/warpred.h:42-53)."""

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


class GpuMetricsC(C.Structure):
    _fields_ = [
        ("kernel_ms", C.c_double),
        ("atomic_requests_to_l2", C.c_uint64),
        ("contributions", C.c_uint64),
        ("records", C.c_uint64),
    ]


class TuneReportC(C.Structure):
    _fields_ = [
        ("us_by_threshold", C.c_double * 33),
        ("chosen", C.c_int32),
        ("profile_iteration", C.c_int32),
        ("reprofile_period", C.c_int32),
    ]


class CameraC(C.Structure):
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


class AdamConfigC(C.Structure):
    _fields_ = [("lr", C.c_float * 5), ("beta1", C.c_float), ("beta2", C.c_float),
                ("eps", C.c_float)]


vp = C.c_void_p
i32, i64, u64 = C.c_int32, C.c_int64, C.c_uint64

# name -> (restype, argtypes); every symbol include/distwar.h declares
SIGNATURES = {
    "dw_version": (C.c_char_p, []),
    "dw_last_error": (C.c_char_p, []),
    "dw_device_count": (C.c_int, []),
    "dw_device_clock_khz": (C.c_int, []),
    "dw_scene_spec_init": (None, [C.POINTER(SceneSpecC)]),
    "dw_trace_generate": (C.c_int, [C.POINTER(SceneSpecC), C.POINTER(vp)]),
    "dw_trace_free": (None, [vp]),
    "dw_trace_record_count": (i64, [vp]),
    "dw_trace_save": (C.c_int, [vp, C.c_char_p, C.c_int]),
    "dw_trace_load": (C.c_int, [C.c_char_p, C.c_int, C.POINTER(vp)]),
    "dw_trace_histogram_distinct": (C.c_int, [vp, vp]),
    "dw_trace_histogram_active": (C.c_int, [vp, vp]),
    "dw_trace_from_arrays": (C.c_int, [i64, i32, i32, vp, vp, vp, vp, vp, C.POINTER(vp)]),
    "dw_trace_arrays": (C.c_int, [vp, C.POINTER(vp), C.POINTER(vp), C.POINTER(vp),
                                  C.POINTER(SceneSpecC)]),
    "dw_trace_ids": (C.c_int, [vp, C.POINTER(vp), C.POINTER(vp)]),
    "dw_trace_set_scene": (C.c_int, [vp, C.POINTER(SceneSpecC)]),
    "dw_trace_upload": (C.c_int, [vp, vp, C.POINTER(vp)]),
    "dw_device_trace_free": (None, [vp]),
    "dw_device_trace_view": (C.c_int, [vp, C.POINTER(vp), C.POINTER(vp), C.POINTER(vp),
                                       C.POINTER(i64), C.POINTER(i32), C.POINTER(i32)]),
    "dw_reduce_records": (C.c_int, [vp, vp, vp, i64, i32, i32, C.c_int, i32, vp, vp, vp]),
    "dw_gpu_run": (C.c_int, [vp, C.c_int, i32, vp, C.POINTER(GpuMetricsC)]),
    "dw_model_costs": (C.c_int, [vp, C.c_int, i32, vp]),
    "dw_tune": (C.c_int, [vp, C.c_int, i32, i32, C.POINTER(TuneReportC)]),
    "dw_tune_report_save_csv": (C.c_int, [C.POINTER(TuneReportC), C.c_char_p]),
    "dw_rasterizer_create": (C.c_int, [C.POINTER(vp)]),
    "dw_rasterizer_free": (None, [vp]),
    "dw_render_forward": (C.c_int, [vp, i32, vp, vp, vp, vp, vp, C.POINTER(CameraC), vp, vp,
                                    C.POINTER(i64), vp]),
    "dw_render_backward": (C.c_int, [vp, vp, C.c_int, i32, vp, C.POINTER(u64), vp]),
    "dw_render_backward_chained": (C.c_int, [vp, vp, C.c_int, i32, vp, vp]),
    "dw_render_backward_views": (C.c_int, [vp, vp, i32, C.c_int, i32, vp, vp]),
    "dw_render_forward_async": (C.c_int, [vp, i32, vp, vp, vp, vp, vp, C.POINTER(CameraC), vp, vp,
                                          vp]),
    "dw_render_forward_views": (C.c_int, [vp, i32, vp, vp, vp, vp, vp, C.POINTER(CameraC), i32,
                                          vp, C.POINTER(i64), vp]),
    "dw_rasterizer_max_stacked_views": (C.c_int, [i32, i32, C.POINTER(i32)]),
    "dw_rasterizer_reserve": (C.c_int, [vp, i32, i32, i32, i64]),
    "dw_rasterizer_num_rendered": (C.c_int, [vp, C.POINTER(i64), C.POINTER(C.c_int)]),
    "dw_rasterizer_last_reds": (C.c_int, [vp, C.POINTER(u64)]),
    "dw_rasterizer_stage_timing": (C.c_int, [vp, i32]),
    "dw_rasterizer_stage_ms": (C.c_int, [vp, vp, C.POINTER(i32)]),
    "dw_preprocess_backward": (C.c_int, [vp, vp, vp, vp, vp, vp, vp]),
    "dw_render_backward_tap": (C.c_int, [vp, vp, i32, vp, i64, C.POINTER(vp), C.POINTER(i64),
                                         vp]),
    "dw_adam_step": (C.c_int, [i32, vp, vp, vp, vp, vp, vp, vp, vp, C.c_void_p, i32, vp]),
    "dw_rasterizer_buffer": (C.c_int, [vp, i32, C.POINTER(vp), C.POINTER(i64)]),
    "dw_render_host": (C.c_int, [vp, i32, vp, vp, vp, vp, vp, C.POINTER(CameraC), vp, C.c_int,
                                 i32, vp, vp, vp]),
    "dw_render_views_host": (C.c_int, [vp, i32, vp, vp, vp, vp, vp, vp, i32, vp, C.c_int, i32,
                                       vp, vp, vp]),
    "dw_render_views": (C.c_int, [vp, i32, vp, vp, vp, vp, vp, vp, i32, vp, C.c_int, i32,
                                  vp, vp, vp]),
    "dw_allreduce_grads": (C.c_int, [vp, vp, i64, vp]),
    "dw_render_views_allreduce": (C.c_int, [vp, i32, vp, vp, vp, vp, vp, vp, i32, vp, C.c_int,
                                            i32, vp, vp, vp, vp, vp]),
    "dw_copy_to_host": (C.c_int, [vp, vp, C.c_size_t]),
    "dw_microbench_red": (C.c_int, [i32, i64, C.POINTER(C.c_double), vp]),
}

_lib = None


def lib() -> C.CDLL:
    """Load libdistwar.so once; raise if it is absent (no fallback path)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(
                f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; "
                f"g.build()'` (or `make -C paper_2401_05345_b200/csrc`)")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def check(status: int) -> None:
    if status == DW_OK:
        return
    msg = lib().dw_last_error().decode()
    if status == DW_ERR_INVALID_ARGUMENT:
        raise InvalidArgument(status, msg)
    if status == DW_ERR_IO:
        raise IOFailure(status, msg)
    raise DistwarError(status, msg)
