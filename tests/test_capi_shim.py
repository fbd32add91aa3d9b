"""libwarpred_gpu.so: the reference's C interface (warpred.h) served by the
B200 -- the drop-in under the reference's own symbol names.

* CPU: it exports exactly the reference library's wr_* symbols; trace files
  it writes (binary WRTRACEB and the text format) and the histogram CSVs are
  byte-identical to the reference's for the same scene; text traces written
  by the reference load back record for record.
* GPU: tests/c/capi_sequence.c -- the reference's test_capi.cpp call
  sequence in C -- passes against the shim, compiled against this repo's
  header AND against the reference's own warpred.h (ABI check), and its
  wr_simulate sweep equals the reference build's field for field on the
  counts (atomic_requests_to_l2, core_instructions, core_fp_adds).
"""
import ctypes as C
import json
import os
import re
import subprocess
import sys

import numpy as np
import pytest

from conftest import REF_AVAILABLE, ROOT

SHIM = os.path.join(ROOT, "paper_2401_05345_b200", "csrc", "libwarpred_gpu.so")
REF_LIB = os.path.join(ROOT, "oracle", "_ref", "libwarpred_ref.so")
SEQ_GPU = os.path.join(ROOT, "tests", "c", "build", "capi_sequence_gpu")
SEQ_REF = os.path.join(ROOT, "oracle", "_ref", "capi_sequence_ref")
SEQ_GPU_REFHDR = os.path.join(ROOT, "oracle", "_ref", "capi_sequence_gpu_refheader")


class Scene(C.Structure):
    _fields_ = [("num_primitives", C.c_int32), ("params_per_primitive", C.c_int32),
                ("image_width", C.c_int32), ("image_height", C.c_int32),
                ("mean_fragment_span", C.c_double), ("fragments_per_pixel_mean", C.c_double),
                ("activity_prob", C.c_double), ("locality", C.c_double), ("seed", C.c_uint64),
                ("quantized_values", C.c_int32)]


def _load(path):
    L = C.CDLL(path)
    L.wr_last_error.restype = C.c_char_p
    L.wr_trace_generate.argtypes = [C.POINTER(Scene), C.POINTER(C.c_void_p)]
    L.wr_trace_save.argtypes = [C.c_void_p, C.c_char_p, C.c_int]
    L.wr_trace_load.argtypes = [C.c_char_p, C.c_int, C.POINTER(C.c_void_p)]
    L.wr_trace_free.argtypes = [C.c_void_p]
    L.wr_trace_record_count.argtypes = [C.c_void_p]
    L.wr_trace_record_count.restype = C.c_int64
    L.wr_trace_write_histograms.argtypes = [C.c_void_p, C.c_char_p]
    L.wr_scene_spec_init.argtypes = [C.POINTER(Scene)]
    return L


_WRITER = r"""
import ctypes as C, json, sys
lib, out, kw = sys.argv[1], sys.argv[2], json.loads(sys.argv[3])
class Scene(C.Structure):
    _fields_ = [("num_primitives", C.c_int32), ("params_per_primitive", C.c_int32),
                ("image_width", C.c_int32), ("image_height", C.c_int32),
                ("mean_fragment_span", C.c_double), ("fragments_per_pixel_mean", C.c_double),
                ("activity_prob", C.c_double), ("locality", C.c_double), ("seed", C.c_uint64),
                ("quantized_values", C.c_int32)]
L = C.CDLL(lib)
L.wr_trace_save.argtypes = [C.c_void_p, C.c_char_p, C.c_int]
L.wr_trace_write_histograms.argtypes = [C.c_void_p, C.c_char_p]
h = C.c_void_p()
if len(sys.argv) > 4:  # load a text trace instead of generating
    assert L.wr_trace_load(sys.argv[4].encode(), 0, C.byref(h)) == 0
    assert L.wr_trace_save(h, (out + "/t.csv").encode(), 0) == 0
    sys.exit(0)
s = Scene()
L.wr_scene_spec_init(C.byref(s))
for k, v in kw.items():
    setattr(s, k, v)
assert L.wr_trace_generate(C.byref(s), C.byref(h)) == 0
assert L.wr_trace_save(h, (out + "/t.csv").encode(), 0) == 0
assert L.wr_trace_save(h, (out + "/t.bin").encode(), 1) == 0
assert L.wr_trace_write_histograms(h, (out + "/hist").encode()) == 0
"""


def _scene(L, **kw):
    s = Scene()
    L.wr_scene_spec_init(C.byref(s))
    for k, v in kw.items():
        setattr(s, k, v)
    return s


def _exports(path):
    out = subprocess.run(["nm", "-D", "--defined-only", path], capture_output=True, text=True,
                         check=True).stdout
    return sorted({line.split()[-1] for line in out.splitlines()
                   if line.split()[-1].startswith("wr_")})


def test_shim_exports_the_header():
    declared = sorted(set(re.findall(r"\b(wr_\w+)\(", open(
        os.path.join(ROOT, "include", "warpred_gpu.h")).read())))
    assert _exports(SHIM) == declared
    assert len(declared) == 19


@pytest.mark.ref
def test_shim_exports_the_reference_symbols():
    if not REF_AVAILABLE:
        pytest.skip("oracle/_ref not built")
    assert _exports(SHIM) == _exports(REF_LIB)


SCENES = [dict(num_primitives=128, params_per_primitive=2, image_width=32, image_height=16,
               locality=0.9, activity_prob=0.8, seed=99),
          dict(num_primitives=700, params_per_primitive=9, image_width=64, image_height=48,
               mean_fragment_span=24.0, fragments_per_pixel_mean=2.5, locality=0.7,
               activity_prob=0.6, quantized_values=0, seed=31)]


@pytest.mark.ref
@pytest.mark.parametrize("kw", SCENES)
def test_files_byte_identical_to_reference(tmp_path, kw):
    if not REF_AVAILABLE:
        pytest.skip("oracle/_ref not built")
    files = {}
    for tag, path in (("gpu", SHIM), ("ref", REF_LIB)):
        # a bare interpreter per library (only ctypes loaded): the reference
        # library is C++ built by the system g++, kept apart from this
        # process's extension modules
        d = tmp_path / tag
        d.mkdir()
        subprocess.run([sys.executable, "-c", _WRITER, path, str(d), json.dumps(kw)], check=True,
                       timeout=300)
        files[tag] = {p: (d / p).read_bytes() for p in
                      ("t.csv", "t.bin", "hist/histogram_distinct.csv",
                       "hist/histogram_active.csv")}
    for p in files["ref"]:
        assert files["gpu"][p] == files["ref"][p], p
    # the reference's text trace loads into the shim and saves back identically
    subprocess.run([sys.executable, "-c", _WRITER, SHIM, str(tmp_path), json.dumps(kw),
                    str(tmp_path / "ref" / "t.csv")], check=True, timeout=300)
    assert (tmp_path / "t.csv").read_bytes() == files["ref"]["t.csv"]


def test_shim_error_conventions():
    L = _load(SHIM)
    h = C.c_void_p()
    assert L.wr_trace_generate(None, None) == 1
    assert L.wr_last_error() == b"null argument"
    assert L.wr_trace_record_count(None) == -1
    bad = _scene(L, activity_prob=7.0)
    assert L.wr_trace_generate(C.byref(bad), C.byref(h)) == 1
    assert b"activity_prob" in L.wr_last_error()
    assert L.wr_trace_load(b"/no/such/file.csv", 0, C.byref(h)) != 0
    L.wr_experiment_run.argtypes = [C.c_char_p, C.c_char_p, C.c_int64, C.c_int]
    assert L.wr_experiment_run(b"/x.json", None, -1, 0) == 3
    assert b"not part of the GPU backend" in L.wr_last_error()


def _run(exe, tmp_path, tag):
    d = tmp_path / tag
    d.mkdir()
    p = subprocess.run([exe, str(d)], capture_output=True, text=True, timeout=600)
    assert p.returncode == 0, (exe, p.stderr[-2000:])
    return json.loads(p.stdout)


@pytest.mark.gpu
def test_reference_call_sequence_on_the_gpu(cuda, tmp_path):
    """The reference's test_capi sequence passes on the B200 backend; built
    against the reference's header too when that binary was built here."""
    got = _run(SEQ_GPU, tmp_path, "gpu")
    assert got["failed"] == 0 and got["total_checks"] > 80
    if os.path.exists(SEQ_GPU_REFHDR):
        got2 = _run(SEQ_GPU_REFHDR, tmp_path, "gpu_refhdr")
        assert got2["failed"] == 0
        for k, v in got["runs"].items():
            assert {f: v[f] for f in ("requests", "instructions", "fp_adds")} == \
                   {f: got2["runs"][k][f] for f in ("requests", "instructions", "fp_adds")}
    if os.path.exists(SEQ_REF):
        ref = _run(SEQ_REF, tmp_path, "ref")
        assert ref["failed"] == 0
        assert set(ref["runs"]) == set(got["runs"])
        for k, v in ref["runs"].items():
            g = got["runs"][k]
            assert (g["requests"], g["instructions"], g["fp_adds"]) == \
                   (v["requests"], v["instructions"], v["fp_adds"]), k
            assert g["cycles"] > 0


@pytest.mark.gpu
def test_model_costs_match_reference_policy_counts(cuda, orc):
    """dw_model_costs (the reference's cost model on the device) == the
    reference policy restatement's instruction / fp-add counts, on the
    reference-written golden traces and every threshold."""
    from conftest import GOLDEN
    from paper_2401_05345_b200 import _lib
    from paper_2401_05345_b200 import warpred as wr

    g = json.load(open(os.path.join(GOLDEN, "golden.json")))["small"]
    lib = _lib.lib()
    for name, rec in g.items():
        tr = wr.Trace.load_binary(os.path.join(GOLDEN, rec["file"]))
        d = wr.DeviceTrace(tr)
        for key, c in rec["policies"].items():
            k, t = key.split(":")
            out = (C.c_uint64 * 2)()
            _lib.check(lib.dw_model_costs(d._h, int(wr.parse_policy_kind(k)), int(t), out))
            assert (out[0], out[1]) == (c["instructions"], c["fp_adds"]), (name, key)
    assert np is not None
