"""run the REFERENCE's machine model on the rasterizer's real
WarpRecords and set its threshold choice beside the one measured on the B200.

CPU part (this container, needs oracle/_ref): render a scene on the CPU
oracle, tap its per-warp records in the GPU reduction kernel's lane layout
(two pixels per lane), write WRTRACEB, and call the reference's own C ABI
(wr_trace_load / wr_machine_preset / wr_tune / wr_simulate, warpred.h:98-122)
for each machine preset. GPU part: tools/ab_backward.py on the same workload
gives the measured sweep. Output: JSON with both sweeps.

    python tools/tap_vs_sim.py --workload c1_10k_256 --out profiles/r01/tap_vs_sim_c1.json
"""
import argparse
import ctypes as C
import json
import os
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


class Machine(C.Structure):  # wr_machine_config, warpred.h:55-66
    _fields_ = [("num_sms", C.c_int32), ("subcores_per_sm", C.c_int32),
                ("lsu_queue_depth", C.c_int32), ("rop_units", C.c_int32),
                ("rop_throughput", C.c_double), ("interconnect_latency", C.c_int32),
                ("interconnect_bandwidth", C.c_int32), ("red_unit_latency_per_add", C.c_int32),
                ("red_pipe_depth", C.c_int32), ("warp_issue_width", C.c_int32)]


class Metrics(C.Structure):  # wr_run_metrics, warpred.h:68-77
    _fields_ = [("total_cycles", C.c_uint64), ("stalls_lsu", C.c_uint64),
                ("stalls_other", C.c_uint64), ("atomic_requests_to_l2", C.c_uint64),
                ("core_instructions", C.c_uint64), ("core_fp_adds", C.c_uint64),
                ("interconnect_packets", C.c_uint64), ("energy_proxy", C.c_double)]


class Tune(C.Structure):  # wr_tune_report, warpred.h:79-84
    _fields_ = [("cycles_by_threshold", C.c_uint64 * 33), ("chosen", C.c_int32),
                ("profile_iteration", C.c_int32), ("reprofile_period", C.c_int32)]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="c1_10k_256")
    ap.add_argument("--presets", default="rtx4090like,rtx3060like")
    ap.add_argument("--tile-stride", type=int, default=1)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    from oracle.bindings import REF_SO, Camera as OCam, Oracle
    from paper_2401_05345_b200.scene import CONFIGS, make_camera, make_dL_dpixels, make_scene

    P, W, H, hc, _ = CONFIGS[a.workload]
    sc = make_scene(P, W, H, seed=0, high_contention=hc)
    cam = make_camera(W, H)
    oc = OCam()
    cc = cam.to_c()
    C.memmove(C.byref(oc), C.byref(cc), C.sizeof(oc))
    orc = Oracle()
    out = orc.gs_render(sc, oc, make_dL_dpixels(W, H, seed=1), threads=8, tap=True, tap_ppt=2,
                        tile_stride=a.tile_stride)
    tap = out["tap"]
    L = C.CDLL(REF_SO)
    L.wr_last_error.restype = C.c_char_p
    L.wr_trace_load.argtypes = [C.c_char_p, C.c_int, C.POINTER(C.c_void_p)]
    L.wr_machine_preset.argtypes = [C.c_char_p, C.POINTER(Machine)]
    L.wr_tune.argtypes = [C.c_void_p, C.POINTER(Machine), C.c_int, C.c_int32, C.POINTER(Tune)]
    L.wr_simulate.argtypes = [C.c_void_p, C.POINTER(Machine), C.c_int, C.c_int, C.POINTER(Metrics)]
    L.wr_trace_free.argtypes = [C.c_void_p]
    res = {"workload": a.workload, "records": tap.num_records,
           "contributions_in_records": tap.contributions(), "pairs": out["pairs"],
           "layout": "two pixels per lane (k_backward_x2)", "presets": {}}
    with tempfile.TemporaryDirectory() as td:
        path = os.path.join(td, "tap.wrtb")
        orc.save_binary(tap, path)
        h = C.c_void_p()
        if L.wr_trace_load(path.encode(), 1, C.byref(h)):
            raise RuntimeError(L.wr_last_error().decode())
        try:
            for name in a.presets.split(","):
                m = Machine()
                if L.wr_machine_preset(name.encode(), C.byref(m)):
                    raise RuntimeError(L.wr_last_error().decode())
                t0 = time.time()
                rep = Tune()
                if L.wr_tune(h, C.byref(m), 1, -1, C.byref(rep)):  # WR_FAMILY_SW_B
                    raise RuntimeError(L.wr_last_error().decode())
                nat = Metrics()
                if L.wr_simulate(h, C.byref(m), 0, 0, C.byref(nat)):
                    raise RuntimeError(L.wr_last_error().decode())
                cyc = list(rep.cycles_by_threshold)
                res["presets"][name] = {
                    "chosen": rep.chosen, "cycles_by_threshold": cyc,
                    "native_cycles": nat.total_cycles,
                    "predicted_speedup_vs_native": nat.total_cycles / cyc[rep.chosen],
                    "sim_seconds": round(time.time() - t0, 1)}
                print(name, rep.chosen, nat.total_cycles / cyc[rep.chosen], flush=True)
        finally:
            L.wr_trace_free(h)
    js = json.dumps(res)
    if a.out:
        open(a.out, "w").write(js + "\n")
    print(js[:300])


if __name__ == "__main__":
    main()
