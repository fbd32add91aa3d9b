"""DISTWAR hot-path benchmark (BASELINE.json metric: backward grad-contributions/s
and ms/iter vs naive-atomic; L2-atomic roofline %).

    python bench.py [--gpus N --steps K --warmup W] [--impl reference]
    torchrun --nproc-per-node N bench.py --gpus N ...

Workload (config.workload): BASELINE configs[4] -- 3M synthetic Gaussians,
1920x1080, a 64-view orbit batch sharded across the ranks (strong scaling:
the batch is fixed, each of N ranks renders 64/N views; `--views-per-gpu V`
switches to weak scaling). Every rank's views are resident in HBM. A STEP is
the backward pass of the rasterizer over the rank's views (DISTWAR SW-B,
balancing threshold tuned on the box with the reference's sweep rule) plus,
for N > 1, the NCCL all-reduce of the per-Gaussian gradient buffer -- run
through paper_2401_05345_b200.dist.view_parallel_backward. One unit = one
gradient contribution = (contributing pixel, Gaussian, param), 9 per pair
(SURVEY.md §8(d)). The north_star's >= 2x target scene (configs[2], 1M
Gaussians, one 1080p view) is timed beside it (`target_config`).

Printed on rank 0 as ONE JSON line; `value` = all ranks' contributions / the
max over ranks of the device-timed steps; `e2e` = the same metric through the
host-buffer C-ABI calls (dw_render_views_host at N = 1; at N > 1
dw_render_views_allreduce: the views, the NCCL all-reduce of the device
gradient over torch's communicator and one D2H in one call), the figure to
compare with the reference arm.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import math
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

# paper_2401_05345_b200.scene.CONFIGS keys: the benchmarked batch is BASELINE
# configs[4] (3M Gaussians, a 64-view batch sharded across 1/2/4/8 GPUs); the
# north_star's >= 2x target is stated on configs[2] (1M, one 1080p view),
# reported beside it as `target_config`
WORKLOAD = "c5_3m_1080p_64views"
TARGET = "c3_1m_1080p"
METRIC = "backward grad-contributions/sec & ms/iter vs naive-atomic; L2 atomic roofline %"
UNIT = "contributions/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default=WORKLOAD)
    ap.add_argument("--views", type=int, default=64,
                    help="the view batch, sharded across ranks (strong scaling; the default)")
    ap.add_argument("--views-per-gpu", type=int, default=0,
                    help="if > 0: this many views per rank instead (weak scaling)")
    ap.add_argument("--naive-steps", type=int, default=0,
                    help="timed steps of the naive comparison (0: max(3, steps // 4))")
    ap.add_argument("--threshold", default="auto", help="SW-B balancing threshold or 'auto'")
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-tile-stride", type=int, default=1)
    ap.add_argument("--no-trace-family", action="store_true")
    return ap.parse_args()


# SURVEY.md §8(d) trace family T, config C3 (reference-pinned workload)
TRACE_C3 = dict(num_primitives=1_000_000, params_per_primitive=9, image_width=1920,
                image_height=1080, mean_fragment_span=48.0, fragments_per_pixel_mean=8.0,
                locality=0.99, activity_prob=0.7, seed=1)


def trace_family() -> dict:
    """The reference's own workload (WarpRecord trace C3, byte-identical to
    workload::generate) through the trace-driven kernels: measured threshold
    sweep (dw_tune) and one device-timed launch per policy."""
    from paper_2401_05345_b200 import warpred as wr

    tr = wr.generate(wr.SceneSpec(**TRACE_C3))
    rep = wr.tune(tr, wr.PolicyFamily.sw_b, iteration=-1, reps=3)
    rep_s = wr.tune(tr, wr.PolicyFamily.sw_s, iteration=-1, reps=1)
    d = wr.DeviceTrace(tr)
    hbm, _ = measured_peaks()
    alg = d.records * (132 + 128 * d.params) + 4 * d.num_primitives * d.params
    out = {"config": "C3 trace: " + json.dumps(TRACE_C3), "records": d.records,
           "sw_b_threshold": rep.chosen, "sw_s_threshold": rep_s.chosen,
           "sw_b_sweep_us": {t: round(v, 2) for t, v in rep.us_by_threshold.items()}}
    for name, pol in (("native", wr.Policy(wr.PolicyKind.native, 0)),
                      ("sw_b", wr.Policy(wr.PolicyKind.sw_b, rep.chosen)),
                      ("sw_s", wr.Policy(wr.PolicyKind.sw_s, rep_s.chosen)),
                      ("cccl", wr.Policy(wr.PolicyKind.cccl, 0))):
        best = None
        for _ in range(3):
            _, m = wr.gpu_run(d, pol, want_sums=False)
            best = m if best is None or m.kernel_ms < best.kernel_ms else best
        out[name] = {"ms": best.kernel_ms, "contributions": best.contributions,
                     "value": best.contributions / (best.kernel_ms * 1e-3),
                     "reds": best.atomic_requests_to_l2,
                     "hbm_frac": alg / (best.kernel_ms * 1e-3) / (hbm * 1e9)}
    out["speedup_sw_b_vs_native"] = out["native"]["ms"] / out["sw_b"]["ms"]
    return out


# --------------------------------------------------------------------- utils
def host_threads() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.p = None
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                                       "-lms", "100", "-i", str(gpu)], stdout=subprocess.PIPE,
                                      stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.p = None

    def stop(self) -> dict:
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.p.terminate()
        out, _ = self.p.communicate(timeout=10)
        sm, smax, reasons, power = [], [], set(), []
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in out.strip().splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                smax.append(float(f[2]))
                power.append(float(f[3]))
            except ValueError:
                continue
            for name, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(name)
        loaded = [s for s, p in zip(sm, power) if p > 200.0] or sm
        return {"sm_mhz": statistics.median(loaded) if loaded else None,
                "sm_max_mhz": max(smax) if smax else None, "reasons": sorted(reasons),
                "samples": len(sm), "power_w_max": max(power) if power else None}


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json)"
    return 6650.0, "fallback (B200_PROFILING.md)"


def to_ocam(cam):
    from oracle.bindings import Camera as OCam

    oc = OCam()
    cc = cam.to_c()
    C.memmove(C.byref(oc), C.byref(cc), C.sizeof(oc))
    return oc


# ----------------------------------------------------------- CPU baselines
def cpu_port_baseline(sc, cam, dL, stride: int, workload: str) -> dict:
    """The oracle port's CPU backward (gradient math + per-address
    accumulation) on this box's host cores: the cpu_baseline of our arm."""
    from oracle.bindings import Oracle

    orc = Oracle()
    threads = host_threads()
    oc = to_ocam(cam)
    st = orc.gs_prepare(sc, oc, threads)
    try:
        secs, pairs, _ = orc.gs_backward_timed(st, oc, dL, threads, stride)
    finally:
        orc.gs_free(st)
    return {"value": 9 * pairs / secs, "unit": UNIT, "cores": threads, "kind": "port",
            "sample": f"view 0 of {workload}, every {stride} tile(s): {pairs} pairs "
                      f"({9 * pairs} contributions) in {secs:.2f} s, oracle/gs_oracle.c "
                      f"backward on {threads} threads"}


def reference_measure(workload: str, steps: int, warmup: int, stride: int, cam=None):
    """The reference's own CPU implementation of the path on this box's host
    cores. The reference (warpred) implements the reduction stage only
    (reducers::apply_policy + per-address summation, oracle/_ref built from
    /root/reference); the per-pair 3DGS gradient math it lacks is the oracle
    port producing the per-warp WarpRecords it consumes (in the GPU reduction
    kernel's two-pixels-per-lane layout). Each step: port gradient math over a
    tile-strided sample of view 0 (all host threads) + the reference's SW-B
    reduction of those records (all host threads). Returns a cpu_baseline dict
    plus the total seconds of the timed steps."""
    from oracle.bindings import REF_SO, Oracle, Ref
    from paper_2401_05345_b200.scene import CONFIGS, make_camera, make_dL_dpixels, make_scene

    P, W, H, hc, _ = CONFIGS[workload]
    sc = make_scene(P, W, H, seed=0, high_contention=hc)
    cam = cam or make_camera(W, H)
    dL = make_dL_dpixels(W, H, seed=1)
    orc = Oracle()
    threads = host_threads()
    oc = to_ocam(cam)
    have_ref = os.path.exists(REF_SO)
    ref = Ref() if have_ref else None
    st = orc.gs_prepare(sc, oc, threads)
    times, contribs = [], 0
    try:
        for i in range(warmup + steps):
            t_math, pairs, tap = orc.gs_backward_timed(st, oc, dL, threads, stride, tap=2)
            if ref is not None:
                h = ref.from_trace(tap)
                t_red, _, _ = ref.time_policy(h, 2, 0, P, threads)
                ref.free(h)
            else:  # reference not built here: the oracle restatement of it
                t0 = time.perf_counter()
                orc.apply_policy(tap, 2, 0, P)
                t_red = time.perf_counter() - t0
            if i >= warmup:
                times.append(t_math + t_red)
                contribs += 9 * pairs
    finally:
        orc.gs_free(st)
    total = sum(times)
    return {"value": contribs / total, "unit": UNIT, "cores": threads,
            "kind": "reference" if have_ref else "port",
            "sample": f"every {stride}th tile of view 0 of {workload}, {steps} step(s): port "
                      "gradient math + reference reducers::apply_policy(sw_b, 0) + per-address "
                      f"sums, {threads} host threads"}, total


def reference_arm(args) -> None:
    """--impl reference: reference_measure() over the arm's --steps/--warmup."""
    from paper_2401_05345_b200.scene import CONFIGS

    from paper_2401_05345_b200.scene import orbit_cameras

    P, W, H, _, _ = CONFIGS[args.workload]
    stride = max(args.cpu_tile_stride, 16)
    # view 0 of the arm's batch (the orbit camera our arm's rank 0 renders first)
    views = args.views_per_gpu * args.gpus if args.views_per_gpu > 0 else args.views
    cam0 = orbit_cameras(W, H, views)[0] if views > 1 else None
    cpu, total = reference_measure(args.workload, args.steps, args.warmup, stride, cam0)
    v = cpu["value"]
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total / args.steps,
        "higher_is_better": True,
        "scaling": "weak" if args.views_per_gpu > 0 else "strong", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic",
        "config": {"workload": args.workload, "gaussians": P, "width": W, "height": H,
                   "views_total": views, "sample": f"every {stride}th tile of view 0"},
        "cpu_baseline": cpu,
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    emit(line)


# The driver reads ONE JSON line from stdout: native libraries (NCCL prints its
# version banner on the first collective) are pointed at stderr, the line goes
# to the original stdout.
_JSON_OUT = None


def quiet_stdout() -> None:
    global _JSON_OUT
    if _JSON_OUT is None:
        sys.stdout.flush()
        _JSON_OUT = os.fdopen(os.dup(1), "w")
        os.dup2(2, 1)


def emit(line: dict) -> None:
    out = _JSON_OUT if _JSON_OUT is not None else sys.stdout
    print(json.dumps(line), file=out, flush=True)


# ----------------------------------------------------------------- our arm
def stage_breakdown(t, cam, P, H, W, prof_key="") -> dict:
    """Per-stage forward times of one view (CUDA events between the stages,
    dw_rasterizer_stage_timing) with each stage's algorithmic bytes and HBM
    fraction; the events serialise the programmatic-dependent launches, so
    the stages sum to slightly more than the untimed forward."""
    import numpy as np
    import torch

    from paper_2401_05345_b200.rasterizer import GaussianRasterizer

    r = GaussianRasterizer()
    r.stage_timing(True)
    best = None
    for _ in range(3):
        r.render_forward(t["means3D"], t["scales"], t["rotations"], t["opacities"],
                         t["colors"], cam)
        ms = r.stage_ms()
        best = ms if best is None else {k: min(best[k], ms[k]) for k in ms}
    torch.cuda.synchronize()
    I = r.num_rendered
    vis = int((r.buffer("radii") > 0).sum())
    hbm, _ = measured_peaks()
    # algorithmic bytes per stage: reads + writes the stage
    # cannot avoid, counted once
    block = os.environ.get("DW_BLOCK_BINNING", "1") != "0" and W <= 255 * 16 and H <= 255 * 16
    alg = {"preprocess": 56 * P + 64 * P,           # scene in; means2D..keys + packed rect out
           "depth_sort": 4 * 16 * vis,              # 4 LSD passes, 8 B in + 8 B out each
           "ranges": 4 * I + 8 * (W // 16 + 1) * (H // 16 + 1),
           "blend": 4 * I + 44 * vis + 20 * H * W}
    if block:
        # block binning (raster_blockbin.cu): Nc = (Gaussian, coarse 8x4-tile
        # block) entries, from the rectangles exactly as the kernels form them
        m2 = r.buffer("means2D").reshape(-1, 2).astype(np.float32)
        rad = r.buffer("radii").astype(np.float32)
        live = rad > 0
        tx, ty = (W + 15) // 16, (H + 15) // 16
        f16 = np.float32(16.0)
        x0 = np.clip(np.trunc((m2[:, 0] - rad) / f16), 0, tx).astype(np.int64)
        y0 = np.clip(np.trunc((m2[:, 1] - rad) / f16), 0, ty).astype(np.int64)
        x1 = np.clip(np.trunc((m2[:, 0] + rad + np.float32(15)) / f16), 0, tx).astype(np.int64)
        y1 = np.clip(np.trunc((m2[:, 1] + rad + np.float32(15)) / f16), 0, ty).astype(np.int64)
        ok = live & (x1 > x0) & (y1 > y0)
        nc = int((((x1 - 1) // 8 - x0 // 8 + 1) * ((y1 - 1) // 4 - y0 // 4 + 1))[ok].sum())
        alg["offsets"] = 8 * vis + 8 * nc           # rects + ids in, entries out
        alg["binning"] = 20 * nc + 4 * nc + 8 * nc + 4 * I  # entry sort pass, count, place
        alg["_entries"] = nc
    else:
        alg["offsets"] = 12 * P                     # areas in, u64 offsets out
        alg["binning"] = 20 * vis + 8 * I + 2 * 16 * I  # duplicate + 2 tile-sort passes
    out = {"_list_construction": "block binning" if block else "duplicate + tile sort",
           "_entries": alg.pop("_entries", None)}
    for k, ms in best.items():
        gbs = alg[k] / (ms * 1e-3) / 1e9 if ms > 0 else None
        out[k] = {"ms": ms, "alg_bytes": alg[k], "GBps": gbs,
                  "hbm_frac": gbs / hbm if gbs else None}
    out["_sum_ms"] = sum(best.values())
    # the blend's binding roofline: SM instruction issue (warp instructions
    # per launch from the committed ncu count of this view's blend, over the
    # event-timed blend stage, vs 148 x 4 issue slots x the max SM clock)
    fi_path = os.path.join(ROOT, "profiles", "forward_inst.json")
    fi = json.load(open(fi_path)).get(prof_key) if os.path.exists(fi_path) else None
    if fi and best.get("blend"):
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
            os.path.join(ROOT, "MEASURED_PEAKS.json")) else {}
        clk = peaks.get("sm_max_mhz", 1965.0)
        ach = fi["k_forward_x2"] / (best["blend"] * 1e-3)
        out["blend_roofline_issue"] = {
            "bound": "issue", "achieved": ach, "peak": 148 * 4 * clk * 1e6, "unit": "warp-inst/s",
            "frac": ach / (148 * 4 * clk * 1e6), "inst_per_launch": fi["k_forward_x2"],
            "ncu_issue_active_pct": fi.get("issue_active_pct"),
            "inst_source": f"profiles/forward_inst.json {prof_key}"}
    out["_note"] = ("CUDA events between stages (serialises the PDL chain); blend is "
                    "issue-bound, the others latency/HBM")
    return out


def main() -> None:
    args = parse()
    quiet_stdout()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        if rank == 0:
            reference_arm(args)
        return

    import torch

    from paper_2401_05345_b200 import _lib
    from paper_2401_05345_b200 import warpred as wr
    from paper_2401_05345_b200.dist import shard_views, view_parallel_backward
    from paper_2401_05345_b200.rasterizer import (GaussianRasterizer, microbench_red,
                                                  render_backward_views,
                                                  nccl_comm_ptr, render_views,
                                                  render_views_allreduce, render_views_host)
    from paper_2401_05345_b200.scene import CONFIGS, make_camera, make_dL_dpixels, make_scene, \
        orbit_cameras

    if os.environ.get("DW_BENCH_BACKEND", "nccl") != "nccl":
        local %= torch.cuda.device_count()  # the test hook's ranks may share a GPU
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist = None
    # DW_BENCH_FORCE_DIST=1 (under torchrun) exercises the NCCL path at N = 1
    if world > 1 or os.environ.get("DW_BENCH_FORCE_DIST") == "1":
        import torch.distributed as dist

        # DW_BENCH_BACKEND=gloo: a test hook that runs the multi-rank logic with
        # several ranks on ONE GPU (NCCL refuses duplicate GPUs); timings from
        # such a run are not scaling numbers
        backend = os.environ.get("DW_BENCH_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)

    P, W, H, hc, cfg_views = CONFIGS[args.workload]
    weak = args.views_per_gpu > 0
    total_views = args.views_per_gpu * world if weak else (args.views or max(cfg_views, 64))
    if total_views < world:
        raise SystemExit("need at least one view per rank")
    my_views = list(shard_views(total_views, world, rank))
    V = len(my_views)
    sc = make_scene(P, W, H, seed=0, high_contention=hc)
    all_cams = orbit_cameras(W, H, total_views) if total_views > 1 else [make_camera(W, H)]
    cams = [all_cams[i] for i in my_views]
    t = {k: torch.from_numpy(v).to(dev) for k, v in sc.items()}
    dLs = [torch.from_numpy(make_dL_dpixels(W, H, seed=1 + i)).to(dev) for i in my_views]
    stream = torch.cuda.current_stream()
    local_of = {g: i for i, g in enumerate(my_views)}

    def ev():
        return torch.cuda.Event(enable_timing=True)

    # ---- forward: resident per-view states (timed for forward fps) -------
    rasts = [GaussianRasterizer() for _ in range(V)]
    fwd_ms = []  # per view: median of 3 warm render_forward calls (after a first, sizing one)
    for i, r in enumerate(rasts):
        reps = []
        for rep in range(4):
            e0, e1 = ev(), ev()
            e0.record()
            r.render_forward(t["means3D"], t["scales"], t["rotations"], t["opacities"],
                             t["colors"], cams[i])
            e1.record()
            torch.cuda.synchronize()
            if rep >= 1:
                reps.append(e0.elapsed_time(e1))
        fwd_ms.append(statistics.median(reps))
    # the rank's forwards without host synchronisation (render_forward_async
    # over a 1.5x reserve: the graph-capturable path), back to back on one
    # stream and rotating over four streams (the batched host path's forward
    # phase); the same cameras, so every state ends as the counted forward left it
    for r in rasts:
        r.reserve(P, W, H, r.num_rendered + r.num_rendered // 2 + 4096)
    img_s = [torch.empty((3, H, W), device=dev) for _ in range(4)]
    rad_s = [torch.empty(P, dtype=torch.int32, device=dev) for _ in range(4)]
    fstreams = [torch.cuda.Stream() for _ in range(4)]

    def forwards_async(nstreams):
        torch.cuda.synchronize()
        e0, e1 = ev(), ev()
        e0.record()
        for fs in fstreams[:nstreams]:
            fs.wait_event(e0)
        for i, r in enumerate(rasts):
            j = i % nstreams
            r.render_forward_async(t["means3D"], t["scales"], t["rotations"], t["opacities"],
                                   t["colors"], cams[i], img_s[j], rad_s[j], stream=fstreams[j])
        for fs in fstreams[:nstreams]:
            torch.cuda.current_stream().wait_stream(fs)
        e1.record()
        torch.cuda.synchronize()
        assert not any(r.instances()[1] for r in rasts), "forward reserve overflow"
        return e0.elapsed_time(e1) / len(rasts)

    fwd_async = {}
    for ns in (1, 4):
        forwards_async(ns)
        fwd_async[ns] = statistics.median(forwards_async(ns) for _ in range(3))
    stages = (stage_breakdown(t, cams[0], P, H, W,
                              f"{args.workload}@view{my_views[0]}/{total_views}")
              if rank == 0 else None)
    grad = torch.zeros((P, 9), dtype=torch.float32, device=dev)

    # ---- contributions per step (counting instantiation, untimed) --------
    pairs_per_view = []
    for r, dL in zip(rasts, dLs):
        _, pairs = r.render_backward(dL, wr.Policy(wr.PolicyKind.native, 0), grad=grad,
                                     count_pairs=True)
        pairs_per_view.append(pairs)
    contrib_rank = 9 * sum(pairs_per_view)

    # ---- roofline microbenchmarks: measured L2 RED throughput ------------
    red_peaks = {name: microbench_red(p, 1 << 28) for p, name in
                 ((0, "distinct"), (1, "same_address_warp"), (2, "v4"), (3, "distwar_9lane"),
                  (4, "same_address_warp_v4"), (5, "fallback_row_scalar"),
                  (6, "fallback_row_vector"), (7, "reduced_row_vector"))}

    def time_view(i, policy, reps=3):
        ms = []
        for _ in range(reps):
            e0, e1 = ev(), ev()
            grad.zero_()
            e0.record()
            rasts[i].render_backward(dLs[i], policy, grad=grad)
            e1.record()
            torch.cuda.synchronize()
            ms.append(e0.elapsed_time(e1))
        return statistics.median(ms)

    # ---- balancing threshold: measured sweep 0..32 (tuner.cpp:29-52) on the
    # timed path itself -- the batch call over the rank's first views (chained
    # launches, padded rows), ms per view -- argmin, ties to the lowest t
    sweep = {}
    nsw = min(8, V)

    def time_batch(policy, reps=3):
        ms = []
        for _ in range(reps):
            e0, e1 = ev(), ev()
            grad.zero_()
            e0.record()
            render_backward_views(rasts[:nsw], dLs[:nsw], policy, grad)
            e1.record()
            torch.cuda.synchronize()
            ms.append(e0.elapsed_time(e1) / nsw)
        return statistics.median(ms)

    if args.threshold == "auto":
        time_batch(wr.Policy(wr.PolicyKind.sw_b, 0), reps=2)
        best = None
        for thr in range(33):
            sweep[thr] = time_batch(wr.Policy(wr.PolicyKind.sw_b, thr))
            if best is None or sweep[thr] < sweep[best]:
                best = thr
        thr = best
        if dist is not None:  # one threshold for the job: rank 0's choice
            b = torch.tensor([thr], device=dev)
            dist.broadcast(b, 0)
            thr = int(b.item())
    else:
        thr = int(args.threshold)
    policy = wr.Policy(wr.PolicyKind.sw_b, thr)

    def last_reds(r):
        v = C.c_uint64()
        _lib.check(_lib.lib().dw_rasterizer_last_reds(r.handle, C.byref(v)))
        return v.value

    reds_distwar = 0
    for r, dL in zip(rasts, dLs):
        r.render_backward(dL, policy, grad=grad, count_pairs=True)
        reds_distwar += last_reds(r)

    # ---- the timed loop: dist.view_parallel_backward over the batch --------
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)

    # The rank's backwards run as one chain (dw_render_backward_chained after
    # the first: the views are independent and already rendered, so a launch
    # need not wait for the previous grid -- its CTAs fill the SMs the
    # previous launch's last wave leaves idle; C5: 0.791 -> 0.745 ms per view,
    # profiles/r02/ab/chained_backward.md). Events bracket the step only (an
    # event between two launches would serialise them); a launch's duration is
    # the step's per-launch share, and view 0 is also timed alone (time_view).
    def run_steps(pol, steps, warmup):
        per_step, per_launch, view0 = [], [], []
        n_local = len(my_views)
        for s in range(warmup + steps):
            flush.fill_(float(s))  # L2 flush (256 MiB > 126 MB L2), outside the events
            torch.cuda.synchronize()
            if dist is not None:
                dist.barrier()
            def backward_views(gs, out):
                render_backward_views([rasts[local_of[g]] for g in gs],
                                      [dLs[local_of[g]] for g in gs], pol, out)

            e_start, e_mid, e_end = ev(), ev(), ev()
            e_start.record()
            grad.zero_()
            view_parallel_backward(None, list(range(total_views)), grad, all_reduce=False,
                                   backward_views=backward_views)
            e_mid.record()
            if dist is not None:
                dist.all_reduce(grad, op=dist.ReduceOp.SUM)
            e_end.record()
            torch.cuda.synchronize()
            if s >= warmup:
                per_step.append(e_start.elapsed_time(e_end))
                per_launch.extend([e_start.elapsed_time(e_mid) / n_local] * n_local)
        total = sum(per_step)
        if dist is not None:
            tt = torch.tensor([total], device=dev, dtype=torch.float64)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            total = float(tt.item())
        return total, per_launch, view0

    sampler = ClockSampler(local)
    time.sleep(0.3)
    total_ms, launches, _ = run_steps(policy, args.steps, args.warmup)
    launches_v0 = [time_view(0, policy, reps=5)]  # view 0 alone (the issue roofline's launch)
    nv_steps = args.naive_steps or max(3, args.steps // 4)
    total_nv_ms, launches_nv, _ = run_steps(wr.Policy(wr.PolicyKind.native, 0), nv_steps,
                                            min(args.warmup, 3))
    clocks = sampler.stop()
    ms_per_step = total_ms / args.steps

    # ---- where the speed-up comes from (view 0): the naive one-pixel kernel,
    # the two-pixel kernel with no warp reduction (SW-B at t = 33: every lane
    # issues its own REDs), and SW-B at the tuned t (PAPER.md:1481-1504 loop)
    # -- and the per-lane REDs as one scalar RED per param (DW_VEC_RED=0: the
    # two-pixel layout alone) or as 3-4 aligned vector REDs per row
    os.environ["DW_VEC_RED"] = "0"
    x2_scalar = time_view(0, wr.Policy(wr.PolicyKind.sw_b, 33), reps=5)
    os.environ.pop("DW_VEC_RED", None)
    dec = {"native_1px_ms": time_view(0, wr.Policy(wr.PolicyKind.native, 0), reps=5),
           "x2_no_reduction_scalar_red_ms": x2_scalar,
           "x2_no_reduction_ms": time_view(0, wr.Policy(wr.PolicyKind.sw_b, 33), reps=5),
           "sw_b_tuned_ms": time_view(0, policy, reps=5)}
    dec["layout_factor"] = dec["native_1px_ms"] / dec["x2_no_reduction_scalar_red_ms"]
    dec["vector_red_factor"] = dec["x2_no_reduction_scalar_red_ms"] / dec["x2_no_reduction_ms"]
    dec["distwar_factor"] = dec["x2_no_reduction_ms"] / dec["sw_b_tuned_ms"]
    dec["total_factor"] = dec["native_1px_ms"] / dec["sw_b_tuned_ms"]
    dec["_note"] = ("native one-pixel kernel -> two-pixel packed-FP32 kernel with no warp "
                    "reduction (t = 33) and scalar per-lane REDs -> the same with the per-lane "
                    "REDs as aligned vector REDs -> SW-B at the tuned t")

    # ---- the step's one exchange, timed alone: NCCL all-reduce
    # of grad[P, 9] fp32, device events, max over ranks; bus bandwidth uses
    # the ring-equivalent factor 2 (n - 1) / n
    allreduce = None
    if dist is not None:
        reps = 10
        for _ in range(3):
            dist.all_reduce(grad)
        torch.cuda.synchronize()
        dist.barrier()
        e0, e1 = ev(), ev()
        e0.record()
        for _ in range(reps):
            dist.all_reduce(grad)
        e1.record()
        torch.cuda.synchronize()
        ar = torch.tensor([e0.elapsed_time(e1) / reps], device=dev, dtype=torch.float64)
        dist.all_reduce(ar, op=dist.ReduceOp.MAX)
        ar_ms = float(ar.item())
        nbytes = grad.numel() * grad.element_size()
        allreduce = {"bytes": nbytes, "ms": ar_ms, "share_of_step": ar_ms / ms_per_step,
                     "busbw_GBps": nbytes * 2 * (world - 1) / world / (ar_ms * 1e-3) / 1e9,
                     "backend": dist.get_backend(), "world": world}
    contrib_job = float(contrib_rank)
    if dist is not None:
        c = torch.tensor([contrib_rank], device=dev, dtype=torch.float64)
        dist.all_reduce(c)
        contrib_job = float(c.item())
    value = contrib_job * args.steps / (total_ms * 1e-3)
    naive_value = contrib_job * nv_steps / (total_nv_ms * 1e-3)

    # ---- e2e through the host-buffer C-ABI calls -------------------------
    # per step: pinned H2D of the scene + the rank's dL/dpixel, forward +
    # backward of every view, D2H of the images; N = 1: dw_render_views_host
    # (gradient D2H inside); N > 1: dw_render_views_allreduce -- the views into
    # a device gradient, the NCCL all-reduce over NVLink (torch's communicator
    # handed to the C ABI), then ONE D2H of the sum, all inside one C call
    pin = {k: torch.from_numpy(v).pin_memory() for k, v in sc.items()}
    dL_h = torch.stack([d.cpu() for d in dLs]).pin_memory()
    img_h = torch.empty((V, 3, H, W), dtype=torch.float32).pin_memory()
    grad_h = torch.empty((P, 9), dtype=torch.float32).pin_memory()
    use_nccl_abi = dist is not None and dist.get_backend() == "nccl"
    comm = nccl_comm_ptr() if use_nccl_abi else None
    grad_d = torch.empty((P, 9), dtype=torch.float32, device=dev) if (
        dist is not None and not use_nccl_abi) else None
    e2e_r = GaussianRasterizer()
    scene_ptrs = [pin[k].data_ptr() for k in ("means3D", "scales", "rotations", "opacities",
                                               "colors")]

    def e2e_step():
        if dist is None:
            render_views_host(e2e_r, scene_ptrs, P, cams, dL_h.data_ptr(), policy,
                              img_h.data_ptr(), grad_h.data_ptr(), stream)
        elif use_nccl_abi:
            render_views_allreduce(e2e_r, scene_ptrs, P, cams, dL_h.data_ptr(), policy,
                                   img_h.data_ptr(), grad_h.data_ptr(), comm, stream)
        else:  # non-NCCL test backend: device gradient, torch all-reduce, one D2H
            render_views(e2e_r, scene_ptrs, P, cams, dL_h.data_ptr(), policy, img_h.data_ptr(),
                         grad_d, stream)
            dist.all_reduce(grad_d)
            grad_h.copy_(grad_d)
            torch.cuda.synchronize()

    e2e_step()  # warm-up (allocations)
    torch.cuda.synchronize()
    if dist is not None:
        dist.barrier()
    t0 = time.perf_counter()
    for _ in range(args.e2e_steps):
        e2e_step()
    torch.cuda.synchronize()
    e2e_s = time.perf_counter() - t0
    if dist is not None:
        tt = torch.tensor([e2e_s], device=dev, dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        e2e_s = float(tt.item())
    e2e_value = contrib_job * args.e2e_steps / e2e_s
    h2d = sum(v.nbytes for v in sc.values()) + 3 * H * W * 4 * V
    d2h = 3 * H * W * 4 * V + P * 9 * 4

    # ---- rooflines of the dominant kernel (k_backward_x2<sw_b>) ----------
    hbm_peak, peak_src = measured_peaks()
    mean_launch_ms = statistics.mean(launches)
    v0_launch_ms = statistics.mean(launches_v0)
    inst = statistics.mean(r.num_rendered for r in rasts)
    vis = statistics.mean(int((r.buffer("radii") > 0).sum()) for r in rasts)
    alg_bytes = 4 * inst + 44 * vis + 20 * H * W + 36 * P
    achieved_gbs = alg_bytes / (mean_launch_ms * 1e-3) / 1e9
    prof_key = f"{args.workload}@view{my_views[0]}/{total_views}"
    spec = f"sw_b:{thr}"

    def prof(name):
        p = os.path.join(ROOT, "profiles", name)
        return json.load(open(p)).get(prof_key, {}) if os.path.exists(p) else {}

    inst_t, dram_t = prof("backward_inst.json"), prof("backward_dram_bytes.json")
    traffic = dram_t.get(spec)
    issue = None
    if inst_t.get(spec) and clocks.get("sm_mhz"):
        ach = inst_t[spec] / (v0_launch_ms * 1e-3)
        peak = 148 * 4 * clocks["sm_mhz"] * 1e6
        issue = {"bound": "issue", "achieved": ach, "peak": peak, "unit": "warp-inst/s",
                 "frac": ach / peak, "inst_per_launch": inst_t[spec],
                 "launch_ms": v0_launch_ms,
                 "_launch": "view 0's backward timed alone (events around one launch, "
                            "[P][9] rows); the instruction count is the timed path's "
                            "(a chained launch into the padded rows, a few % fewer "
                            "instructions), so this alone-fraction reads slightly low",
                 # the timed chain: launches overlap their neighbours' tails,
                 # so the step's per-launch share keeps the issue slots busier
                 "chained": {"launch_ms": mean_launch_ms,
                             "frac": inst_t[spec] / (mean_launch_ms * 1e-3) / peak,
                             "_note": "view 0's instruction count over the timed chain's "
                                      "per-launch share (views' counts are alike)"},
                 "inst_source": f"ncu sm__inst_executed.sum, {prof_key} {spec} "
                                f"(profiles/backward_inst.json: {inst_t.get('csv')})",
                 "peak_source": "148 SMs x 4 schedulers x 1 warp-inst/cycle x median SM clock "
                                "of this run"}
    reds_per_launch = reds_distwar / V
    red_rate = reds_per_launch / (mean_launch_ms * 1e-3)
    naive_launch_ms = statistics.mean(launches_nv)
    naive_red_rate = (contrib_rank / V) / (naive_launch_ms * 1e-3)

    # ---- the north_star target scene (BASELINE configs[2]): one view, naive
    # vs DISTWAR at its own tuned threshold
    target = None
    if rank == 0 and args.workload != TARGET:
        Pc, Wc, Hc, hcc, _ = CONFIGS[TARGET]
        tc = {k: torch.from_numpy(v).to(dev)
              for k, v in make_scene(Pc, Wc, Hc, seed=0, high_contention=hcc).items()}
        rc = GaussianRasterizer()
        rc.render_forward(tc["means3D"], tc["scales"], tc["rotations"], tc["opacities"],
                          tc["colors"], make_camera(Wc, Hc))
        dLc = torch.from_numpy(make_dL_dpixels(Wc, Hc, seed=1)).to(dev)
        gc = torch.zeros((Pc, 9), device=dev)

        def tc_ms(pol, reps=5):
            ms = []
            for _ in range(reps):
                e0, e1 = ev(), ev()
                e0.record()
                rc.render_backward(dLc, pol, grad=gc)
                e1.record()
                torch.cuda.synchronize()
                ms.append(e0.elapsed_time(e1))
            return statistics.median(ms)

        _, pc = rc.render_backward(dLc, wr.Policy(wr.PolicyKind.native, 0), grad=gc,
                                   count_pairs=True)
        sw = {tt: tc_ms(wr.Policy(wr.PolicyKind.sw_b, tt), reps=3) for tt in range(33)}
        tbest = min(sw, key=lambda k: (sw[k], k))
        nat = tc_ms(wr.Policy(wr.PolicyKind.native, 0))
        swb = tc_ms(wr.Policy(wr.PolicyKind.sw_b, tbest))
        target = {"workload": TARGET, "pairs": pc, "threshold": tbest, "native_ms": nat,
                  "sw_b_ms": swb, "speedup": nat / swb,
                  "sw_b_contributions_per_s": 9 * pc / (swb * 1e-3),
                  "north_star_target": ">= 2x naive-atomic"}
        del rc, tc, gc, dLc

    tfam = None
    if rank == 0 and not args.no_trace_family:
        tfam = trace_family()

    cpu = cpu_port = None
    if rank == 0 and not args.no_cpu_baseline:
        # the reference's CPU path (oracle/_ref) on a bounded sample of view 0,
        # and the oracle port's whole backward of view 0, on this box's cores
        cpu, _ = reference_measure(args.workload, 3, 1, 16, cams[0])
        cpu_port = cpu_port_baseline(sc, cams[0], make_dL_dpixels(W, H, seed=1 + my_views[0]),
                                     args.cpu_tile_stride, args.workload)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "weak" if weak else "strong", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic",
            "config": {"workload": args.workload, "gaussians": P, "width": W, "height": H,
                       "views_total": total_views, "views_per_gpu": V,
                       "policy": "sw_b", "threshold": thr,
                       "parallelism": f"dp{world} (views) + "
                                      f"{(dist.get_backend() if dist else 'nccl').upper()} "
                                      f"all-reduce of grad[P,9]"
                       if world > 1 else "dp1",
                       "l2": "flushed between steps (256 MiB write, outside the events)"},
            # per step: the rank's V backward launches + the padded-row fold
            "gpu_launches": args.steps * (V + 1),
            "clocks": clocks,
            "naive": {"value": naive_value, "ms_per_step": total_nv_ms / nv_steps,
                      "steps": nv_steps,
                      "speedup_distwar_vs_naive": naive_value and value / naive_value},
            "decomposition_view0": dec,
            "target_config": target,
            "forward": {"ms_per_view": statistics.mean(fwd_ms),
                        "fps": 1e3 / statistics.mean(fwd_ms),
                        "async_one_stream": {"ms_per_view": fwd_async[1],
                                             "fps": 1e3 / fwd_async[1]},
                        "async_four_streams": {"ms_per_view": fwd_async[4],
                                               "fps": 1e3 / fwd_async[4]},
                        "_async": "the rank's views back to back without host synchronisation "
                                  "(render_forward_async over a 1.5x reserve), on one stream / "
                                  "rotating over four (the batched host path's forward phase)",
                        "_timing": "render_forward (counted: one host read of the instance "
                                   "count mid-forward), per view the median of 3 warm calls, "
                                   "mean over the rank's views",
                        "stages_view0": stages},
            "contributions_per_step": contrib_job, "pairs_per_view": pairs_per_view,
            "instances_per_view": [r.num_rendered for r in rasts],
            "threshold_sweep_ms": sweep,
            "_threshold_sweep": "ms per view of the batch call (chained launches into the "
                                "padded rows) over the rank's first min(8, V) views, median "
                                "of 3, L2 not flushed; argmin, ties to the lowest t",
            "roofline": {"bound": "hbm", "achieved": achieved_gbs, "peak": hbm_peak,
                         "unit": "GB/s", "frac": achieved_gbs / hbm_peak,
                         "traffic": traffic, "traffic_source": f"ncu dram bytes, {prof_key} {spec}",
                         "kernel": "k_backward_x2<sw_b>", "alg_bytes_per_launch": alg_bytes,
                         "mean_launch_ms": mean_launch_ms, "peak_source": peak_src},
            "roofline_binding": "issue",
            "roofline_issue": issue,
            "roofline_l2_atomic": {
                "distwar": {"reds_per_launch": reds_per_launch, "achieved": red_rate,
                            "peak": red_peaks["distwar_9lane"],
                            "frac": red_rate / red_peaks["distwar_9lane"]},
                "naive": {"reds_per_launch": contrib_rank / V, "achieved": naive_red_rate,
                          "peak": red_peaks["same_address_warp"],
                          "frac": naive_red_rate / red_peaks["same_address_warp"]},
                "measured_red_peaks_per_s": red_peaks, "unit": "REDs/s"},
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h, "steps": args.e2e_steps,
                    "path": ("dw_render_views_host" if dist is None else
                             "dw_render_views_allreduce: views into a device gradient + NCCL "
                             "all-reduce (torch's communicator) + one D2H")
                            + ": pinned H2D scene + V dL/dpixel, forward + backward of V views, "
                              "D2H V images + grad"},
            "allreduce": allreduce,
            "cpu_baseline": cpu,
            "cpu_port": cpu_port,
            "trace_family": tfam,
        }
        emit(line)
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
