"""Generate tests/golden/ from the REFERENCE itself (oracle/_ref, built from
/root/reference by oracle/Makefile). Run here, where /root/reference exists:

    python -m oracle.gen_golden

Outputs (committed, small):
  tests/golden/small_*.wrtb     WRTRACEB files written by trace_io::save_trace_binary
  tests/golden/golden.json      per trace: record count, contributions, sha256
                                of the reference's WRTRACEB bytes and of its
                                oracle_sum (f64, densified, + touched mask), and
                                per (policy, threshold) the reference's request /
                                instruction / fp-add counts and the sha256 of
                                its per-address sums.
  tests/golden/records.json     single-record request streams (apply_policy)
                                for random convergent / divergent records.
  tests/golden/criterion1.json  the first CRIT1_TRACES traces of the
                                reference's acceptance criterion 1 (its own
                                mt19937_64 draw sequence, acceptance.cpp:93-146):
                                spec, and per (policy, threshold) drawn the
                                reference's request count and sums sha256.
The BASELINE trace family (C1..C4) is recorded by hash only.
"""
from __future__ import annotations

import hashlib
import json
import os
import random
import tempfile

import numpy as np

from .bindings import NATIVE, SW_B, SW_S, CCCL, Ref, build, scene

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "tests", "golden")

# (name, SceneSpec kwargs, store-file?)
SMALL = [
    ("small_default", {}, True),
    ("small_conservation_911", dict(num_primitives=200, params_per_primitive=3, image_width=64,
                                    image_height=32, locality=0.9, activity_prob=0.7, seed=911),
     True),
    ("small_fullrange_414", dict(num_primitives=100, params_per_primitive=2, image_width=32,
                                 image_height=32, locality=0.9, activity_prob=0.8,
                                 quantized_values=0, seed=414), True),
    ("small_n9_divergent", dict(num_primitives=300, params_per_primitive=9, image_width=64,
                                image_height=64, mean_fragment_span=24, fragments_per_pixel_mean=2,
                                locality=0.6, activity_prob=0.5, seed=7), True),
    ("small_n1_lowact", dict(num_primitives=50, params_per_primitive=1, image_width=40,
                             image_height=24, fragments_per_pixel_mean=1.5, locality=0.8,
                             activity_prob=0.3, seed=3301), True),
    ("small_n5_generic", dict(num_primitives=120, params_per_primitive=5, image_width=48,
                              image_height=32, fragments_per_pixel_mean=2.0, locality=0.7,
                              activity_prob=0.6, seed=55), True),
]
# BASELINE trace family T: hashes only.
FAMILY_T = [
    ("C1", dict(num_primitives=10_000, params_per_primitive=9, image_width=256, image_height=256,
                mean_fragment_span=48, fragments_per_pixel_mean=8, locality=0.99,
                activity_prob=0.7, seed=1)),
    ("C2", dict(num_primitives=100_000, params_per_primitive=9, image_width=800, image_height=800,
                mean_fragment_span=48, fragments_per_pixel_mean=8, locality=0.99,
                activity_prob=0.7, seed=1)),
    ("C3", dict(num_primitives=1_000_000, params_per_primitive=9, image_width=1920,
                image_height=1080, mean_fragment_span=48, fragments_per_pixel_mean=8,
                locality=0.99, activity_prob=0.7, seed=1)),
    ("C4", dict(num_primitives=200_000, params_per_primitive=9, image_width=1920,
                image_height=1080, mean_fragment_span=4096, fragments_per_pixel_mean=8,
                locality=1.0, activity_prob=0.9, seed=1)),
]
THRESHOLDS = [0, 1, 8, 16, 24, 32, 33]
CRIT1_TRACES = 200


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def file_sha(path: str) -> str:
    with open(path, "rb") as f:
        return hashlib.sha256(f.read()).hexdigest()


def describe(ref: Ref, h, P: int, policies=True, thresholds=THRESHOLDS) -> dict:
    tr = ref.to_numpy(h)
    sums, touched = ref.oracle_sum(h, P)
    d = {"records": tr.num_records, "contributions": tr.contributions(),
         "oracle_sum_sha256": sha(sums), "touched_sha256": sha(touched.astype(np.uint8)),
         "oracle_abs_sum": float(np.abs(sums).sum()), "policies": {}}
    if policies:
        for kind, name in ((NATIVE, "native"), (SW_S, "sw_s"), (SW_B, "sw_b"), (CCCL, "cccl")):
            for t in (thresholds if kind in (SW_S, SW_B) else [0]):
                s, c = ref.apply_policy(h, kind, t, P)
                d["policies"][f"{name}:{t}"] = dict(c, sums_sha256=sha(s))
    return d


def main() -> None:
    build(ref=True)
    ref = Ref()
    os.makedirs(OUT, exist_ok=True)
    golden = {"generated_by": "oracle/gen_golden.py from /root/reference (warpred) built by "
                              "oracle/Makefile", "small": {}, "family_t": {}}
    for name, kw, store in SMALL:
        spec = scene(**kw)
        h = ref.generate(spec)
        path = os.path.join(OUT, name + ".wrtb")
        ref.save_binary(h, path)
        golden["small"][name] = dict(spec=kw, file=os.path.basename(path),
                                     wrtraceb_sha256=file_sha(path),
                                     **describe(ref, h, spec.num_primitives))
        ref.free(h)
    with tempfile.TemporaryDirectory() as td:
        for name, kw in FAMILY_T:
            spec = scene(**kw)
            h = ref.generate(spec)
            path = os.path.join(td, name + ".wrtb")
            ref.save_binary(h, path)
            golden["family_t"][name] = dict(
                spec=kw, wrtraceb_sha256=file_sha(path),
                **describe(ref, h, spec.num_primitives, thresholds=[0, 16, 33]))
            ref.free(h)
            print(name, golden["family_t"][name]["records"])
    with open(os.path.join(OUT, "golden.json"), "w") as f:
        json.dump(golden, f, indent=1, sort_keys=True)

    # single-record request streams
    rng = random.Random(2024)
    recs = []
    for i in range(48):
        n = rng.choice([1, 2, 3, 4, 9])
        convergent = i % 2 == 0
        active = rng.getrandbits(32) if i % 7 else 0xFFFFFFFF
        base = rng.randrange(16)
        prim = [base if convergent else rng.randrange(6) for _ in range(32)]
        if i % 11 == 0:
            prim[rng.randrange(32)] = -1
        grads = [0.0] * (32 * n)
        for l in range(32):
            if active >> l & 1:
                for p in range(n):
                    grads[l * n + p] = (1 + rng.randrange(255)) / 256.0 if i % 3 else \
                        rng.uniform(-1, 1)
        for kind in (NATIVE, SW_S, SW_B, CCCL):
            for t in ([0, 5, 16, 32, 33] if kind in (SW_S, SW_B) else [0]):
                reqs, ins, fp = ref.record_policy(active, prim, grads, kind, t)
                recs.append(dict(active=active, prim=prim, grads=grads, n=n, kind=kind,
                                 threshold=t, requests=reqs, instructions=ins, fp_adds=fp))
    with open(os.path.join(OUT, "records.json"), "w") as f:
        json.dump(recs, f)
    write_criterion1(ref)
    print("wrote", OUT)


def write_criterion1(ref: Ref) -> None:
    traces = []
    for spec_kw, thr in ref.criterion1_draws(CRIT1_TRACES):
        spec = scene(**spec_kw)
        h = ref.generate(spec)
        P = spec.num_primitives
        sums, _ = ref.oracle_sum(h, P)
        runs = {}
        # per preset, the acceptance loop runs native, sw_s, sw_b, cccl (and
        # hw_atomred, which has no core policy); thresholds as drawn
        for ss, sb in thr:
            for kind, name, t in ((NATIVE, "native", 0), (SW_S, "sw_s", ss), (SW_B, "sw_b", sb),
                                  (CCCL, "cccl", 0)):
                key = f"{name}:{t}"
                if key in runs:
                    continue
                s, c = ref.apply_policy(h, kind, t, P)
                runs[key] = {"requests": c["requests"], "sums_sha256": sha(s)}
        traces.append({"spec": spec_kw, "records": ref.to_numpy(h).num_records,
                       "oracle_sum_sha256": sha(sums), "runs": runs})
        ref.free(h)
    with open(os.path.join(OUT, "criterion1.json"), "w") as f:
        json.dump({"generated_by": "oracle/gen_golden.py (reference acceptance criterion-1 draws)",
                   "traces": traces}, f, indent=0, sort_keys=True)


if __name__ == "__main__":
    main()
