"""CPU: the C oracle restatement pinned against the reference.

1. The reference's own known-answer tests for the hot path
   (proj/tests/test_reducers.cpp) restated against oracle/liboracle.so.
2. tests/golden/ (written by the reference itself, oracle/gen_golden.py):
   WRTRACEB bytes, oracle sums and per-policy request / instruction / fp-add
   counts must match hash for hash.
3. When oracle/_ref is built (this container), randomised differential tests
   against the reference library directly.
"""
import hashlib
import json
import os
import random
import tempfile

import numpy as np
import pytest

from conftest import GOLDEN

NATIVE, SW_S, SW_B, CCCL, HW = 0, 1, 2, 3, 4


def grid(rng):  # test_reducers.cpp:27-29
    return (1 + rng.randrange(255)) / 256.0


def rec(active, n, prim=None):
    return active, np.array(prim if prim is not None else [-1] * 32, np.int32), np.zeros(32 * n)


def tree_sum(g, n, p):  # test_reducers.cpp:52-66
    v = [g[l * n + p] for l in range(32)]
    off = 16
    while off >= 1:
        nxt = list(v)
        for i in range(32 - off):
            nxt[i] = v[i] + v[i + off]
        for i in range(32 - off, 32):
            nxt[i] = v[i] + v[i]
        v = nxt
        off //= 2
    return v[0]


def sum_requests(reqs):
    out = {}
    for prim, param, val in reqs:
        out[(prim, param)] = out.get((prim, param), 0.0) + val
    return out


def test_native_known_answers(orc):  # test_reducers.cpp:70-100
    rng = random.Random(3)
    a, prim, g = rec(0xFFFFFFFF, 3, [5] * 32)
    for i in range(96):
        g[i] = grid(rng)
    reqs, ins, fp = orc.record_policy(a, prim, g, NATIVE, 0)
    assert len(reqs) == 96 and ins == 96 and fp == 0
    assert orc.record_policy(0, prim, np.zeros(96), NATIVE, 0)[0] == []
    prim = np.full(32, -1, np.int32)
    prim[0], prim[2] = 4, 9
    g = np.zeros(64)
    g[0], g[1], g[4], g[5] = 0.5, 0.25, 0.125, 0.75
    reqs, _, _ = orc.record_policy(0b101, prim, g, NATIVE, 0)
    assert reqs == [(4, 0, 0.5), (4, 1, 0.25), (9, 0, 0.125), (9, 1, 0.75)]


def test_serial_full_warp(orc):  # :102-120
    rng = random.Random(11)
    g = np.array([grid(rng) for _ in range(96)])
    reqs, _, fp = orc.record_policy(0xFFFFFFFF, [42] * 32, g, SW_S, 16)
    assert len(reqs) == 3
    for p in range(3):
        expect = 0.0
        for l in range(32):
            expect += g[l * 3 + p]
        assert reqs[p] == (42, p, expect)
    assert fp == 31 * 3


def test_serial_below_threshold_falls_back(orc):  # :122-140
    rng = random.Random(12)
    g = np.zeros(64)
    for l in range(5):
        for p in range(2):
            g[l * 2 + p] = grid(rng)
    reqs, _, fp = orc.record_policy(0b11111, [8] * 32, g, SW_S, 8)
    assert len(reqs) == 10 and fp == 0
    assert reqs == [(8, p, g[l * 2 + p]) for l in range(5) for p in range(2)]


def _random_record(rng, n, num_prims, convergent):  # :31-43
    active = rng.getrandbits(32)
    base = rng.randrange(num_prims)
    prim = [base if convergent else rng.randrange(num_prims) for _ in range(32)]
    g = np.zeros(32 * n)
    for l in range(32):
        if active >> l & 1:
            for p in range(n):
                g[l * n + p] = grid(rng)
    return active, prim, g


def test_serial_threshold_0_is_1_and_33_is_native(orc):  # :142-172
    rng = random.Random(13)
    for _ in range(50):
        a, prim, g = _random_record(rng, 2, 16, False)
        r0, i0, _ = orc.record_policy(a, prim, g, SW_S, 0)
        r1, i1, _ = orc.record_policy(a, prim, g, SW_S, 1)
        assert r0 == r1 and i0 == i1
        groups = {prim[l] for l in range(32) if a >> l & 1}
        assert len(r0) == 2 * len(groups)
    for _ in range(50):
        a, prim, g = _random_record(rng, 3, 8, False)
        s, _, fp = orc.record_policy(a, prim, g, SW_S, 33)
        nat, _, _ = orc.record_policy(a, prim, g, NATIVE, 0)
        assert sum_requests(s) == sum_requests(nat) and len(s) == len(nat) and fp == 0


def test_bfly_known_answers(orc):  # :174-227
    rng = random.Random(15)
    g = np.array([grid(rng) for _ in range(96)])
    reqs, _, fp = orc.record_policy(0xFFFFFFFF, [5] * 32, g, SW_B, 16)
    assert len(reqs) == 3 and fp == 32 * 5 * 3
    for p in range(3):
        assert reqs[p] == (5, p, tree_sum(g, 3, p)) == (5, p, sum(g[l * 3 + p] for l in range(32)))
    g = np.zeros(64)
    for l in range(10):
        g[2 * l], g[2 * l + 1] = grid(rng), grid(rng)
    reqs, _, fp = orc.record_policy(0x3FF, [9] * 32, g, SW_B, 16)
    assert len(reqs) == 20 and fp == 0
    prim = [3] * 32
    prim[17] = 4
    for t in (0, 16, 32):
        assert len(orc.record_policy(0xFFFFFFFF, prim, np.full(32, 0.5), SW_B, t)[0]) == 32
    for t in (0, 1, 16):
        assert orc.record_policy(0, [1] * 32, np.zeros(64), SW_B, t)[0] == []


def test_cccl_accounting(orc):  # :229-268
    rng = random.Random(17)
    g = np.array([grid(rng) for _ in range(96)])
    c, ci, _ = orc.record_policy(0xFFFFFFFF, [2] * 32, g, CCCL, 0)
    b, bi, _ = orc.record_policy(0xFFFFFFFF, [2] * 32, g, SW_B, 0)
    assert len(c) == 3 and sum_requests(c) == sum_requests(b)
    assert ci == 3 * (4 + 5 + 1) and bi == 4 + 15 + 3 and ci > bi
    rng = random.Random(18)
    for trial in range(50):
        a, prim, g = _random_record(rng, 1, 4, trial % 2 == 0)
        assert orc.record_policy(a, prim, g, CCCL, 0)[0] == orc.record_policy(a, prim, g, SW_B, 0)[0]


def test_request_count_monotone_in_threshold(orc):  # :342-359
    rng = random.Random(20)
    for trial in range(100):
        a, prim, g = _random_record(rng, 2, 6, trial % 3 == 0)
        prev = [0, 0]
        for t in range(33):
            cur = [len(orc.record_policy(a, prim, g, k, t)[0]) for k in (SW_S, SW_B)]
            if t:
                assert cur[0] >= prev[0] and cur[1] >= prev[1]
            prev = cur


def test_eligible_groups_emit_n(orc):  # :361-373
    rng = random.Random(23)
    for k in (1, 2, 7, 19, 32):
        a = 0xFFFFFFFF if k == 32 else (1 << k) - 1
        g = np.zeros(128)
        for l in range(k):
            for p in range(4):
                g[l * 4 + p] = grid(rng)
        assert len(orc.record_policy(a, [6] * 32, g, SW_S, k)[0]) == 4
        if k == 32:
            assert len(orc.record_policy(a, [6] * 32, g, SW_B, 32)[0]) == 4


def test_threshold_validation_and_hw_atomred(orc):  # :375-380, reducers.cpp:232-236
    for kind, t in ((SW_S, -1), (SW_S, 34), (SW_B, 34)):
        with pytest.raises(RuntimeError, match="threshold"):
            orc.record_policy(1, [0] * 32, np.zeros(32), kind, t)
    with pytest.raises(RuntimeError, match="hw_atomred"):
        orc.record_policy(1, [0] * 32, np.zeros(32), HW, 0)


def test_oracle_sum_known_answer_and_conservation(orc):  # :270-312
    from oracle.bindings import Trace, scene

    one = Trace(scene(params_per_primitive=2), np.zeros(1, np.int32), np.zeros(1, np.int32),
                np.array([1], np.uint32), np.array([7] * 32, np.int32),
                np.array([0.5, 0.25] + [0.0] * 62))
    sums, touched = orc.oracle_sum(one, 10)
    assert sums[14] == 0.5 and sums[15] == 0.25 and touched.sum() == 2
    spec = scene(num_primitives=200, params_per_primitive=3, image_width=64, image_height=32,
                 locality=0.9, activity_prob=0.7, seed=911)
    tr = orc.generate(spec)
    want, _ = orc.oracle_sum(tr, 200)
    for kind in (NATIVE, SW_S, SW_B, CCCL):
        for t in ((0, 8, 16, 24, 32) if kind in (SW_S, SW_B) else (0,)):
            s, _ = orc.apply_policy(tr, kind, t, 200)
            assert np.array_equal(s, want)


def test_full_range_conservation_1e6(orc):  # :314-340
    from oracle.bindings import scene

    spec = scene(num_primitives=100, params_per_primitive=2, image_width=32, image_height=32,
                 locality=0.9, activity_prob=0.8, quantized_values=0, seed=414)
    tr = orc.generate(spec)
    want, _ = orc.oracle_sum(tr, 100)
    for kind in (SW_S, SW_B):
        s, _ = orc.apply_policy(tr, kind, 8, 100)
        assert np.all(np.abs(s - want) <= 1e-6 * np.maximum(1.0, np.abs(want)))


def _sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def _golden():
    return json.load(open(os.path.join(GOLDEN, "golden.json")))


@pytest.mark.parametrize("name", sorted(_golden()["small"]))
def test_golden_small_traces(orc, name):
    from oracle.bindings import scene

    g = _golden()["small"][name]
    path = os.path.join(GOLDEN, g["file"])
    assert hashlib.sha256(open(path, "rb").read()).hexdigest() == g["wrtraceb_sha256"]
    # the restated generator writes the same bytes as the reference
    tr = orc.generate(scene(**g["spec"]))
    with tempfile.TemporaryDirectory() as td:
        p2 = os.path.join(td, "t.wrtb")
        orc.save_binary(tr, p2)
        assert hashlib.sha256(open(p2, "rb").read()).hexdigest() == g["wrtraceb_sha256"]
    loaded = orc.load_binary(path)
    P = loaded.spec.num_primitives
    assert loaded.num_records == g["records"] and loaded.contributions() == g["contributions"]
    sums, touched = orc.oracle_sum(loaded, P)
    assert _sha(sums) == g["oracle_sum_sha256"]
    assert _sha(touched.astype(np.uint8)) == g["touched_sha256"]
    for key, c in g["policies"].items():
        name_, t = key.split(":")
        kind = {"native": NATIVE, "sw_s": SW_S, "sw_b": SW_B, "cccl": CCCL}[name_]
        s, cnt = orc.apply_policy(loaded, kind, int(t), P)
        assert cnt == {k: c[k] for k in ("requests", "instructions", "fp_adds")}, key
        assert _sha(s) == c["sums_sha256"], key


def test_golden_records(orc):
    recs = json.load(open(os.path.join(GOLDEN, "records.json")))
    for r in recs:
        reqs, ins, fp = orc.record_policy(r["active"], r["prim"], r["grads"], r["kind"],
                                          r["threshold"])
        assert [list(x) for x in reqs] == r["requests"]
        assert ins == r["instructions"] and fp == r["fp_adds"]


@pytest.mark.parametrize("name", ["C1", "C2"])
def test_golden_family_t(orc, name):
    """BASELINE-size traces: byte-identical generation and equal oracle/policy
    results to what the reference produced (hash-pinned)."""
    from oracle.bindings import scene

    g = _golden()["family_t"][name]
    tr = orc.generate(scene(**g["spec"]))
    with tempfile.TemporaryDirectory() as td:
        p = os.path.join(td, "t.wrtb")
        orc.save_binary(tr, p)
        assert hashlib.sha256(open(p, "rb").read()).hexdigest() == g["wrtraceb_sha256"]
    P = g["spec"]["num_primitives"]
    sums, _ = orc.oracle_sum(tr, P)
    assert _sha(sums) == g["oracle_sum_sha256"]
    s, cnt = orc.apply_policy(tr, SW_B, 16, P)
    assert cnt["requests"] == g["policies"]["sw_b:16"]["requests"]
    assert _sha(s) == g["policies"]["sw_b:16"]["sums_sha256"]


@pytest.mark.ref
def test_random_differential_vs_reference(orc, ref):
    from oracle.bindings import scene

    mix = random.Random(20240801)  # the acceptance criterion-1 generator shape
    for _ in range(60):
        kw = dict(num_primitives=50 + mix.randrange(400), params_per_primitive=1 + mix.randrange(9),
                  image_width=32 + 8 * mix.randrange(5), image_height=16 + 4 * mix.randrange(5),
                  mean_fragment_span=8.0 + mix.randrange(48),
                  fragments_per_pixel_mean=1.0 + 0.25 * mix.randrange(5),
                  locality=0.5 + 0.5 * mix.randrange(101) / 100,
                  activity_prob=0.3 + 0.7 * mix.randrange(101) / 100,
                  quantized_values=mix.randrange(2), seed=mix.getrandbits(64))
        spec = scene(**kw)
        a = orc.generate(spec)
        h = ref.generate(spec)
        b = ref.to_numpy(h)
        for f in ("warp_id", "iteration", "active", "prim", "grads"):
            assert np.array_equal(getattr(a, f), getattr(b, f)), f
        P = spec.num_primitives
        assert np.array_equal(orc.oracle_sum(a, P)[0], ref.oracle_sum(h, P)[0])
        for kind in (NATIVE, SW_S, SW_B, CCCL):
            t = mix.randrange(34)
            x, cx = orc.apply_policy(a, kind, t, P)
            y, cy = ref.apply_policy(h, kind, t, P)
            assert np.array_equal(x, y) and cx == cy, (kw, kind, t)
        ref.free(h)


def test_criterion1_golden_against_restatement(orc):
    """The C restatement on the reference's own criterion-1 traces
    (tests/golden/criterion1.json, written by the reference from
    acceptance.cpp:93-146's draw sequence): oracle_sum and every drawn
    (policy, threshold) run -- request counts and per-address sums -- equal
    the reference's, hash for hash."""
    from oracle.bindings import scene

    g = json.load(open(os.path.join(GOLDEN, "criterion1.json")))["traces"]
    for i, rec in enumerate(g):
        tr = orc.generate(scene(**rec["spec"]))
        assert tr.num_records == rec["records"], i
        P = rec["spec"]["num_primitives"]
        sums, _ = orc.oracle_sum(tr, P)
        assert _sha(sums) == rec["oracle_sum_sha256"], i
        for key, want in rec["runs"].items():
            k, t = key.split(":")
            s, c = orc.apply_policy(tr, {"native": 0, "sw_s": 1, "sw_b": 2, "cccl": 3}[k], int(t), P)
            assert c["requests"] == want["requests"], (i, key)
            assert _sha(s) == want["sums_sha256"], (i, key)
