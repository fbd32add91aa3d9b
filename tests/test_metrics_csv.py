"""the metrics.csv this repo writes from measured ncu counters
(tools/metrics_csv.py, reference layout experiment.cpp:376-378 /
hwsim.cpp:515-527) is accepted by the REFERENCE's own reader,
experiment::read_metrics_csv (experiment.cpp:319-336, via oracle/_ref), row
for row and value for value."""
import csv
import glob
import os
import subprocess
import sys

import pytest

from conftest import REF_AVAILABLE, ROOT

pytestmark = pytest.mark.ref

SWEEP = os.path.join(ROOT, "profiles", "r01", "x2", "thr_sweep_csv")
POLICY = {"native": 0, "sw_s": 1, "sw_b": 2, "cccl": 3}


def _check(ref, path):
    rows = list(csv.reader(open(path)))
    assert rows[0][:3] == ["machine", "policy", "threshold"] and len(rows[0]) == 13
    got = ref.read_metrics_csv(path)
    assert len(got) == len(rows) - 1 > 0
    for want, (pol, thr, ints, energy, gs, e2e) in zip(rows[1:], got):
        assert pol == POLICY[want[1]]
        assert thr == (None if want[2] == "-" else int(want[2]))
        assert ints == [int(x) for x in want[3:10]]
        assert energy == pytest.approx(float(want[10]), rel=1e-12)
        assert gs == pytest.approx(float(want[11]), rel=1e-12)
        assert e2e == pytest.approx(float(want[12]), rel=1e-12)


def test_generated_metrics_csv_reads_back_in_reference(ref, tmp_path):
    if not REF_AVAILABLE:
        pytest.skip("oracle/_ref not built")
    files = sorted(glob.glob(os.path.join(SWEEP, "thr_sweep_*.csv")))
    assert files
    out = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "metrics_csv.py"), *files],
                         capture_output=True, text=True, check=True).stdout
    p = tmp_path / "metrics.csv"
    p.write_text(out)
    _check(ref, str(p))


def test_committed_metrics_csv_reads_back_in_reference(ref):
    if not REF_AVAILABLE:
        pytest.skip("oracle/_ref not built")
    _check(ref, os.path.join(ROOT, "profiles", "r01", "x2", "metrics.csv"))
