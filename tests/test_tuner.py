"""Online threshold re-tuning; mirrors the reference's tuner
tests (proj/tests/test_tuner.cpp: flat sweep ties low, argmin dominates the
endpoints) with an injected cost, plus the re-profiling period."""
import pytest

from paper_2401_05345_b200.rasterizer import ThresholdTuner
from paper_2401_05345_b200.warpred import PolicyKind


def test_flat_sweep_ties_to_lowest():  # test_tuner.cpp:31-47
    tu = ThresholdTuner(period=10, timer=lambda t: 1.0)
    assert tu.policy().threshold == 0


def test_interior_argmin_and_endpoints():  # test_tuner.cpp:70-89
    cost = {t: (t - 11) ** 2 + 5.0 for t in range(33)}
    tu = ThresholdTuner(period=10, timer=cost.__getitem__)
    p = tu.policy()
    assert p.kind == PolicyKind.sw_b and p.threshold == 11
    _, chosen, sweep = tu.history[0]
    assert sweep[chosen] <= sweep[0] and sweep[chosen] <= sweep[32]


def test_reprofiles_every_period():
    calls = []

    def timer(t):
        calls.append(t)
        return float(t == 3 if len(calls) <= 33 else t != 20)  # optimum moves 0 -> 20

    tu = ThresholdTuner(period=4, timer=timer)
    got = [tu.policy().threshold for _ in range(9)]
    assert got[:4] == [0] * 4 and got[4:8] == [20] * 4 and len(tu.history) == 3
    assert [h[0] for h in tu.history] == [0, 4, 8]
    assert len(calls) == 3 * 33


def test_validation():
    with pytest.raises(ValueError):
        ThresholdTuner(period=0)
    with pytest.raises(ValueError):
        ThresholdTuner(kind=PolicyKind.native)


@pytest.mark.gpu
def test_cuda_timer_on_device(cuda):
    import torch

    from paper_2401_05345_b200.rasterizer import GaussianRasterizer
    from paper_2401_05345_b200.scene import make_camera, make_dL_dpixels, make_scene

    sc = {k: torch.from_numpy(v).to(cuda) for k, v in make_scene(20_000, 320, 240, seed=1).items()}
    r = GaussianRasterizer()
    r.render_forward(sc["means3D"], sc["scales"], sc["rotations"], sc["opacities"], sc["colors"],
                     make_camera(320, 240))
    dL = torch.from_numpy(make_dL_dpixels(320, 240)).to(cuda)
    tu = ThresholdTuner(period=2000)
    p = tu.policy(r, dL)
    assert 0 <= p.threshold <= 32 and len(tu.history[0][2]) == 33
    assert tu.policy(r, dL).threshold == p.threshold and len(tu.history) == 1
