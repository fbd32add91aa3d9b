"""CPU, world_size 2 over gloo: the view-parallel backward + gradient
all-reduce equals the single-process sum over all views (the oracle's CPU
backward stands in for the per-rank GPU backward)."""
import ctypes as C
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2401_05345_b200.dist import shard_views


def test_shard_views_partition():
    for n in (1, 5, 8, 64, 67):
        for w in (1, 2, 3, 8):
            ids = [i for r in range(w) for i in shard_views(n, w, r)]
            assert ids == list(range(n))
            sizes = [len(shard_views(n, w, r)) for r in range(w)]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        shard_views(4, 2, 2)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _views():
    from paper_2401_05345_b200.scene import orbit_cameras

    return orbit_cameras(64, 48, 5)


def _backward_fn(orc, sc):
    from oracle.bindings import Camera as OCam
    from paper_2401_05345_b200.scene import make_dL_dpixels

    def run(cam, grad):
        oc = OCam()
        cc = cam.to_c()
        C.memmove(C.byref(oc), C.byref(cc), C.sizeof(oc))
        seed = int(round((cam.viewmatrix[0, 2] + 1) * 1000))
        out = orc.gs_render(sc, oc, make_dL_dpixels(64, 48, seed=seed))
        grad += torch.from_numpy(out["grad"])

    return run


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle.bindings import Oracle
    from paper_2401_05345_b200.dist import view_parallel_backward
    from paper_2401_05345_b200.scene import make_scene

    sc = make_scene(300, 64, 48, seed=3)
    grad = torch.zeros((300, 9), dtype=torch.float64)
    view_parallel_backward(_backward_fn(Oracle(), sc), _views(), grad)
    out[rank] = grad.numpy().copy()
    dist.destroy_process_group()


def test_two_rank_allreduce_equals_single_process(orc):
    from paper_2401_05345_b200.scene import make_scene

    sc = make_scene(300, 64, 48, seed=3)
    want = torch.zeros((300, 9), dtype=torch.float64)
    fn = _backward_fn(orc, sc)
    for cam in _views():
        fn(cam, want)
    mgr = mp.Manager()
    out = mgr.dict()
    mp.start_processes(_worker, args=(2, _free_port(), out), nprocs=2, start_method="spawn")
    for r in (0, 1):
        np.testing.assert_allclose(out[r], want.numpy(), rtol=1e-12, atol=1e-12)


def _train_fns(orc, sc, params, state):
    """CPU oracle stand-ins for the per-rank GPU training step: the view's
    2D + 3D backward (gs_train_grads) and a float64 Adam on the replica."""
    from oracle.bindings import Camera as OCam, gs_adam, gs_train_grads
    from paper_2401_05345_b200.scene import make_dL_dpixels

    def grads_view(cam, grad3d):
        oc = OCam()
        cc = cam.to_c()
        C.memmove(C.byref(oc), C.byref(cc), C.sizeof(oc))
        seed = int(round((cam.viewmatrix[0, 2] + 1) * 1000))
        _, g3 = gs_train_grads(orc, sc, oc, make_dL_dpixels(64, 48, seed=seed), threads=2)
        grad3d += torch.from_numpy(g3)

    def update(grad3d):
        state["step"] += 1
        g = grad3d.numpy()
        gs_adam(orc, params, np.ascontiguousarray(g.reshape(-1)), state["m"], state["v"], 1e-3,
                0.9, 0.999, 1e-8, state["step"])

    return grads_view, update


def _train_worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle.bindings import Oracle
    from paper_2401_05345_b200.dist import view_parallel_train_step
    from paper_2401_05345_b200.scene import make_scene

    sc = make_scene(300, 64, 48, seed=3)
    params = np.zeros(300 * 14, np.float64)
    state = {"step": 0, "m": np.zeros_like(params), "v": np.zeros_like(params)}
    grads_view, update = _train_fns(Oracle(), sc, params, state)
    grad3d = torch.zeros((300, 14), dtype=torch.float64)
    view_parallel_train_step(grads_view, _views(), grad3d, update)
    out[rank] = (grad3d.numpy().copy(), params.copy())
    dist.destroy_process_group()


def test_two_rank_train_step_equals_single_process(orc):
    """World size 2 over gloo: the summed 3D gradients (per-view preprocess
    backward before the one all-reduce) and the replicas after the optimizer
    step equal the single-process step over all views, on both ranks."""
    from paper_2401_05345_b200.dist import view_parallel_train_step
    from paper_2401_05345_b200.scene import make_scene

    sc = make_scene(300, 64, 48, seed=3)
    params = np.zeros(300 * 14, np.float64)
    state = {"step": 0, "m": np.zeros_like(params), "v": np.zeros_like(params)}
    grads_view, update = _train_fns(orc, sc, params, state)
    want_g = torch.zeros((300, 14), dtype=torch.float64)
    view_parallel_train_step(grads_view, _views(), want_g, update)
    mgr = mp.Manager()
    out = mgr.dict()
    mp.start_processes(_train_worker, args=(2, _free_port(), out), nprocs=2, start_method="spawn")
    for r in (0, 1):
        g, p = out[r]
        np.testing.assert_allclose(g, want_g.numpy(), rtol=1e-12, atol=1e-12)
        np.testing.assert_allclose(p, params, rtol=1e-12, atol=1e-15)
