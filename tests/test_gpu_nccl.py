"""The C ABI's communicator-aware calls (SURVEY §8(b) wr_gs_allreduce_grads)
on a one-rank NCCL process group in this process: dw_allreduce_grads reduces
in place on the caller's stream through the NCCL library torch loaded, and
dw_render_views_allreduce -- views, the all-reduce and the one D2H -- gives
the same gradient and images as dw_render_views_host. (Only one GPU is
available to the tests; the two-rank reduction itself is covered on CPU by
tests/test_dist_gloo.py.)"""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def nccl_world(cuda):
    import torch
    import torch.distributed as dist

    if dist.is_initialized():
        dist.destroy_process_group()
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0,
                            world_size=1, device_id=cuda)
    yield
    dist.destroy_process_group()


def test_allreduce_grads_one_rank(cuda, nccl_world):
    import torch

    from paper_2401_05345_b200.rasterizer import allreduce_grads, nccl_comm_ptr

    comm = nccl_comm_ptr()
    assert comm != 0
    g = torch.randn(1_000_003, device=cuda)
    want = g.clone()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    allreduce_grads(g, comm, stream=s)
    s.synchronize()
    assert torch.equal(g, want)  # the sum over one rank


def test_render_views_allreduce_matches_host_call(cuda, nccl_world):
    import torch

    from paper_2401_05345_b200 import warpred as wr
    from paper_2401_05345_b200.rasterizer import (GaussianRasterizer, nccl_comm_ptr,
                                                  render_views_allreduce, render_views_host)
    from paper_2401_05345_b200.scene import make_dL_dpixels, make_scene, orbit_cameras

    P, W, H, V = 20000, 320, 256, 4
    sc = make_scene(P, W, H, seed=9)
    cams = orbit_cameras(W, H, V)
    pin = {k: torch.from_numpy(v).pin_memory() for k, v in sc.items()}
    ptrs = [pin[k].data_ptr() for k in ("means3D", "scales", "rotations", "opacities", "colors")]
    dL = torch.from_numpy(np.stack([make_dL_dpixels(W, H, seed=20 + k) for k in range(V)]))
    dL = dL.float().pin_memory()
    pol = wr.Policy(wr.PolicyKind.sw_b, 16)
    out = {}
    for name in ("host", "allreduce"):
        img = torch.empty((V, 3, H, W)).pin_memory()
        grad = torch.empty((P, 9)).pin_memory()
        r = GaussianRasterizer()
        if name == "host":
            render_views_host(r, ptrs, P, cams, dL.data_ptr(), pol, img.data_ptr(),
                              grad.data_ptr())
        else:
            render_views_allreduce(r, ptrs, P, cams, dL.data_ptr(), pol, img.data_ptr(),
                                   grad.data_ptr(), nccl_comm_ptr())
        out[name] = (img.numpy().copy(), grad.numpy().astype(np.float64))
    assert np.array_equal(out["host"][0], out["allreduce"][0])
    a, b = out["host"][1], out["allreduce"][1]
    assert np.linalg.norm(a - b) <= 1e-6 * np.linalg.norm(a)  # RED summation order only


def test_allreduce_null_comm_is_invalid(cuda):
    import ctypes as C

    from paper_2401_05345_b200 import _lib

    rc = _lib.lib().dw_allreduce_grads(None, None, 0, None)
    assert rc == 1 and b"null" in _lib.lib().dw_last_error()
