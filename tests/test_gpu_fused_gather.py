"""Fused slab gather: the final pass of each slab stores straight into the output volume.

DESIGN.md 7 explains the design. The output volume can be another buffer on the same GPU, a peer GPU's
memory, or another process's allocation mapped through CUDA IPC. Everything here runs on one GPU. That
GPU stands in for the gathering GPU; it does not stand in for extra ranks. No kernel waits on another.
"""
import os
import subprocess
import sys

import numpy as np
import pytest

import paper_1104_5243_b200 as bp
from oracle import oracle as O
from tests.helpers import baseline_small, bitwise_equal

pytestmark = pytest.mark.gpu


def _torch_cuda():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch


@pytest.mark.parametrize("view_batch", [5, 32])
def test_output_volume_streaming_two_slabs(view_batch):
    torch = _torch_cuda()
    px, mats = baseline_small(n_views=23, shrink=8)
    n, isy, isx = px.shape
    L = 48
    ref, _ = O.reconstruct(px, mats, L)
    full = torch.full((L, L, L), float("nan"), dtype=torch.float32, device="cuda")
    bounds = bp.partition_slabs(mats, isx, isy, L, 2)
    for s in range(2):
        z0, z1 = int(bounds[s]), int(bounds[s + 1])
        with bp.GpuContext(L, isx, isy, z_begin=z0, z_end=z1, view_batch=view_batch,
                           output_volume=full.data_ptr() + 4 * z0 * L * L) as ctx:
            for k in range(n):
                ctx.backproject(px[k], mats[k])
            ctx.finish(readback=False)
    torch.cuda.synchronize()
    assert bitwise_equal(full.cpu().numpy(), ref)


def test_output_volume_with_readback_and_resident():
    torch = _torch_cuda()
    px, mats = baseline_small(n_views=20, shrink=8)
    n, isy, isx = px.shape
    L = 32
    ref, _ = O.reconstruct(px, mats, L)
    out = torch.zeros((L, L, L), dtype=torch.float32, device="cuda")
    with bp.GpuContext(L, isx, isy, view_batch=8, output_volume=out.data_ptr()) as ctx:
        for k in range(n):
            ctx.backproject(px[k], mats[k])
        host, _ = ctx.finish()            # read back from the output volume
        assert bitwise_equal(host, ref)
        ctx.upload_views(px, mats)        # resident path: last batch of each pass stores to `out`
        out.zero_()
        torch.cuda.synchronize()
        ctx.time_resident(2)
    torch.cuda.synchronize()
    assert bitwise_equal(out.cpu().numpy(), ref)


def test_ipc_fused_gather_across_processes(tmp_path):
    torch = _torch_cuda()
    px, mats = baseline_small(n_views=12, shrink=8)
    n, isy, isx = px.shape
    L = 32
    ref, _ = O.reconstruct(px, mats, L)
    path = str(tmp_path / "stack.npz")
    np.savez(path, pixels=px, mats=mats)
    # a small allocation first, so that `full` sits at a nonzero offset inside the caching
    # allocator's segment (IPC maps whole allocations; the token carries the offset)
    pad = torch.zeros(1000, dtype=torch.float32, device="cuda")
    full = torch.full((L, L, L), float("nan"), dtype=torch.float32, device="cuda")
    torch.cuda.synchronize()
    handle = bp.ipc_handle(full.data_ptr())
    assert int.from_bytes(handle[64:], "little") > 0
    bounds = bp.partition_slabs(mats, isx, isy, L, 2)
    z0, z1 = int(bounds[0]), int(bounds[1])
    # the other "rank": a separate process maps this process's volume and writes slab 1
    repo = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, PYTHONPATH=repo + os.pathsep + os.environ.get("PYTHONPATH", ""))
    r = subprocess.run([sys.executable, os.path.join(repo, "tests", "ipc_child.py"), handle.hex(),
                        str(L), str(z1), str(L), path], capture_output=True, text=True, env=env,
                       timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]
    # this process writes slab 0 into its own volume
    with bp.GpuContext(L, isx, isy, z_begin=z0, z_end=z1,
                       output_volume=full.data_ptr() + 4 * z0 * L * L) as ctx:
        for k in range(n):
            ctx.backproject(px[k], mats[k])
        ctx.finish(readback=False)
    torch.cuda.synchronize()
    assert bitwise_equal(full.cpu().numpy(), ref)
    assert not pad.any()  # nothing landed outside the slab ranges
