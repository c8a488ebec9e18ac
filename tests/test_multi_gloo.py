"""World-size-2 test of the multi-GPU host logic on CPU (gloo).

Mirrors what bench.py / a multi-rank deployment does per rank: identical
work-balanced partition on every rank (bp_partition_slabs), per-view row windows
(bp_slab_row_window) -- each rank only "receives" its window rows (all other rows
are zeroed here) -- per-rank slab reconstruction, then the single exchange step:
a gather of the slabs to rank 0.  The slab compute is the oracle (CPU) standing in
for the per-GPU kernel, whose slab/row-window parity is tested on the GPU in
tests/test_gpu_parity.py::test_slab_and_virtual_slabs_equal_full.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, L, out_path):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import paper_1104_5243_b200 as bp
    from oracle import oracle as O
    from tests.helpers import baseline_small

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    px, mats = baseline_small(n_views=12, shrink=8, seed=11)
    n, isy, isx = px.shape
    bounds = bp.partition_slabs(mats, isx, isy, L, world)
    # every rank must derive the same partition
    t = torch.tensor(bounds, dtype=torch.int64)
    all_b = [torch.zeros_like(t) for _ in range(world)]
    dist.all_gather(all_b, t)
    assert all(torch.equal(all_b[0], x) for x in all_b)
    z0, z1 = int(bounds[rank]), int(bounds[rank + 1])
    mine = px.copy()
    h2d_rows = 0
    for k in range(n):
        r0, r1 = bp.slab_row_window(mats[k], isy, L, z0, z1)
        mine[k, :r0] = 0.0
        mine[k, r1:] = 0.0
        h2d_rows += r1 - r0
    slab, _ = O.reconstruct(mine, mats, L, z0=z0, z1=z1, threads=2)
    # gather slabs (variable sizes) to rank 0
    if rank == 0:
        vol = np.zeros((L, L, L), np.float32)
        vol[z0:z1] = slab
        for src in range(1, world):
            a, b_ = int(bounds[src]), int(bounds[src + 1])
            buf = torch.empty((b_ - a, L, L), dtype=torch.float32)
            dist.recv(buf, src=src)
            vol[a:b_] = buf.numpy()
        ref, _ = O.reconstruct(px, mats, L, threads=2)
        ok = np.array_equal(vol.view(np.uint32), ref.view(np.uint32))
        np.save(out_path, np.array([int(ok), h2d_rows, n * isy]))
    else:
        dist.send(torch.from_numpy(slab), dst=0)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("L", [32, 40])
def test_two_rank_slab_gather_equals_single(tmp_path, L):
    out = str(tmp_path / "res.npy")
    mp.start_processes(_worker, args=(2, _free_port(), L, out), nprocs=2, join=True,
                       start_method="spawn")
    ok, rows, full_rows = np.load(out)
    assert ok == 1
    assert rows < full_rows  # rank 0 received only its row window
