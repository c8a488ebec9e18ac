"""Child process of tests/test_gpu_fused_gather.py: maps the parent's full volume through CUDA IPC and
backprojects one z-slab whose final pass stores straight into it. This is the fused slab gather of
bench.py at N > 1, on one GPU.

Args: handle_hex L z0 z1 npz_path
"""
import sys

import numpy as np

import paper_1104_5243_b200 as bp


def main():
    handle = bytes.fromhex(sys.argv[1])
    L, z0, z1 = int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
    g = np.load(sys.argv[5])
    px, mats = g["pixels"], g["mats"]
    n, isy, isx = px.shape
    base = bp.ipc_open(handle)
    try:
        with bp.GpuContext(L, isx, isy, z_begin=z0, z_end=z1,
                           output_volume=base + 4 * z0 * L * L) as ctx:
            for k in range(n):
                ctx.backproject(px[k], mats[k])
            ctx.finish(readback=False)
    finally:
        bp.ipc_close(base)
    print("ok")


if __name__ == "__main__":
    main()
