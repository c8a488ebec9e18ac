"""Generate the golden fixtures under tests/golden/ from the REFERENCE itself.

Runs the unmodified reference sources (compiled by oracle/Makefile into
oracle/_ref/libbackproject_ref.so from /root/reference/proj/src) on small seeded
inputs and stores inputs + outputs as .npz.  Run in the build container (where
/root/reference exists):  python tests/golden/make_golden.py
The fixtures travel with the repo; the GPU box never needs /root/reference.
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
from oracle import oracle as O  # noqa: E402


def save(name, **arrays):
    np.savez_compressed(os.path.join(HERE, name), **arrays)
    print("wrote", name, {k: v.shape for k, v in arrays.items()})


def main():
    R = O.ref()
    assert R is not None, "reference library not built (needs /root/reference)"
    # 1. reference datagen + reconstruction, small_stack geometry (test_support.hpp:104-109)
    px, mats = O.ref_make_stack("spheres3", 6, 64, 48, pitch=0.32 * 1248 / 64)
    vol, st = O.ref_reconstruct(px, mats, 16, threads=2, lanes=8, block_b=4, clip=True)
    save("recon_spheres3_16.npz", pixels=px, mats=mats, volume=vol,
         voxel_updates=np.array(st["voxel_updates"]))
    # 2. shell phantom at an odd edge length with a non-multiple-of-4 detector
    px, mats = O.ref_make_stack("shell", 8, 58, 46, pitch=0.32 * 1248 / 58)
    vol, _ = O.ref_reconstruct(px, mats, 23, threads=1)
    save("recon_shell_23.npz", pixels=px, mats=mats, volume=vol)
    # 3. BASELINE-shaped seeded stack (library datagen) through the reference
    import paper_1104_5243_b200 as bp
    s = bp.Stack.baseline(n_views=12, isx=156, isy=120, pitch_mm=0.32 * 8, seed=7)
    px, mats = s.pixels.copy(), s.matrices.copy()
    vol, _ = O.ref_reconstruct(px, mats, 32, threads=4, lanes=4, block_b=3)
    vol_off, _ = O.ref_reconstruct(px, mats, 32, offset=(60.0, 0.0, 0.0), threads=4)
    save("recon_baseline_32.npz", pixels=px, mats=mats, volume=vol, volume_offset60=vol_off)
    # 4. sampled lines at a larger grid (8c sampled-line oracle)
    ys = np.array([0, 17, 63, 100, 127], np.int32)
    zs = np.array([5, 64, 64, 90, 127], np.int32)
    lines = O.ref_reconstruct_lines(px, mats, 128, ys, zs)
    save("lines_baseline_128.npz", pixels=px, mats=mats, ys=ys, zs=zs, lines=lines)
    # 5. known-answer line (test_kernel.cpp:84-101): pixel-centre hits accumulate c*r^2
    g = O.Grid.cube(256)
    A = np.array([1, 0, 0, 0, 1, 0, 0, 0, 0, 127.5, 127.5 - (g.oz + 136 * g.MM), 1], np.float64)
    img = np.full((1, 32, 32), 0.8125, np.float32)
    line = O.ref_reconstruct_lines(img, A[None], 256, np.array([130], np.int32),
                                   np.array([136], np.int32))
    save("line_pixel_centre.npz", image=img, mats=A[None], line=line)
    # 6. clip statistics and the full per-line clip table (build_clip_table)
    tot = O.ref_clip_total(mats, 156, 120, 32)
    save("clip_baseline_32.npz", mats=mats, total=np.array(tot, np.uint64))
    ranges, tot2 = O.ref_clip_table(mats, 156, 120, 32)
    assert tot2 == tot
    save("clip_ranges_baseline_32.npz", mats=mats, ranges=ranges, total=np.array(tot, np.uint64))
    # 7. reciprocal ladder (recip.hpp:14-23): reconstructions in approx12 / approx12_nr
    px, mats = O.ref_make_stack("spheres3", 6, 64, 48, pitch=0.32 * 1248 / 64)
    v12, _ = O.ref_reconstruct(px, mats, 16, threads=2, recip=1)
    vnr, _ = O.ref_reconstruct(px, mats, 16, threads=2, recip=2)
    save("recon_recip_16.npz", pixels=px, mats=mats, approx12=v12, approx12_nr=vnr)


if __name__ == "__main__":
    main()
