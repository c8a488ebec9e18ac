"""Where do the computed-but-invisible updates of the 32x32x8 block cull come from, and how much of
them would block-uniform sub-block culls remove?  (CPU only, sampled voxels.)

For sampled views, every voxel (stride 2 in x, y, z) is projected; a voxel is visible when its
bilinear footprint touches the detector (clip_stats semantics).  A (block, view) pair is computed when
any of its voxels is visible.  Reported, as fractions of the visible updates: the waste of the
whole-block cull, and what remains with a cull per z-half, per z-line, per y-half, per xy-quadrant.
Usage: python tools/cull_waste.py [L] [views]"""
import sys
sys.path.insert(0, ".")
import numpy as np
import paper_1104_5243_b200 as bp

L = int(sys.argv[1]) if len(sys.argv) > 1 else 512
nv = int(sys.argv[2]) if len(sys.argv) > 2 else 31
isx, isy = 1248, 960
s = bp.Stack.baseline(n_views=496, isx=isx, isy=isy)
A = np.asarray(s.matrices, np.float64).reshape(-1, 12)[:: 496 // nv][:nv]
mm = 256.0 / L
c = ((np.arange(0, L, 2) - (L - 1) / 2) * mm).astype(np.float32)
n = len(c)
X = c[None, None, :]; Y = c[None, :, None]; Z = c[:, None, None]
tot = dict(vis=0, block=0, zhalf=0, zline=0, yhalf=0, quad=0)
bx = 16; bz = 4  # block 32x32x8 in sampled units
for a in A.astype(np.float32):
    w = a[2] * X + a[5] * Y + a[8] * Z + a[11]
    u = (a[0] * X + a[3] * Y + a[6] * Z + a[9]) / w
    v = (a[1] * X + a[4] * Y + a[7] * Z + a[10]) / w
    vis = (u > -1) & (u < isx) & (v > -1) & (v < isy)
    B = vis.reshape(n // bz, bz, n // bx, bx, n // bx, bx)  # zb, zi, yb, yi, xb, xi
    vox = bz * bx * bx
    tot["vis"] += int(vis.sum())
    tot["block"] += int(B.any(axis=(1, 3, 5)).sum()) * vox
    tot["zhalf"] += int(B.reshape(n // bz, 2, bz // 2, n // bx, bx, n // bx, bx).any(axis=(2, 4, 6)).sum()) * vox // 2
    tot["zline"] += int(B.any(axis=(3, 5)).sum()) * vox // bz
    tot["yhalf"] += int(B.reshape(n // bz, bz, n // bx, 2, bx // 2, n // bx, bx).any(axis=(1, 4, 6)).sum()) * vox // 2
    tot["quad"] += int(B.reshape(n // bz, bz, n // bx, 2, bx // 2, n // bx, 2, bx // 2).any(axis=(1, 4, 7)).sum()) * vox // 4
v = tot["vis"]
print(f"L={L}, {nv} views, voxels sampled at stride 2: visible fraction of nominal {v / (nv * n ** 3):.3f}")
for k in ("block", "zhalf", "zline", "yhalf", "quad"):
    print(f"  cull per {k:6s}: computed / visible = {tot[k] / v:.4f}")
