"""Lower bound of the bench kernel's DRAM traffic per launch from its wave structure.

A wave of resident CTAs covers about one z-layer of 32x32x8 blocks (256 blocks at 512^3, 296 CTAs
resident).  Its CTAs walk the launch's views in step, so what the wave needs from L2 is, per view, the
band of pair rows its z-layer projects to.  If that working set (all views of the launch) exceeds the L2,
every wave re-reads its bands from DRAM: traffic >= sum over z-layers and views of the band bytes.
Usage: python tools/dram_floor.py [L] [views per launch]
"""
import sys
sys.path.insert(0, ".")
import numpy as np
import paper_1104_5243_b200 as bp

L = int(sys.argv[1]) if len(sys.argv) > 1 else 512
B = int(sys.argv[2]) if len(sys.argv) > 2 else 248
isx, isy = 1248, 960
s = bp.Stack.baseline(n_views=496, isx=isx, isy=isy)
A = np.asarray(s.matrices, np.float64).reshape(-1, 12)[:B]
mm = 256.0 / L
c = (np.arange(L) - (L - 1) / 2) * mm
xs = np.array([c[0], c[-1]]); ys = xs
total = 0.0; per_layer = []
for z0 in range(0, L, 8):
    zs = np.array([c[z0], c[z0 + 7]])
    X, Y, Z = np.meshgrid(xs, ys, zs, indexing="ij")
    X, Y, Z = X.ravel(), Y.ravel(), Z.ravel()
    # the circle of the FOV is what is visible; corners of the square overestimate a little, so use
    # the disc of radius L/2 voxels sampled on its rim
    th = np.linspace(0, 2 * np.pi, 64, endpoint=False)
    R = 0.5 * L * mm * np.sqrt(2)  # blocks cover the whole square
    Xr = np.concatenate([R * np.cos(th)] * 2); Yr = np.concatenate([R * np.sin(th)] * 2)
    Zr = np.concatenate([np.full(64, zs[0]), np.full(64, zs[1])])
    rows = 0
    for a in A:
        w = a[2] * Xr + a[5] * Yr + a[8] * Zr + a[11]
        v = (a[1] * Xr + a[4] * Yr + a[7] * Zr + a[10]) / w
        lo, hi = max(0.0, np.floor(v.min()) - 1), min(isy, np.floor(v.max()) + 3)
        rows += max(0.0, hi - lo)
    per_layer.append(rows * isx * 8)
    total += rows * isx * 8
per_layer = np.array(per_layer)
print(f"L={L}, {B}-view launch: band working set per z-layer: min {per_layer.min() / 1e6:.0f} MB, "
      f"median {np.median(per_layer) / 1e6:.0f} MB, max {per_layer.max() / 1e6:.0f} MB (L2: 126 MB)")
print(f"sum over the {len(per_layer)} z-layers: {total / 1e9:.1f} GB per launch "
      f"(pair rows read once: {B * (isy + 1) * isx * 8 / 1e9:.2f} GB)")
