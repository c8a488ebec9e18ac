import numpy as np, sys
sys.path.insert(0, ".")
import paper_1104_5243_b200 as bp
L = 512
s = bp.Stack.baseline(n_views=62, isx=1248, isy=960, filter=0, threads=8)
mats = s.matrices
MM = 256.0 / L; off = -0.5 * (L - 1) * MM
rng = np.random.default_rng(1)

def wavefronts(addrs):
    a = np.unique(addrs)
    return np.bincount(a % 32, minlength=32).max()

def eval_mapping(lane_xyz, P, nsamp=300):
    tot = 0; n = 0
    for _ in range(nsamp):
        A = mats[rng.integers(0, len(mats))]
        x0, y0, z0 = rng.integers(0, L - 64, size=3)
        X = (x0 + lane_xyz[:, 0]) * MM + off
        Y = (y0 + lane_xyz[:, 1]) * MM + off
        Z = (z0 + lane_xyz[:, 2]) * MM + off
        w = A[2]*X + A[5]*Y + A[8]*Z + A[11]
        u = (A[0]*X + A[3]*Y + A[6]*Z + A[9]) / w; v = (A[1]*X + A[4]*Y + A[7]*Z + A[10]) / w
        base = np.floor(v).astype(np.int64) * P + np.floor(u).astype(np.int64)
        for d in (0, 1, P, P + 1):
            tot += wavefronts(base + d); n += 1
    return tot / n

i = np.arange(32)
maps = {
 "M1cur": np.stack([2 * (i % 16), i // 16, 0 * i], 1),
 "32x": np.stack([i, 0 * i, 0 * i], 1),
 "32x_s2": np.stack([2 * i, 0 * i, 0 * i], 1),
 "16x2z": np.stack([i % 16, 0 * i, i // 16], 1),
 "8x4z": np.stack([i % 8, 0 * i, i // 8], 1),
 "8x4y": np.stack([i % 8, i // 8, 0 * i], 1),
 "4x8z": np.stack([i % 4, 0 * i, i // 4], 1),
 "4x4y2z": np.stack([i % 4, (i // 4) % 4, i // 16], 1),
 "8x2y2z": np.stack([i % 8, (i // 8) % 2, i // 16], 1),
 "16xs2_2z": np.stack([2 * (i % 16), 0 * i, i // 16], 1),
 "2x16z": np.stack([i % 2, 0 * i, i // 2], 1),
 "32z": np.stack([0 * i, 0 * i, i], 1),
}
for P in (128, 132, 136, 144, 120, 124, 116):
    print("pitch", P, {k: round(eval_mapping(m, P), 2) for k, m in maps.items()}, flush=True)
print("---- more patterns")
maps2 = {
 "8x4y": np.stack([i % 8, i // 8, 0 * i], 1),
 "16x2y": np.stack([i % 16, i // 16, 0 * i], 1),
 "4x8y": np.stack([i % 4, i // 4, 0 * i], 1),
 "32y": np.stack([0 * i, i, 0 * i], 1),
 "2x16y": np.stack([i % 2, i // 2, 0 * i], 1),
 "8x2y2z": np.stack([i % 8, (i // 8) % 2, i // 16], 1),
 "4x4y2z": np.stack([i % 4, (i // 4) % 4, i // 16], 1),
 "xy_diag": np.stack([i % 8, (i // 8) + (i % 8) // 2, 0*i], 1),
}
for P in (116, 120, 136, 144, 152):
    print("pitch", P, {k: round(eval_mapping(m, P, 250), 2) for k, m in maps2.items()}, flush=True)
