import numpy as np, sys
sys.path.insert(0, ".")
import paper_1104_5243_b200 as bp
L = 512
s = bp.Stack.baseline(n_views=62, isx=1248, isy=960, filter=0, threads=8)
mats = s.matrices
MM = 256.0 / L; off = -0.5 * (L - 1) * MM
def run(maps, pitches, nsamp=300, seed=1):
    rng = np.random.default_rng(seed)
    samples = []
    for _ in range(nsamp):
        A = mats[rng.integers(0, len(mats))]
        x0, y0, z0 = rng.integers(0, L - 64, size=3)
        samples.append((A, x0, y0, z0))
    for P in pitches:
        res = {}
        for k, m in maps.items():
            tot = 0; n = 0
            for A, x0, y0, z0 in samples:
                X = (x0 + m[:, 0]) * MM + off; Y = (y0 + m[:, 1]) * MM + off; Z = (z0 + m[:, 2]) * MM + off
                w = A[2]*X + A[5]*Y + A[8]*Z + A[11]
                u = (A[0]*X + A[3]*Y + A[6]*Z + A[9]) / w; v = (A[1]*X + A[4]*Y + A[7]*Z + A[10]) / w
                base = np.floor(v).astype(np.int64) * P + np.floor(u).astype(np.int64)
                for d in (0, 1, P, P + 1):
                    a = np.unique(base + d)
                    tot += np.bincount(a % 32, minlength=32).max(); n += 1
            res[k] = round(tot / n, 3)
        print("pitch", P, res, flush=True)
i = np.arange(32)
maps = {
 "8x4y": np.stack([i % 8, i // 8, 0 * i], 1),
 "8x4y_ys2": np.stack([i % 8, 2 * (i // 8), 0 * i], 1),
 "8x4y_ys4": np.stack([i % 8, 4 * (i // 8), 0 * i], 1),
 "8xs2_4y": np.stack([2 * (i % 8), i // 8, 0 * i], 1),
 "4x8y": np.stack([i % 4, i // 4, 0 * i], 1),
 "16x2y": np.stack([i % 16, i // 16, 0 * i], 1),
 "8x2y2z": np.stack([i % 8, (i // 8) % 2, i // 16], 1),
 "4x4y2z": np.stack([i % 4, (i // 4) % 4, i // 16], 1),
 "8x4yskew": np.stack([(i % 8 + 2 * (i // 8)) % 8, i // 8, 0 * i], 1),
}
run(maps, [144, 148, 152, 160, 168, 176, 180, 184, 188, 196])
