import numpy as np, sys
sys.path.insert(0, ".")
import paper_1104_5243_b200 as bp
L = 512
s = bp.Stack.baseline(n_views=496, isx=1248, isy=960, filter=0, threads=8)
mats = s.matrices
MM = 256.0 / L; off = -0.5 * (L - 1) * MM
i = np.arange(32)
lanes = np.stack([i % 8, i // 8, 0 * i], 1)
pitches = [144, 148, 152, 156, 164, 168, 172, 176, 180, 184, 188, 196, 200]
rng = np.random.default_rng(3)
views = list(range(0, 496, 31))
res = np.zeros((len(views), len(pitches)))
for vi, k in enumerate(views):
    A = mats[k]
    samples = [rng.integers(0, L - 64, size=3) for _ in range(150)]
    for pi, P in enumerate(pitches):
        tot = n = 0
        for x0, y0, z0 in samples:
            X = (x0 + lanes[:, 0]) * MM + off; Y = (y0 + lanes[:, 1]) * MM + off; Z = (z0 + lanes[:, 2]) * MM + off
            w = A[2]*X + A[5]*Y + A[8]*Z + A[11]
            u = (A[0]*X + A[3]*Y + A[6]*Z + A[9]) / w; v = (A[1]*X + A[4]*Y + A[7]*Z + A[10]) / w
            base = np.floor(v).astype(np.int64) * P + np.floor(u).astype(np.int64)
            for d in (0, 1, P, P + 1):
                a = np.unique(base + d)
                tot += np.bincount(a % 32, minlength=32).max(); n += 1
        res[vi, pi] = tot / n
np.set_printoptions(precision=2, linewidth=200)
print("pitches", pitches)
for vi, k in enumerate(views): print(k, res[vi])
print("mean per pitch", res.mean(0))
print("mean of per-view best", res.min(1).mean(), "best fixed", res.mean(0).min())
