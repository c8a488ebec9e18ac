"""Bank-conflict simulation of the pair ring: 64-bit loads served per half-warp (16 bank pairs),
4 (x) x 4 (y) voxels per half-warp, tile pitch sweep.  Usage: python tools/bank_sim64.py [L]"""
import numpy as np, sys
sys.path.insert(0, ".")
import paper_1104_5243_b200 as bp
L = int(sys.argv[1]) if len(sys.argv)>1 else 512
s = bp.Stack.baseline(n_views=62, isx=1248, isy=960, filter=0, threads=8)
mats = s.matrices
MM = 256.0 / L; off = -0.5 * (L - 1) * MM
def mk(f): return np.array([f(l) for l in range(32)])
lay = mk(lambda l:(l%4+4*(l//16),(l//4)%4,0))
rng = np.random.default_rng(1)
samples=[]
for _ in range(300):
    A = mats[rng.integers(0, len(mats))]
    x0, y0, z0 = rng.integers(0, L - 64, size=3)
    samples.append((A,x0,y0,z0))
def wf64(W):
    t=0
    for h in (W[:16],W[16:]):
        a=np.unique(h); t+=np.bincount(a%16,minlength=16).max()
    return t
res=[]
for P in range(80,176,4):
    t64=0;n=0
    for A,x0,y0,z0 in samples:
        X = (x0 + lay[:, 0]) * MM + off; Y = (y0 + lay[:, 1]) * MM + off; Z = (z0 + lay[:, 2]) * MM + off
        w = A[2]*X + A[5]*Y + A[8]*Z + A[11]
        u = (A[0]*X + A[3]*Y + A[6]*Z + A[9]) / w; v = (A[1]*X + A[4]*Y + A[7]*Z + A[10]) / w
        base=np.floor(v).astype(np.int64)*P+np.floor(u).astype(np.int64)
        t64+=wf64(base)+wf64(base+1); n+=1
    res.append((P,round(t64/n/32,3)))
print(res)
