"""Bank-conflict simulation of candidate lane layouts on the BASELINE geometry: 64-bit pair-ring loads
(half-warp phases, 16 bank pairs) and 128-bit quad-texel loads (quarter-warp phases, 8 bank quads), each
layout with its best tile pitch.  The phase sizes are the ones tools/lds_wavefront_probe.cu measured on
B200.  Usage: python tools/bank_sim_layouts.py [L]"""
import sys
import numpy as np
sys.path.insert(0, ".")
import paper_1104_5243_b200 as bp
L = int(sys.argv[1]) if len(sys.argv)>1 else 512
s = bp.Stack.baseline(n_views=62, isx=1248, isy=960, filter=0, threads=8)
mats = s.matrices
MM = 256.0 / L; off = -0.5 * (L - 1) * MM
rng = np.random.default_rng(1)
samples=[]
for _ in range(400):
    A = mats[rng.integers(0, len(mats))]
    x0, y0, z0 = rng.integers(0, L - 64, size=3)
    samples.append((A,x0,y0,z0))
def wf(W, group, nb):
    t=0
    for g in range(0,32,group):
        a=np.unique(W[g:g+group]); t+=np.bincount(a%nb,minlength=nb).max()
    return t
def uvs(lay):
    out=[]
    for A,x0,y0,z0 in samples:
        X = (x0 + lay[:, 0]) * MM + off; Y = (y0 + lay[:, 1]) * MM + off; Z = (z0 + lay[:, 2]) * MM + off
        w = A[2]*X + A[5]*Y + A[8]*Z + A[11]
        u = (A[0]*X + A[3]*Y + A[6]*Z + A[9]) / w; v = (A[1]*X + A[4]*Y + A[7]*Z + A[10]) / w
        out.append((np.floor(u).astype(np.int64), np.floor(v).astype(np.int64)))
    return out
def layout(gx,gy,gz, sx=1,sy=1,sz=1):
    # phase group of gx*gy*gz lanes, x fastest; the rest of the warp continues in x
    g=gx*gy*gz; L=[]
    for l in range(32):
        p, i = divmod(l, g)
        x = i % gx; y=(i//gx)%gy; z=i//(gx*gy)
        L.append(((x+gx*p)*sx, y*sy, z*sz))
    return np.array(L)
res=[]
for (gx,gy,gz) in [(4,4,1),(2,8,1),(8,2,1),(4,2,2),(2,4,2),(2,2,4),(4,1,4),(1,4,4),(2,1,8),(1,2,8),(8,1,2),(16,1,1),(1,16,1),(1,1,16)]:
    uv=uvs(layout(gx,gy,gz))
    best=min((sum(wf(v*P+u,16,16)+wf(v*P+u+1,16,16) for u,v in uv)/len(uv)/32,P) for P in range(144,162,2))
    res.append(("LDS64",gx,gy,gz,round(best[0],4),best[1]))
    print(res[-1],flush=True)
for (gx,gy,gz) in [(4,2,1),(2,4,1),(8,1,1),(1,8,1),(2,2,2),(4,1,2),(1,4,2),(2,1,4),(1,2,4),(1,1,8)]:
    uv=uvs(layout(gx,gy,gz))
    best=min((sum(wf(v*P+u,8,8) for u,v in uv)/len(uv)/32,P) for P in range(144,160,1))
    print(("LDS128",gx,gy,gz,round(best[0],4),best[1]),flush=True)
