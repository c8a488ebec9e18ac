"""Pair-ring bank conflicts at 512^3: fixed pitches, an oracle choice of the best pitch per (block, view)
sample, the conflict-free ideal, and per-lane left/right load-order swaps.  Usage: python
tools/bank_sim_pitch_oracle.py [L]"""
import numpy as np, sys
sys.path.insert(0, ".")
import paper_1104_5243_b200 as bp
L = int(sys.argv[1]) if len(sys.argv)>1 else 512
s = bp.Stack.baseline(n_views=62, isx=1248, isy=960, filter=0, threads=8)
mats = s.matrices
MM = 256.0 / L; off = -0.5 * (L - 1) * MM
lay = np.array([(l%4+4*(l//16),(l//4)%4,0) for l in range(32)])
rng = np.random.default_rng(1)
uv=[]
for _ in range(600):
    A = mats[rng.integers(0, len(mats))]
    x0, y0, z0 = rng.integers(0, L - 64, size=3)
    X = (x0 + lay[:, 0]) * MM + off; Y = (y0 + lay[:, 1]) * MM + off; Z = (z0 + lay[:, 2]) * MM + off
    w = A[2]*X + A[5]*Y + A[8]*Z + A[11]
    u = (A[0]*X + A[3]*Y + A[6]*Z + A[9]) / w; v = (A[1]*X + A[4]*Y + A[7]*Z + A[10]) / w
    uv.append((np.floor(u).astype(np.int64), np.floor(v).astype(np.int64)))
def wf(W):
    t=0
    for g in (0,16):
        a=np.unique(W[g:g+16]); t+=np.bincount(a%16,minlength=16).max()
    return t
pats={"none":np.zeros(32,int),"lane&1":np.arange(32)&1,"x&1":lay[:,0]&1,"y&1":lay[:,1]&1,"(x^y)&1":(lay[:,0]^lay[:,1])&1,
      "x>>1&1":(lay[:,0]>>1)&1,"y>>1&1":(lay[:,1]>>1)&1, "(x+y)>>1&1":((lay[:,0]+lay[:,1])>>1)&1}
for P in (150,152,154):
  for name,o in pats.items():
    t=sum(wf(v*P+u+o)+wf(v*P+u+1-o) for u,v in uv)/len(uv)/32
    print(P,name,round(t,4))
Ps=list(range(144,162,2))
M=np.array([[wf(v*P+u)+wf(v*P+u+1) for P in Ps] for u,v in uv])/32
print("fixed", dict(zip(Ps, M.mean(0).round(4))))
print("oracle-best per sample", M.min(1).mean().round(4))
# ideal (only unique-word limited, no conflicts)
ideal=np.mean([ (sum(max(1,int(np.ceil(len(np.unique((v*152+u)[g:g+16]))/16))) for g in (0,16))*2)/32 for u,v in uv])
print("ideal", ideal)
