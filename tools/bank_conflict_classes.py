"""Which lane pairs conflict in the pair ring (pitch 152): (row difference, column difference) classes of
same-bank-pair, different-word lanes in each half-warp, and the row spread of a half-warp.  Usage:
python tools/bank_conflict_classes.py"""
import numpy as np, sys, collections
sys.path.insert(0, ".")
import paper_1104_5243_b200 as bp
L = 512
s = bp.Stack.baseline(n_views=62, isx=1248, isy=960, filter=0, threads=8)
mats = s.matrices
MM = 256.0 / L; off = -0.5 * (L - 1) * MM
lay = np.array([(l%4+4*(l//16),(l//4)%4,0) for l in range(32)])
rng = np.random.default_rng(1)
P=152
cls=collections.Counter(); extra=0; n=0
rowspread=collections.Counter()
for _ in range(1500):
    A = mats[rng.integers(0, len(mats))]
    x0, y0, z0 = rng.integers(0, L - 64, size=3)
    X = (x0 + lay[:, 0]) * MM + off; Y = (y0 + lay[:, 1]) * MM + off; Z = (z0 + lay[:, 2]) * MM + off
    w = A[2]*X + A[5]*Y + A[8]*Z + A[11]
    u = np.floor((A[0]*X + A[3]*Y + A[6]*Z + A[9]) / w).astype(int); v = np.floor((A[1]*X + A[4]*Y + A[7]*Z + A[10]) / w).astype(int)
    for h in (slice(0,16),slice(16,32)):
        uu,vv=u[h],v[h]
        rowspread[vv.max()-vv.min()]+=1
        words={}
        for a,b in zip(uu,vv): words[(b,a)]=1
        wl=list(words)
        banks=collections.defaultdict(list)
        for (r,c) in wl: banks[(r*P+c)%16].append((r,c))
        deg=max(len(x) for x in banks.values()); extra+=deg-1; n+=1
        for b,lst in banks.items():
            for i in range(len(lst)):
                for j in range(i+1,len(lst)):
                    dr=abs(lst[i][0]-lst[j][0]); dc=lst[j][1]-lst[i][1] if lst[j][0]>=lst[i][0] else lst[i][1]-lst[j][1]
                    cls[(dr,dc)]+=1
print("mean extra wavefronts per half-warp LDS", extra/n)
print("row spread within half-warp", sorted(rowspread.items()))
print(cls.most_common(12))
