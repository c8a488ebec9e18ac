"""Footprint rows (8-row TMA boxes) and widths per (block, view) on the BASELINE geometry.
Env SHAPE=BX,BY,BZ (default 32,32,8)."""
import numpy as np, sys
sys.path.insert(0, ".")
import paper_1104_5243_b200 as bp
L = 512
s = bp.Stack.baseline(n_views=62, isx=1248, isy=960, filter=0, threads=8)
mats = s.matrices
MM = 256.0 / L; off = -0.5 * (L - 1) * MM
import os
BX,BY,BZ=[int(v) for v in os.environ.get("SHAPE","32,32,8").split(",")]
rows=[];widths=[]
rng=np.random.default_rng(0)
for t in range(4000):
    A = mats[rng.integers(0, len(mats))]
    bx,by,bz = rng.integers(0,L//BX), rng.integers(0,L//BY), rng.integers(0,L//BZ)
    cx = np.array([bx*BX, bx*BX+BX-1]); cy=np.array([by*BY,by*BY+BY-1]); cz=np.array([bz*BZ,bz*BZ+BZ-1])
    X,Y,Z = np.meshgrid(cx*MM+off, cy*MM+off, cz*MM+off)
    w = A[2]*X + A[5]*Y + A[8]*Z + A[11]
    u = (A[0]*X + A[3]*Y + A[6]*Z + A[9]) / w; v = (A[1]*X + A[4]*Y + A[7]*Z + A[10]) / w
    umin,umax=np.floor(u.min()),np.floor(u.max()); vmin,vmax=np.floor(v.min()),np.floor(v.max())
    iu0=(int(umin)-1)&~3; iu1=umax+2; iv0=vmin-1; iv1=vmax+2
    if iu1<0 or iu0>1247 or iv1<0 or iv0>959: continue
    rows.append((int(iv1-iv0)+8)&~7); widths.append(iu1-iu0+1)
rows=np.array(rows); widths=np.array(widths)
print("rows pct", np.percentile(rows,[5,25,50,75,95,100]), "mean", rows.mean())
print("width pct", np.percentile(widths,[5,25,50,75,95,100]))
