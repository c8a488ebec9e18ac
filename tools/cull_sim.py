"""Share of computed voxel updates that finer culling (per z-slice, per consumer warp, per (warp, slice))
would skip, on the BASELINE geometry: 32x32x8 blocks, sampled (block, view) pairs.  Usage: python tools/cull_sim.py [L]"""
import numpy as np, sys
sys.path.insert(0, ".")
import paper_1104_5243_b200 as bp
L = int(sys.argv[1]) if len(sys.argv) > 1 else 512
s = bp.Stack.baseline(n_views=62, isx=1248, isy=960, filter=0, threads=8)
mats = s.matrices
MM = 256.0 / L; off = -0.5 * (L - 1) * MM
BX,BY,BZ=32,32,8
rng=np.random.default_rng(0)
xs,ys,zs=np.meshgrid(np.arange(BX),np.arange(BY),np.arange(BZ),indexing='ij')
tot_comp=0; tot_vis=0; slice_cull=0; warp_cull=0; both=0
for t in range(6000):
    A = mats[rng.integers(0, len(mats))]
    bx,by,bz = rng.integers(0,L//BX), rng.integers(0,L//BY), rng.integers(0,L//BZ)
    X=(bx*BX+xs)*MM+off; Y=(by*BY+ys)*MM+off; Z=(bz*BZ+zs)*MM+off
    w = A[2]*X + A[5]*Y + A[8]*Z + A[11]
    u = (A[0]*X + A[3]*Y + A[6]*Z + A[9]) / w; v = (A[1]*X + A[4]*Y + A[7]*Z + A[10]) / w
    iu=np.floor(u); iv=np.floor(v)
    vis=(iu>=-1)&(iu<=1247)&(iv>=-1)&(iv<=959)
    if not vis.any(): continue   # culled block (producer)
    tot_comp+=vis.size; tot_vis+=vis.sum()
    # per-slice culling: slice z invisible entirely
    sl=~vis.any(axis=(0,1))  # per z
    slice_cull+=sl.sum()*BX*BY
    # per-warp (DY layout): warp w covers x in [16*(w%2), +16), y rows {4*(w//2)+0..3} and +16
    wc=0
    for wi in range(8):
        x0=16*(wi%2); yy=[4*(wi//2)+k for k in range(4)]+[4*(wi//2)+16+k for k in range(4)]
        sub=vis[x0:x0+16][:,yy,:]
        if not sub.any(): wc+=sub.size
    warp_cull+=wc
    # combined: per (warp, slice)
    c=0
    for wi in range(8):
        x0=16*(wi%2); yy=[4*(wi//2)+k for k in range(4)]+[4*(wi//2)+16+k for k in range(4)]
        sub=vis[x0:x0+16][:,yy,:]
        c+=(~sub.any(axis=(0,1))).sum()*16*8
    both+=c
print(f"L={L}: invisible share of computed {1-tot_vis/tot_comp:.4f}; per-slice cull {slice_cull/tot_comp:.4f}; per-warp cull {warp_cull/tot_comp:.4f}; per-(warp,slice) {both/tot_comp:.4f}")
