"""Pair ring vs raw-tile fast kernel: bitwise check and interleaved timing.

Resident projections, one process, two contexts (BP_NO_PAIR is read at context
construction).  Env: AB_L (512), AB_BATCH (124), AB_REPS (5), AB_ARCP (0).
"""
import os, statistics, sys
sys.path.insert(0, ".")
import paper_1104_5243_b200 as bp

L = int(os.environ.get("AB_L", "512"))
B = int(os.environ.get("AB_BATCH", "124"))
reps = int(os.environ.get("AB_REPS", "5"))
recip = 3 if os.environ.get("AB_ARCP") == "1" else 0
s = bp.Stack.baseline(n_views=496, isx=1248, isy=960)
ctx = {}
for name, flag in (("raw", "1"), ("pair", "0")):
    os.environ["BP_NO_PAIR"] = flag
    c = bp.GpuContext(L, 1248, 960, device=0, strict=False, view_batch=B,
                      ring_batches=(496 + B - 1) // B, recip_mode=recip)
    c.upload_stack(s)
    c.time_resident(1)
    ctx[name] = c
os.environ.pop("BP_NO_PAIR", None)
mx, mr, rms, nb = ctx["pair"].compare_with(ctx["raw"])
print(f"L={L} B={B}: pair vs raw max|d|={mx:.3e} max|ref|={mr:.3e} rms={rms:.3e} bitwise-diff={nb}")
t = {k: [] for k in ctx}
for _ in range(reps):
    for k, c in ctx.items():
        ms, st = c.time_resident(1)
        t[k].append((ms, st.kernel_ms, st.tile_w, st.tile_h, st.fallback_pairs))
for k, v in t.items():
    med = statistics.median(x[0] for x in v)
    print(f"{k:5s}: median {med:.2f} ms -> {496 * L ** 3 / med / 1e6:.1f} GUP/s nominal "
          f"(tile {v[0][2]}x{v[0][3]}, fallback {v[0][4]}, all {[round(x[0], 2) for x in v]})")
for c in ctx.values():
    c.close()
