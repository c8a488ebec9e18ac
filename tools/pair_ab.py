"""Pair ring vs raw-tile fast kernel: bitwise check and interleaved timing.

Resident projections, one process, one context per variant (the BP_* switches are read
at context construction); every variant is compared bitwise with the first.
Env: AB_L (512), AB_BATCH (124), AB_REPS (5), AB_ARCP (0),
AB_VARIANTS ("raw=BP_NO_PAIR:1;pair_fixed=BP_PAIR_FIXED:1;pair=").
"""
import os, statistics, sys
sys.path.insert(0, ".")
import paper_1104_5243_b200 as bp

L = int(os.environ.get("AB_L", "512"))
B = int(os.environ.get("AB_BATCH", "124"))
reps = int(os.environ.get("AB_REPS", "5"))
recip = 3 if os.environ.get("AB_ARCP") == "1" else 0
s = bp.Stack.baseline(n_views=496, isx=1248, isy=960)
spec = os.environ.get("AB_VARIANTS", "raw=BP_NO_PAIR:1;pair_fixed=BP_PAIR_FIXED:1;pair=")
ctx = {}
for item in spec.split(";"):
    name, envs = item.split("=", 1)
    kv = [e.split(":") for e in envs.split(",") if e]
    for k, v in kv:
        os.environ[k] = v
    c = bp.GpuContext(L, 1248, 960, device=0, strict=False, view_batch=B,
                      ring_batches=(496 + B - 1) // B, recip_mode=recip)
    for k, _ in kv:
        os.environ.pop(k, None)
    c.upload_stack(s)
    c.time_resident(1)
    ctx[name] = c
first = next(iter(ctx))
for name, c in ctx.items():
    if name != first:
        mx, mr, rms, nb = c.compare_with(ctx[first])
        print(f"L={L} B={B}: {name} vs {first} max|d|={mx:.3e} max|ref|={mr:.3e} rms={rms:.3e} "
              f"bitwise-diff={nb}")
t = {k: [] for k in ctx}
for _ in range(reps):
    for k, c in ctx.items():
        ms, st = c.time_resident(1)
        t[k].append((ms, st.kernel_ms, st.tile_w, st.tile_h, st.fallback_pairs))
for k, v in t.items():
    med = statistics.median(x[0] for x in v)
    print(f"{k:10s}: median {med:.2f} ms -> {496 * L ** 3 / med / 1e6:.1f} GUP/s nominal "
          f"(tile {v[0][2]}x{v[0][3]}, fallback {v[0][4]}, all {[round(x[0], 2) for x in v]})")
for c in ctx.values():
    c.close()
