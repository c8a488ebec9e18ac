"""Median resident-projection time at 512^3 (or AB_L) for one library build.

Used for compile-time A/B: run once per build with BP_LIB_PATH pointing at it.
Env: AB_L (512), AB_BATCH (64), AB_STRICT (0), AB_REPS (5)."""
import os, statistics, sys
sys.path.insert(0, ".")
import paper_1104_5243_b200 as bp
L = int(os.environ.get("AB_L", "512"))
B = int(os.environ.get("AB_BATCH", "64"))
reps = int(os.environ.get("AB_REPS", "5"))
s = bp.Stack.baseline(n_views=496, isx=1248, isy=960)
with bp.GpuContext(L, 1248, 960, device=0, strict=os.environ.get("AB_STRICT") == "1",
                   view_batch=B, ring_batches=(496 + B - 1) // B,
                   profile_launches=True) as c:
    c.upload_stack(s)
    c.time_resident(1)
    v, kv = [], []
    for _ in range(reps):
        ms, st = c.time_resident(1)
        v.append(ms)
        kv.append(st.kernel_ms)
med = statistics.median(v)
kmed = statistics.median(kv)
print(f"{os.environ.get('AB_TAG', bp.LIB_PATH)}: L={L} B={B} median {med:.2f} ms -> "
      f"{496 * L ** 3 / med / 1e6:.1f} GUP/s; backprojection kernels {kmed:.2f} ms (tile {st.tile_w}x{st.tile_h}, fallback {st.fallback_pairs})")
