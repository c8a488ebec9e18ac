"""Wall time of the one-shot C-ABI reconstruction bp_reconstruct (pinned host stack in, host
volume out), checked bitwise against the streaming module path.
Env: AB_L (512), AB_REPS (5), AB_STRICT (0)."""
import os, statistics, sys, time
sys.path.insert(0, ".")
import numpy as np
import paper_1104_5243_b200 as bp
L = int(os.environ.get("AB_L", "512"))
reps = int(os.environ.get("AB_REPS", "5"))
strict = os.environ.get("AB_STRICT") == "1"
s = bp.Stack.baseline(n_views=496, isx=1248, isy=960)
prm = bp.recon_params(L, block_b=32, strict_mode=int(strict))
vol, st = bp.reconstruct(s, prm)  # warm-up (context creation, pinned pool)
v = []
for _ in range(reps):
    t0 = time.perf_counter()
    vol, st = bp.reconstruct(s, prm)
    v.append((time.perf_counter() - t0) * 1e3)
med = statistics.median(v)
with bp.GpuContext(L, 1248, 960, device=0, strict=strict, view_batch=32) as c:
    c.backproject_stack(s)
    ref, _ = c.finish()
same = np.array_equal(vol.data.view(np.int32), ref.view(np.int32))
print(f"bp_reconstruct L={L}: median {med:.2f} ms -> "
      f"{496 * L ** 3 / med / 1e6:.1f} GUP/s (all {[round(x, 1) for x in v]}); bitwise == module path: {same}")
