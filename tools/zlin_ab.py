"""A/B of the z-linearised fast kernel (BP_ZLIN=1, default) against the exact-coordinate fast
kernel (BP_ZLIN=0): accuracy of both against GPU strict (== the reference, bitwise) over the
full volume, and resident timing (interleaved rounds).
Usage: python tools/zlin_ab.py [L ...]   (AB_ROUNDS=3, AB_ACC=1)
"""
import os, sys, statistics
sys.path.insert(0, ".")
import paper_1104_5243_b200 as bp

Ls = [int(a) for a in sys.argv[1:]] or [512]
rounds = int(os.environ.get("AB_ROUNDS", "3"))
s = bp.Stack.baseline()
for L in Ls:
    off = (60.0, 0.0, 0.0) if L == 2048 else (0.0, 0.0, 0.0)
    if os.environ.get("AB_ACC", "1") == "1":
        strict = bp.GpuContext(L, 1248, 960, offset=off, strict=True)
        strict.backproject_stack(s)
        strict.finish(readback=False)
        for z in ("0", "1"):
            os.environ["BP_ZLIN"] = z
            c = bp.GpuContext(L, 1248, 960, offset=off, strict=False)
            c.backproject_stack(s)
            _, st = c.finish(readback=False)
            mx, peak, sq, nbit = c.compare_with(strict)
            print(f"L={L} BP_ZLIN={z}: max {mx / peak:.2e} rms {sq / peak:.2e} of max|ref|, "
                  f"fallback pairs {st.fallback_pairs}, tile {st.tile_w}x{st.tile_h}", flush=True)
            c.close()
        strict.close()
    B = 248
    res = {"0": [], "1": []}
    for r in range(rounds):
        for z in ("0", "1"):
            os.environ["BP_ZLIN"] = z
            with bp.GpuContext(L, 1248, 960, offset=off, strict=False, view_batch=B,
                               ring_batches=(496 + B - 1) // B, profile_launches=True) as c:
                c.upload_stack(s)
                c.time_resident(1)
                for _ in range(3):
                    ms, st = c.time_resident(1)
                    res[z].append(ms)
    for z in ("0", "1"):
        med = statistics.median(res[z])
        print(f"L={L} BP_ZLIN={z}: median {med:.2f} ms min {min(res[z]):.2f} -> "
              f"{496 * L ** 3 / med / 1e6:.1f} GUP/s nominal", flush=True)
