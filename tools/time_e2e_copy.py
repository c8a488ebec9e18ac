"""Wall time of bench.py's e2e_copy leg: bp_gpu_backproject (copy semantics) per view from
PAGEABLE numpy buffers, bp_gpu_finish into a PAGEABLE volume, next to the pinned zero-copy
e2e leg.  One library build per run (BP_LIB_PATH).  Env: AB_L (512), AB_BATCH (32), AB_REPS (3), AB_LEG (e2e,e2e_copy), AB_STRICT (0), AB_VIEWS (views hint, 496; 0: none)."""
import os, statistics, sys, time
import numpy as np
sys.path.insert(0, ".")
import paper_1104_5243_b200 as bp
L = int(os.environ.get("AB_L", "512"))
B = int(os.environ.get("AB_BATCH", "32"))
reps = int(os.environ.get("AB_REPS", "3"))
s = bp.Stack.baseline(n_views=496, isx=1248, isy=960)
legs = os.environ.get("AB_LEG", "e2e,e2e_copy").split(",")
mats = s.matrices
if "e2e_copy" in legs:
    pg_px = np.array(s.pixels, copy=True)
    pg_vol = np.zeros((L, L, L), np.float32)
vol = bp.Volume.create(L)
res = {}
with bp.GpuContext(L, 1248, 960, device=0, view_batch=B,
                   strict=os.environ.get("AB_STRICT") == "1",
                   views=int(os.environ.get("AB_VIEWS", "496"))) as c:
    for leg in legs:
        for r in range(reps + 1):
            t0 = time.perf_counter()
            if leg == "e2e":
                c.backproject_stack(s)
                _, st = c.finish(out=vol.data)
            else:
                for k in range(pg_px.shape[0]):
                    c.backproject(pg_px[k], mats[k], copy=True)
                t1 = time.perf_counter()
                _, st = c.finish(out=pg_vol)
                if r:
                    res.setdefault("calls", []).append((t1 - t0) * 1e3)
            if r:
                res.setdefault(leg, []).append((time.perf_counter() - t0) * 1e3)
        calls = f" (backproject calls {statistics.median(res['calls']):.1f} ms)" if leg == "e2e_copy" else ""
        print(f"{os.environ.get('AB_TAG', bp.LIB_PATH)}: {leg}{calls} L={L} B={B} median "
              f"{statistics.median(res[leg]):.2f} ms all {[round(x, 1) for x in res[leg]]} "
              f"(h2d {st.h2d_ms:.1f} ms, d2h {st.d2h_ms:.1f} ms)")
if "e2e" in res and "e2e_copy" in res:
    d = np.abs(pg_vol.astype(np.float64) - vol.data.reshape(pg_vol.shape)).max()
    print("e2e_copy volume == e2e volume:", d == 0.0)
