"""Wall time of the streamed reconstruction (bench.py's e2e leg): pinned host stack ->
bp_gpu_backproject_async x views -> bp_gpu_finish(host volume).  One library build per run
(BP_LIB_PATH).  Env: AB_L (512), AB_BATCH (32), AB_REPS (3), AB_STRICT (0), AB_FILTER (0),
AB_VIEWS (views hint, 0: none), AB_TAIL (tail batches, -1: default)."""
import os, statistics, sys, time
sys.path.insert(0, ".")
import paper_1104_5243_b200 as bp
L = int(os.environ.get("AB_L", "512"))
B = int(os.environ.get("AB_BATCH", "32"))
reps = int(os.environ.get("AB_REPS", "3"))
s = bp.Stack.baseline(n_views=496, isx=1248, isy=960)
vol = bp.Volume.create(L)
filt = (750.0, 1200.0, 0.32) if os.environ.get("AB_FILTER") == "1" else None
with bp.GpuContext(L, 1248, 960, device=0, strict=os.environ.get("AB_STRICT") == "1",
                   view_batch=B, filter=filt, views=int(os.environ.get("AB_VIEWS", "0")),
                   tail_batches=int(os.environ.get("AB_TAIL", "-1"))) as c:
    c.backproject_stack(s)
    c.finish(out=vol.data)
    v = []
    for _ in range(reps):
        t0 = time.perf_counter()
        c.backproject_stack(s)
        _, st = c.finish(out=vol.data)
        v.append((time.perf_counter() - t0) * 1e3)
med = statistics.median(v)
print(f"{os.environ.get('AB_TAG', bp.LIB_PATH)}: e2e L={L} B={B} median {med:.2f} ms -> "
      f"{496 * L ** 3 / med / 1e6:.1f} GUP/s (h2d {st.h2d_ms:.1f} ms, d2h {st.d2h_ms:.1f} ms, "
      f"device {st.device_ms:.1f} ms, launches {st.launches}+{st.prep_launches}) all {[round(x, 1) for x in v]}")
