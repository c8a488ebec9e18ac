"""E2E of single z-slabs at 1024^3 (outer slabs of the 8-way partition) with the band-tail timeline
(BP_BAND_TRACE=1): where does a slab's end-to-end time go.
Usage: python tools/slab_e2e_probe.py [z0 z1]   Env: AB_BATCH (62), AB_TAIL (-1), AB_REPS (3)"""
import sys, time, os
sys.path.insert(0, ".")
import paper_1104_5243_b200 as bp
s = bp.Stack.baseline(n_views=496, isx=1248, isy=960)
L = 1024
z0, z1 = (int(sys.argv[1]), int(sys.argv[2])) if len(sys.argv) > 2 else (808, 1024)
B = int(os.environ.get("AB_BATCH", "62")); tb = int(os.environ.get("AB_TAIL", "-1"))
out = bp.Volume.create(L).data[z0:z1]
with bp.GpuContext(L, 1248, 960, device=0, z_begin=z0, z_end=z1, strict=False, view_batch=B,
                   tail_batches=tb, views=496) as c:
    c.backproject_stack(s); c.finish(out=out)
    ts = []
    for _ in range(int(os.environ.get("AB_REPS", "3"))):
        t0 = time.perf_counter(); c.backproject_stack(s); _, st = c.finish(out=out)
        ts.append((time.perf_counter() - t0) * 1e3)
print(f"slab [{z0},{z1}) B={B} tail={tb}: e2e {[round(t, 1) for t in ts]} ms, h2d {st.h2d_ms:.1f} ms "
      f"({st.h2d_bytes / 1e9:.2f} GB), d2h {st.d2h_ms:.1f} ms ({st.d2h_bytes / 1e9:.2f} GB), device {st.device_ms:.1f} ms, "
      f"launches {st.launches}+{st.prep_launches}", flush=True)
