"""E2E of single z-slabs at 1024^3 (thick outer vs thin middle slab of the 8-way partition) with
different deferred-tail depths: where does a slab's end-to-end time go."""
import sys, time, os
sys.path.insert(0, "/root/repo")
import paper_1104_5243_b200 as bp
s = bp.Stack.baseline(n_views=496, isx=1248, isy=960)
L=1024
for (z0, z1) in ((0, 224), (416, 512)):
    out = bp.Volume.create(L).data[z0:z1]
    for tb in (-1, 5, 6):
        with bp.GpuContext(L, 1248, 960, device=0, z_begin=z0, z_end=z1, strict=False, view_batch=32, tail_batches=tb) as c:
            c.backproject_stack(s); c.finish(out=out)
            t0 = time.perf_counter(); c.backproject_stack(s); _, st = c.finish(out=out); dt = (time.perf_counter() - t0) * 1e3
        print(f"slab [{z0},{z1}) tail={tb}: e2e {dt:.1f} ms, h2d {st.h2d_ms:.1f} ms ({st.h2d_bytes/1e9:.2f} GB), d2h {st.d2h_ms:.1f} ms, device {st.device_ms:.1f} ms", flush=True)
