import sys, time
sys.path.insert(0, ".")
import paper_1104_5243_b200 as bp
L = int(sys.argv[1]) if len(sys.argv) > 1 else 512
strict = len(sys.argv) > 2 and sys.argv[2] == "strict"
s = bp.Stack.baseline(n_views=496, isx=1248, isy=960)
with bp.GpuContext(L, 1248, 960, device=0, strict=strict, view_batch=32, ring_batches=16, profile_launches=True) as c:
    c.upload_stack(s)
    for i in range(2):
        ms, st = c.time_resident(1)
        print(f"L={L} strict={strict} ms={ms:.2f} nominal GUP/s={496*L**3/ms/1e6:.1f} kernel_ms={st.kernel_ms:.2f}", st.tile_w, st.tile_h, st.fallback_pairs)
