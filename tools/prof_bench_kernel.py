"""One resident 512^3 reconstruction with the bench's launch shape (248-view launches), for
ncu captures of the hot kernel: ncu -k regex:bp_tile_kernel --launch-skip 1 --launch-count 1 ...
Env: AB_L (512), AB_BATCH (248), AB_STRICT (0)."""
import os, sys
sys.path.insert(0, ".")
import paper_1104_5243_b200 as bp
L = int(os.environ.get("AB_L", "512"))
B = int(os.environ.get("AB_BATCH", "248"))
s = bp.Stack.baseline(n_views=496, isx=1248, isy=960)
with bp.GpuContext(L, 1248, 960, device=0, strict=os.environ.get("AB_STRICT") == "1",
                   view_batch=B, ring_batches=(496 + B - 1) // B) as c:
    c.upload_stack(s)
    ms, st = c.time_resident(1)
    print(f"L={L} B={B} ms={ms:.2f} tile {st.tile_w}x{st.tile_h}")
