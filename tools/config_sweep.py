"""Single-B200 throughput for every BASELINE config (1-5), on the BASELINE stack.

For each config it reports:
- resident GUP/s: projections in HBM, device-event timing, nominal views·L³ per second (248-view launches,
  124 at 2048³);
- visible GUP/s: clip_stats semantics;
- e2e ms: pinned host stack in, host volume out, through the C ABI streaming call (view count
  given: band tail; library-default view batch: 32, 62 from 1024³ up).

Config 5 is the 2048³ grid offset +60 mm in x. Its volume is 32 GB on one GPU here; BASELINE shards it
over 8 GPUs.

Usage: python tools/config_sweep.py [L ...]
"""
import sys
import time

sys.path.insert(0, ".")
import numpy as np

import paper_1104_5243_b200 as bp

Ls = [int(a) for a in sys.argv[1:]] or [128, 256, 512, 1024, 2048]
s = bp.Stack.baseline(n_views=496, isx=1248, isy=960)
n = 496
print("| config | L | offset | resident GUP/s (nominal) | visible GUP/s | resident ms | e2e ms | e2e GUP/s |")
print("|---|---|---|---|---|---|---|---|")
for L in Ls:
    off = (60.0, 0.0, 0.0) if L == 2048 else (0.0, 0.0, 0.0)
    cfg = {128: 1, 256: 2, 512: 3, 1024: 4, 2048: 5}.get(L, "-")
    with bp.GpuContext(L, 1248, 960, offset=off, count_visible=True, view_batch=32) as c:
        c.backproject_stack(s)
        _, vst = c.finish(readback=False)
    B = 124 if L >= 2048 else 248  # measured best resident launch size per L
    with bp.GpuContext(L, 1248, 960, offset=off, strict=False, view_batch=B,
                       ring_batches=(n + B - 1) // B) as c:
        c.upload_stack(s)
        c.time_resident(1)
        ms = min(c.time_resident(1)[0] for _ in range(3))
    host = bp.Volume.create(L)  # pinned host volume (32 GB at 2048^3)
    out = host.data
    with bp.GpuContext(L, 1248, 960, offset=off, strict=False, view_batch=0, views=n) as c:
        c.backproject_stack(s)
        c.finish(out=out)
        reps = []
        for _ in range(3):
            t0 = time.perf_counter()
            c.backproject_stack(s)
            c.finish(out=out)
            reps.append((time.perf_counter() - t0) * 1e3)
        e2e = min(reps)  # best of 3, like the resident column
        print("e2e reps", [round(r, 1) for r in reps], file=sys.stderr, flush=True)
    nom = n * L ** 3
    print(f"| {cfg} | {L} | {off[0]:+.0f} mm | {nom / ms / 1e6:.0f} | {vst.visible_updates / ms / 1e6:.0f} | "
          f"{ms:.1f} | {e2e:.1f} | {nom / e2e / 1e6:.0f} |", flush=True)
