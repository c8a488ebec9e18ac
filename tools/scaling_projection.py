"""Projected multi-GPU scaling from per-slab measurements on ONE B200 (not a scaling
measurement: no NVLink, no concurrent PCIe links).

For G = 1, 2, 4, 8 the volume is split into the work-balanced z-slabs every rank would
build (bp_partition_slabs); each slab is reconstructed on this GPU:
- resident: views in HBM, device-event time of the slab's kernels (bench `value` path);
- e2e: the slab's streamed reconstruction through the C ABI, uploading only the slab's
  detector-row window per view and reading back only its slab.
A G-GPU run takes as long as its slowest slab (each GPU has its own PCIe link on an
8 x B200 box), plus the fused slab gather (the final kernel stores into rank 0's volume
over NVLink; not modelled). Efficiency = T1 / (G * max_g T_g).
Usage: python tools/scaling_projection.py [L=1024]   (L = 2048: BASELINE config 5, grid offset +60 mm in x)
Env: GS (slab counts, default 1,2,4,8), E2E_BATCH (views per launch of a z-slab's streamed run when G > 1; default 62, the
measured best of 32/62/124 at 1024^3, G = 8: with 124 and the 5-batch deferred tail every
batch is deferred and the slab's upload no longer overlaps its compute), VERBOSE=1 (per-slab times), NO_VIEWS_HINT=1 (e2e without the band tail)."""
import os, sys, time
sys.path.insert(0, ".")
import paper_1104_5243_b200 as bp

L = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
off = (60.0, 0.0, 0.0) if L == 2048 else (0.0, 0.0, 0.0)  # BASELINE config 5: 2048^3 offset +60 mm in x
s = bp.Stack.baseline(n_views=496, isx=1248, isy=960)
px, mats = s.pixels, s.matrices
n = 496
B = 248 if L < 2048 else 124
EB = int(os.environ.get("E2E_BATCH", "62"))
verbose = os.environ.get("VERBOSE") == "1"
res, e2e = {}, {}
host = bp.Volume.create(L)  # one pinned host volume; each slab reads back into its part
print(f"| G | slab bounds | slowest slab, resident ms | projected resident efficiency | slowest slab, e2e ms | projected e2e efficiency |")
print("|---|---|---|---|---|---|")
GS = [int(g) for g in os.environ.get("GS", "1,2,4,8").split(",")]
for G in GS:
    bounds = [int(b) for b in bp.partition_slabs(mats, 1248, 960, L, G, offset=off)] if G > 1 else [0, L]
    tr, te = [], []
    for g in range(G):
        z0, z1 = bounds[g], bounds[g + 1]
        with bp.GpuContext(L, 1248, 960, device=0, offset=off, z_begin=z0, z_end=z1, strict=False, view_batch=B,
                           ring_batches=(n + B - 1) // B) as c:
            c.upload_stack(s)
            c.time_resident(1)
            tr.append(min(c.time_resident(1)[0] for _ in range(2)))
        out = host.data[z0:z1]
        eb = 0 if G == 1 else EB  # G = 1: the library default for a whole volume (62 from 1024^3 up)
        with bp.GpuContext(L, 1248, 960, device=0, offset=off, z_begin=z0, z_end=z1, strict=False, view_batch=eb,
                           views=n if os.environ.get("NO_VIEWS_HINT") != "1" else 0) as c:
            c.backproject_stack(s)
            c.finish(out=out)
            best = 1e30
            for _ in range(2):
                t0 = time.perf_counter()
                c.backproject_stack(s)
                c.finish(out=out)
                best = min(best, (time.perf_counter() - t0) * 1e3)
            te.append(best)
        if verbose:
            print(f"  G={G} slab [{z0},{z1}): resident {tr[-1]:.1f} ms, e2e {te[-1]:.1f} ms (batch {eb})",
                  flush=True)
    res[G], e2e[G] = max(tr), max(te)
    if 1 in res:
        print(f"| {G} | {bounds} | {res[G]:.1f} | {res[1] / (G * res[G]):.3f} | {e2e[G]:.1f} | "
              f"{e2e[1] / (G * e2e[G]):.3f} |", flush=True)
    else:
        print(f"| {G} | {bounds} | {res[G]:.1f} | - | {e2e[G]:.1f} | - |", flush=True)
