"""Per-z-chunk kernel cost at L (default 1024) on one B200, against the partitioner's cost
model (bp_slab_work), and the slab bounds each gives.

Every CH-slice chunk (default 32 = 4 block layers) is reconstructed resident (248-view
launches, best of 2 passes, device-event time).  The measured cost per slice (chunk time /
CH) is partitioned with bp_partition_by_cost; the model's with bp_partition_slabs.  For G in
GS both partitions' slabs are then timed the same way: the slowest slab against ideal
T1 / G is the projected resident efficiency (tools/scaling_projection.py).
Usage: python tools/slab_cost_probe.py [L]   Env: CH (32), GS (4,8), OUT (json path)."""
import json, os, sys
sys.path.insert(0, ".")
import numpy as np
import paper_1104_5243_b200 as bp

L = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
CH = int(os.environ.get("CH", "32"))
GS = [int(g) for g in os.environ.get("GS", "4,8").split(",")]
s = bp.Stack.baseline(n_views=496, isx=1248, isy=960)
mats = s.matrices
n, B = 496, 248


def resident_ms(z0, z1):
    with bp.GpuContext(L, 1248, 960, device=0, z_begin=z0, z_end=z1, strict=False, view_batch=B,
                       ring_batches=(n + B - 1) // B) as c:
        c.upload_stack(s)
        c.time_resident(1)
        return min(c.time_resident(1)[0] for _ in range(2))


t1 = resident_ms(0, L)
chunk = [resident_ms(z, min(L, z + CH)) for z in range(0, L, CH)]
model = bp.slab_work(mats, 1248, 960, L)
mchunk = [float(model[z:z + CH].sum()) for z in range(0, L, CH)]
scale = sum(chunk) / sum(mchunk)
print(f"L={L}: whole volume {t1:.1f} ms; sum of {len(chunk)} chunks {sum(chunk):.1f} ms")
print("| z-chunk | measured ms | model (scaled) ms | measured / model |")
print("|---|---|---|---|")
for i, (a, b) in enumerate(zip(chunk, mchunk)):
    print(f"| {i * CH}-{min(L, (i + 1) * CH)} | {a:.2f} | {b * scale:.2f} | {a / (b * scale):.3f} |")
cost = np.repeat(np.array(chunk) / CH, CH)[:L]
out = {"L": L, "chunk_slices": CH, "t1_ms": t1, "chunk_ms": chunk, "model_chunk": mchunk, "G": {}}
for G in GS:
    row = {}
    for name, bounds in (("model", [int(b) for b in bp.partition_slabs(mats, 1248, 960, L, G)]),
                         ("measured", [int(b) for b in bp.partition_by_cost(cost, G, 8)])):
        ts = [resident_ms(bounds[g], bounds[g + 1]) for g in range(G)]
        row[name] = {"bounds": bounds, "slab_ms": ts, "efficiency": t1 / (G * max(ts))}
        print(f"G={G} {name:8s} bounds {bounds}: slabs {[round(t, 1) for t in ts]} ms -> "
              f"efficiency {t1 / (G * max(ts)):.3f}", flush=True)
    out["G"][G] = row
if os.environ.get("OUT"):
    json.dump(out, open(os.environ["OUT"], "w"), indent=1)
