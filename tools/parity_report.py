"""Comparison harness: the GPU path against the CPU oracle at every BASELINE config.

The oracle is oracle/bp_oracle.c, itself pinned bitwise to the reference sources in
tests/test_oracle.py. What gets compared:
- configs 1-2: full volumes, strict against the oracle;
- configs 3-5: sampled lines, strict against the oracle;
- every config: the fast and hardware-reciprocal tiers against strict (== reference) over the FULL volume,
  on the device.

Writes a markdown table to stdout. Test infrastructure: it imports the oracle.
Usage: python tools/parity_report.py [L ...]
"""
import sys

sys.path.insert(0, ".")
import numpy as np

import paper_1104_5243_b200 as bp
from oracle import oracle as O

Ls = [int(a) for a in sys.argv[1:]] or [128, 256, 512, 1024, 2048]
s = bp.Stack.baseline()
px, mats = s.pixels, s.matrices


def ctx(L, off, **kw):
    c = bp.GpuContext(L, 1248, 960, offset=off, **kw)
    c.backproject_stack(s)
    _, st = c.finish(readback=False)
    return c, st


print("| config | L | strict vs oracle | fast vs reference: max / RMS of max\\|ref\\| | hw-rcp tier: max / RMS | fallback pairs |")
print("|---|---|---|---|---|---|")
for L in Ls:
    off = (60.0, 0.0, 0.0) if L == 2048 else (0.0, 0.0, 0.0)
    cfg = {128: 1, 256: 2, 512: 3, 1024: 4, 2048: 5}.get(L, "-")
    strict, sst = ctx(L, off, strict=True)
    fb = int(sst.fallback_pairs)
    if L <= 256:
        ref, _ = O.reconstruct(px, mats, L, offset=off)
        c2 = bp.GpuContext(L, 1248, 960, offset=off, strict=True)
        c2.backproject_stack(s)
        got, st = c2.finish()
        c2.close()
        nb = int(np.count_nonzero(got.view(np.uint32) != ref.view(np.uint32)))
        sv = f"full volume: {'bitwise' if nb == 0 else f'{nb} voxels differ'}"
    else:
        rng = np.random.default_rng(L)
        n = 32 if L <= 1024 else 12
        ys = rng.integers(0, L, n).astype(np.int32)
        zs = rng.integers(0, L, n).astype(np.int32)
        got = strict.read_lines(ys, zs)
        ref = O.reconstruct_lines(px, mats, L, ys, zs, offset=off)
        nb = int(np.count_nonzero(got.view(np.uint32) != ref.view(np.uint32)))
        sv = f"{n} sampled lines: {'bitwise' if nb == 0 else f'{nb} voxels differ'}"
    out = []
    for kw in (dict(strict=False), dict(strict=False, recip_mode=bp.BP_RECIP_HW_APPROX)):
        c, cst = ctx(L, off, **kw)
        fb += int(cst.fallback_pairs)
        mx, peak, sq, nbit = c.compare_with(strict)
        out.append(f"{mx / peak:.1e} / {sq / peak:.1e}")
        c.close()
    strict.close()
    print(f"| {cfg} | {L}{' +60 mm' if off[0] else ''} | {sv} | {out[0]} | {out[1]} | {fb} |", flush=True)
