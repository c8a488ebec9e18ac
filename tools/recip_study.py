"""Reciprocal accuracy ladder on the GPU (acceptance.cpp:169-188).

It reconstructs the BASELINE stack (496 views of 1248x960) at L (default 256, BASELINE config 2) with every
reciprocal strategy and prints the PSNR of each against the strict, bitwise-reference volume. The
reference's acceptance criterion 4 asks for:
- PSNR(approx12_nr) >= 90 dB;
- PSNR(approx12) at least 20 dB below it.

The GPU adds two arithmetic paths:
- the tiled kernel's fast mode (exact reciprocal, FMA-lerp bilinear);
- the raw hardware rcp.approx.ftz.f32 (BP_RECIP_HW_APPROX).

Usage: python tools/recip_study.py [L]
"""
import sys
import time

sys.path.insert(0, ".")
import numpy as np

import paper_1104_5243_b200 as bp

L = int(sys.argv[1]) if len(sys.argv) > 1 else 256
s = bp.Stack.baseline(n_views=496, isx=1248, isy=960)


def run(**kw):
    t0 = time.perf_counter()
    out, st = bp.reconstruct_ex(s, L, **kw)
    return out, time.perf_counter() - t0


exact, t_exact = run(strict=True)
peak = float(np.abs(exact).max())
rows = [("exact 1/w, strict (== reference bitwise)", exact, t_exact)]
fast, t = run(strict=False)
rows.append(("exact 1/w, fast mode (FMA-lerp bilinear)", fast, t))
v, t = run(strict=False, recip_mode=bp.BP_RECIP_HW_APPROX)
rows.append(("hardware rcp.approx, fast mode (tiled kernel)", v, t))
for mode, name in ((bp.BP_RECIP_APPROX12_NR, "approx12_nr (recip.hpp:20-23)"),
                   (bp.BP_RECIP_APPROX12, "approx12 (recip.hpp:14-18)"),
                   (bp.BP_RECIP_HW_APPROX, "hardware rcp.approx.ftz.f32 (GPU only)")):
    v, t = run(recip_mode=mode)
    rows.append((name, v, t))
print(f"| reciprocal (L={L}, 496 views) | PSNR vs exact (dB) | max abs diff / max abs ref | RMS / max abs ref |")
print("|---|---|---|---|")
for name, v, t in rows:
    d = v.astype(np.float64) - exact
    mse = float(np.mean(d * d))
    psnr = float("inf") if mse == 0 else 10 * np.log10(peak * peak / mse)
    print(f"| {name} | {psnr:.1f} | {np.abs(d).max() / peak:.2e} | {np.sqrt(mse) / peak:.2e} |")
