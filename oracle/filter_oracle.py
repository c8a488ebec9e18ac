"""FDK projection preprocessing oracle -- TEST INFRASTRUCTURE ONLY.

The reference has no filter. It benchmarks backprojection of already-filtered projections:
PAPER.md:104-108 names the "2D pre-processing steps" of the Feldkamp algorithm, and SPEC.md:157 puts them
outside the benchmark. SURVEY.md 8f rank 1 asks for them on the GPU, so this module restates the published
algorithm in float64 numpy, independently of the product's FFT route. It follows Feldkamp, Davis & Kress
(1984) and Kak & Slaney, *Principles of Computerized Tomographic Imaging*, ch. 3:

* cosine weight: p~(u, v) = p(u, v) * sdd / sqrt(sdd^2 + du^2 + dv^2), where du and dv are measured from
  the detector centre in mm;
* Ram-Lak kernel sampled at the isocentre spacing tau = pitch * sid / sdd:
  h[0] = 1/(4 tau^2), h[n odd] = -1/(pi^2 n^2 tau^2), h[n even] = 0;
* each row is convolved linearly with h (|n| <= isx-1) and scaled by tau: p'(u) = tau * sum_u' h[u-u'] p~(u').

This is a direct spatial-domain convolution, with no FFT. It checks the product's zero-padded FFT
convolution (host bph::cosine_ramp_filter and GPU bp_filter.cu) to floating-point tolerance.

Parity is not pinned to the reference, because the reference has no such function. The pins are
analytic known answers instead; see tests/test_filter.py.
"""
from __future__ import annotations

import numpy as np


def ramp_kernel(isx: int, tau: float) -> np.ndarray:
    """h[n] for n = -(isx-1) .. isx-1 (index n + isx - 1)."""
    n = np.arange(-(isx - 1), isx, dtype=np.float64)
    h = np.zeros_like(n)
    h[n == 0] = 1.0 / (4.0 * tau * tau)
    odd = (np.abs(n) % 2) == 1
    h[odd] = -1.0 / (np.pi ** 2 * n[odd] ** 2 * tau * tau)
    return h


def cosine_weight(isx: int, isy: int, sdd: float, pitch: float) -> np.ndarray:
    du = (np.arange(isx, dtype=np.float64) - 0.5 * (isx - 1)) * pitch
    dv = (np.arange(isy, dtype=np.float64) - 0.5 * (isy - 1)) * pitch
    return sdd / np.sqrt(sdd * sdd + du[None, :] ** 2 + dv[:, None] ** 2)


def filter_views(pixels: np.ndarray, sid: float, sdd: float, pitch: float) -> np.ndarray:
    """(n, isy, isx) or (isy, isx) float images -> float64 filtered images."""
    px = np.asarray(pixels, np.float64)
    single = px.ndim == 2
    if single:
        px = px[None]
    n, isy, isx = px.shape
    tau = pitch * sid / sdd
    h = ramp_kernel(isx, tau)
    w = cosine_weight(isx, isy, sdd, pitch)
    out = np.empty_like(px)
    for k in range(n):
        x = px[k] * w
        for v in range(isy):
            # full linear convolution; output u sits at index u + isx - 1
            out[k, v] = tau * np.convolve(x[v], h)[isx - 1:2 * isx - 1]
    return out[0] if single else out
