"""The band tail (bp_gpu_config.views) changes only WHEN the last views'
detector rows are uploaded and in which z-chunk order the deferred batches run, never
the per-voxel view order: every volume must be bitwise equal to the run without the
hint.  Covered: the BASELINE stack at 512^3 (pair ring, fast and strict), the raw-tile
kernels of small L, hints that under- and over-state the view count, a pageable
destination (bounce readback), a z-slab with row windows, two reconstructions in a row on
one context, and copy-semantics uploads (which do not withhold the tail).
"""
import numpy as np
import pytest

import paper_1104_5243_b200 as bp
from tests.helpers import bitwise_equal, small_stack

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def stack():
    return bp.Stack.baseline()


def _recon(px, mats, L, views_hint, *, strict, batch=32, copy=False, pageable_out=False,
           z=(0, 0), reps=1, filt=None):
    isy, isx = px.shape[1], px.shape[2]
    z0, z1 = z
    outs = []
    with bp.GpuContext(L, isx, isy, device=0, strict=strict, view_batch=batch, views=views_hint,
                       z_begin=z0, z_end=z1, filter=filt) as c:
        nz = c.z_end - c.z_begin
        for _ in range(reps):
            for k in range(px.shape[0]):
                c.backproject(px[k], mats[k], copy=copy)
            if pageable_out:
                out = np.empty((nz, L, L), np.float32)
            else:
                out = bp.Volume.create(L).data[:nz]
            vol, st = c.finish(out=out)
            assert st.fallback_pairs == 0
            outs.append(np.array(vol, copy=True))
    return outs


@pytest.mark.parametrize("strict", [False, True])
def test_band_tail_bitwise_at_512(stack, strict):
    px, mats = stack.pixels, stack.matrices
    ref = _recon(px, mats, 512, 0, strict=strict)[0]
    band = _recon(px, mats, 512, px.shape[0], strict=strict)[0]
    assert bitwise_equal(band, ref)


@pytest.mark.parametrize("L", [64, 128, 256])
def test_band_tail_small_L_and_raw_tile(L):
    px, mats = small_stack("spheres3", 90, 312, 240)
    ref = _recon(px, mats, L, 0, strict=False, batch=16)[0]
    for hint in (90, 60, 200):  # exact, understated (extra views stream view-major), overstated
        band = _recon(px, mats, L, hint, strict=False, batch=16)[0]
        assert bitwise_equal(band, ref), hint


def test_band_tail_copy_pageable_slab_and_repeat():
    px, mats = small_stack("spheres3", 70, 312, 240)
    L = 128
    ref = _recon(px, mats, L, 0, strict=True, batch=8)[0]
    a, b = _recon(px, mats, L, 70, strict=True, batch=8, pageable_out=True, reps=2)
    assert bitwise_equal(a, ref) and bitwise_equal(b, ref)
    # copy semantics: the tail is not withheld (host-paced views), same result
    c = _recon(px, mats, L, 70, strict=True, batch=8, copy=True)[0]
    assert bitwise_equal(c, ref)
    s = _recon(px, mats, L, 70, strict=True, batch=8, z=(40, 104))[0]
    assert bitwise_equal(s, ref[40:104])


def test_band_tail_bitwise_at_1024_whole_and_outer_slab(stack):
    # config 4: the two-y-row pair kernel, and a z-slab with the 186-view slab tail
    px, mats = stack.pixels, stack.matrices
    for z in ((0, 0), (0, 216)):
        ref = _recon(px, mats, 1024, 0, strict=False, z=z, batch=32 if z == (0, 0) else 62)[0]
        band = _recon(px, mats, 1024, px.shape[0], strict=False, z=z, batch=32 if z == (0, 0) else 62)[0]
        assert bitwise_equal(band, ref), z
        del ref, band


def test_band_tail_odd_width_and_filter():
    # an odd detector width (ring pitch != width: per-view band copies) and FDK filtering
    # (band runs of whole row pairs, filtered band by band) both stay bitwise
    px, mats = small_stack("spheres3", 60, 250, 200)
    ref = _recon(px, mats, 128, 0, strict=False, batch=16)[0]
    assert bitwise_equal(_recon(px, mats, 128, 60, strict=False, batch=16)[0], ref)
    geom = (750.0, 1200.0, 0.32 * 1248.0 / 250)
    ref = _recon(px, mats, 128, 0, strict=False, batch=16, filt=geom)[0]
    assert bitwise_equal(_recon(px, mats, 128, 60, strict=False, batch=16, filt=geom)[0], ref)
