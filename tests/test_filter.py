"""FDK preprocessing (cosine weight + Ram-Lak row filter), SURVEY.md 8f rank 1.

The reference has no filter (SPEC.md:157 puts it outside the benchmark). Parity is therefore anchored on
oracle/filter_oracle.py, a float64 direct-convolution restatement of the published algorithm. That oracle
is itself pinned to analytic known answers:
- the ramp response to a cosine;
- the cosine weight at the detector centre.

Tolerances for the float32 FFT paths against the float64 oracle:
    max|d| <= 2e-5 * max|ref|   and   RMS(d) <= 2e-6 * max|ref|
The float32 FFT round-off is about log2(M) * 2^-24 of the row norm.
"""
import numpy as np
import pytest

import paper_1104_5243_b200 as bp
from oracle import filter_oracle as F
from tests.helpers import baseline_small, bitwise_equal, err_stats

FTOL_MAX, FTOL_RMS = 2e-5, 2e-6
SID, SDD = 750.0, 1200.0


def _ok(got, ref):
    emax, erms = err_stats(got, ref)
    assert emax <= FTOL_MAX and erms <= FTOL_RMS, (emax, erms)


# ---- oracle known answers (CPU) ---------------------------------------------------

@pytest.mark.parametrize("kappa", [0.05, 0.125, 0.3])
def test_oracle_ramp_response_to_cosine(kappa):
    # The band-limited ramp |f| passes cos(2 pi f u) with gain |f|.
    # With f = kappa / tau cycles/mm, the central output is kappa / tau * cos(.).
    # The truncated kernel tail (|h| ~ 1/n^2) limits the agreement to ~1e-3.
    isx, pitch = 4001, 0.5
    tau = pitch * SID / SDD
    u = np.arange(isx) - (isx - 1) / 2
    row = np.cos(2 * np.pi * kappa * u)
    # undo the cosine weight on a single central row so the input to the ramp is the cosine
    img = np.zeros((1, isx))
    img[0] = row / F.cosine_weight(isx, 1, SDD, pitch)[0]
    out = F.filter_views(img, SID, SDD, pitch)[0]
    c = slice(isx // 2 - 50, isx // 2 + 51)
    np.testing.assert_allclose(out[c], kappa / tau * row[c], rtol=0, atol=2e-3 * kappa / tau)


def test_oracle_cosine_weight_centre_and_symmetry():
    w = F.cosine_weight(5, 3, SDD, 0.32)
    assert w[1, 2] == 1.0
    assert np.allclose(w, w[::-1, ::-1])
    assert w.max() == 1.0 and w.min() < 1.0


def test_host_datagen_filter_matches_oracle():
    # bp_stack_generate_baseline(filter = 1) runs bph::cosine_ramp_filter (double FFT)
    raw, _ = baseline_small(n_views=2, shrink=16, filter=0)
    filt, _ = baseline_small(n_views=2, shrink=16, filter=1)
    ref = F.filter_views(raw, SID, SDD, 0.32 * 16)
    _ok(filt, ref)
    emax, _ = err_stats(filt, ref)
    assert emax <= 1e-6  # double FFT, float output


# ---- GPU ---------------------------------------------------------------------------

@pytest.mark.gpu
@pytest.mark.parametrize("isx,isy", [(2, 2), (3, 5), (9, 4), (64, 48), (100, 37), (1248, 6), (5000, 3)])
def test_gpu_filter_matches_oracle(isx, isy):
    rng = np.random.default_rng(isx * 7 + isy)
    px = rng.uniform(-1.0, 2.0, size=(2, isy, isx)).astype(np.float32)
    pitch = 400.0 / isx
    got = bp.filter_views(px, SID, SDD, pitch)
    _ok(got, F.filter_views(px, SID, SDD, pitch))


@pytest.mark.gpu
def test_gpu_filter_matches_host_filter_on_projections():
    raw, _ = baseline_small(n_views=3, shrink=4, filter=0)
    host, _ = baseline_small(n_views=3, shrink=4, filter=1)
    got = bp.filter_views(raw, SID, SDD, 0.32 * 4)
    _ok(got, host)
    # in place
    buf = raw.copy()
    bp.filter_views(buf, SID, SDD, 0.32 * 4, out=buf)
    assert bitwise_equal(buf, got)


@pytest.mark.gpu
def test_gpu_filter_linear_and_row_independent():
    rng = np.random.default_rng(5)
    a = rng.normal(size=(1, 10, 300)).astype(np.float32)
    b = rng.normal(size=(1, 10, 300)).astype(np.float32)
    fa, fb = bp.filter_views(a, SID, SDD, 1.0), bp.filter_views(b, SID, SDD, 1.0)
    fab = bp.filter_views(a + b, SID, SDD, 1.0)
    _ok(fab, fa.astype(np.float64) + fb)
    # A zero row stays zero up to the round-off it shares with its paired row:
    # rows (2i, 2i+1) are one complex FFT. A row's result does not depend on other views.
    z = a.copy()
    z[0, 3] = 0
    assert np.abs(bp.filter_views(z, SID, SDD, 1.0)[0, 3]).max() <= FTOL_RMS * np.abs(fa).max()
    two = bp.filter_views(np.concatenate([a, b]), SID, SDD, 1.0)
    assert bitwise_equal(two[0], fa[0]) and bitwise_equal(two[1], fb[0])


@pytest.mark.gpu
@pytest.mark.parametrize("view_batch,row_windows", [(32, True), (5, True), (8, False)])
def test_in_pipeline_filter_equals_prefiltered_views(view_batch, row_windows):
    # filtering inside the streaming pipeline (ring slot, row window) is bitwise
    # the same as filtering the whole stack first and streaming the result
    raw, mats = baseline_small(n_views=21, shrink=8, filter=0)
    geom = (SID, SDD, 0.32 * 8)
    pre = bp.filter_views(raw, *geom)
    n, isy, isx = raw.shape
    for L, z in ((48, (0, 0)), (48, (11, 30))):
        kw = dict(view_batch=view_batch, row_windows=row_windows, z_begin=z[0], z_end=z[1])
        with bp.GpuContext(L, isx, isy, filter=geom, **kw) as ctx:
            for k in range(n):
                ctx.backproject(raw[k], mats[k])
            got, _ = ctx.finish()
        with bp.GpuContext(L, isx, isy, **kw) as ctx:
            for k in range(n):
                ctx.backproject(pre[k], mats[k])
            ref, _ = ctx.finish()
        assert bitwise_equal(got, ref)


@pytest.mark.gpu
def test_reconstruct_ex_filter_and_fdk_quality():
    raw, mats = baseline_small(n_views=40, shrink=8, filter=0)
    host, _ = baseline_small(n_views=40, shrink=8, filter=1)
    geom = (SID, SDD, 0.32 * 8)
    got, st = bp.reconstruct_ex(bp.Stack.from_arrays(raw, mats), 64, filter=geom)
    pre = bp.filter_views(raw, *geom)
    ref, _ = bp.reconstruct_ex(bp.Stack.from_arrays(pre, mats), 64)
    assert bitwise_equal(got, ref)
    # against the double-precision host filter: the backprojected error stays
    # within the north_star fast-mode tolerance
    from oracle import oracle as O
    vol_host, _ = O.reconstruct(host, mats, 64)
    emax, erms = err_stats(got, vol_host)
    assert emax <= 1e-4 and erms <= 1e-6, (emax, erms)


@pytest.mark.gpu
def test_filter_rejects_bad_geometry():
    px = np.zeros((1, 4, 8), np.float32)
    with pytest.raises(bp.BPError) as e:
        bp.filter_views(px, SID, 0.0, 1.0)
    assert e.value.code == bp.BP_EINVAL
    with pytest.raises(bp.BPError):
        bp.filter_views(np.zeros((1, 2, 9000), np.float32), SID, SDD, 1.0)


@pytest.mark.gpu
def test_in_pipeline_filter_pair_ring_fast_mode():
    # the fast mode's pair ring is built on the prep stream from the FILTERED ring
    # slots: at 512^3 (32x32x8 pair-ring kernel) the in-pipeline filter must still equal
    # streaming prefiltered views, bitwise
    raw, mats = baseline_small(n_views=21, shrink=1, filter=0)
    geom = (SID, SDD, 0.32)
    pre = bp.filter_views(raw, *geom)
    n, isy, isx = raw.shape
    kw = dict(view_batch=8, strict=False)
    with bp.GpuContext(512, isx, isy, filter=geom, **kw) as ctx:
        for k in range(n):
            ctx.backproject(raw[k], mats[k])
        got, st = ctx.finish()
    with bp.GpuContext(512, isx, isy, **kw) as ctx:
        for k in range(n):
            ctx.backproject(pre[k], mats[k])
        ref, st2 = ctx.finish()
    assert st.tile_w == 152 and st.prep_launches == 2 * ((n + 7) // 8)  # filter + expansion
    assert st2.prep_launches == (n + 7) // 8
    assert bitwise_equal(got, ref)
