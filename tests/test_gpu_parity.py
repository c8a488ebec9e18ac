"""GPU parity: the sm_100a kernels against the CPU oracle (oracle/bp_oracle.c,
itself pinned bitwise to the reference in tests/test_oracle.py).

strict mode must be BITWISE identical to bp::reconstruct (proj/src/scheduler.cpp:24-133);
fast mode must satisfy the north_star tolerance
    max|d| <= 1e-4 * max|ref|   and   RMS <= 1e-6 * max|ref|.
Known-answer cases port proj/tests/test_kernel.cpp:74-198.
"""
import numpy as np
import pytest

import paper_1104_5243_b200 as bp
from oracle import oracle as O
from tests.helpers import (TOL_MAX, TOL_RMS, baseline_small, bitwise_equal, err_stats,
                           random_image, random_matrix, small_stack)

pytestmark = pytest.mark.gpu


def gpu_recon(px, mats, L, *, offset=(0.0, 0.0, 0.0), strict=True, kernel=0, view_batch=32,
              distance_weight=True, copy=True, z_begin=0, z_end=0, count_visible=False,
              row_windows=True):
    n, isy, isx = px.shape
    with bp.GpuContext(L, isx, isy, offset=offset, strict=strict, kernel=kernel,
                       view_batch=view_batch, distance_weight=distance_weight, z_begin=z_begin,
                       z_end=z_end, count_visible=count_visible, row_windows=row_windows) as ctx:
        for k in range(n):
            ctx.backproject(px[k], mats[k], copy=copy)
        vol, st = ctx.finish()
    return vol, st


# ---- reciprocal -------------------------------------------------------------

def test_rcp_pair_matches_frcp_rn():
    # every float in [1, 2) and in [512, 1024) (w at the BASELINE geometry)
    assert bp.selftest_rcp(0x3F800000, 0x40000000) == 0
    assert bp.selftest_rcp(0x44000000, 0x44800000) == 0


# ---- bitwise strict parity ------------------------------------------------------

@pytest.mark.parametrize("L", [16, 24, 32, 48, 64])
@pytest.mark.parametrize("kernel", [0, 1])
def test_strict_bitwise_small_stack(L, kernel):
    px, mats = small_stack("spheres3", 6, 64, 48)
    ref, _ = O.reconstruct(px, mats, L)
    got, st = gpu_recon(px, mats, L, kernel=kernel)
    assert bitwise_equal(got, ref), err_stats(got, ref)


@pytest.mark.parametrize("L", [32, 64, 128])
def test_strict_bitwise_baseline_shaped(L):
    px, mats = baseline_small(n_views=40, shrink=4)
    ref, _ = O.reconstruct(px, mats, L)
    got, st = gpu_recon(px, mats, L, strict=True)
    assert st.fallback_pairs == 0
    assert bitwise_equal(got, ref), err_stats(got, ref)


def test_strict_bitwise_full_detector_128():
    # config 1 geometry (1248x960 detector) on a reduced view count
    px, mats = baseline_small(n_views=24, shrink=1)
    ref, _ = O.reconstruct(px, mats, 128)
    got, st = gpu_recon(px, mats, 128, strict=True)
    assert st.tile_pairs > 0 and st.fallback_pairs == 0
    assert bitwise_equal(got, ref), err_stats(got, ref)


def test_strict_bitwise_offset_grid():
    # config 5 shape: grid centre offset laterally (+60 mm), lines partly off-detector
    px, mats = baseline_small(n_views=24, shrink=4)
    ref, _ = O.reconstruct(px, mats, 64, offset=(60.0, 0.0, 0.0))
    got, st = gpu_recon(px, mats, 64, offset=(60.0, 0.0, 0.0))
    assert st.skipped_pairs > 0
    assert bitwise_equal(got, ref), err_stats(got, ref)


@pytest.mark.parametrize("view_batch", [1, 5, 32, 64])
def test_batch_invariance(view_batch):
    # projection blocking invariance (test_scheduler.cpp:63-133, acceptance C3)
    px, mats = baseline_small(n_views=37, shrink=4)
    ref, _ = O.reconstruct(px, mats, 64)
    got, _ = gpu_recon(px, mats, 64, view_batch=view_batch)
    assert bitwise_equal(got, ref)


def test_plain_fx_switch():
    # distance_weight = 0 (test_kernel.cpp:185-198)
    px, mats = small_stack("shell", 5, 56, 48)
    ref, _ = O.reconstruct(px, mats, 32, distance_weight=False)
    for kernel in (0, 1):
        got, _ = gpu_recon(px, mats, 32, distance_weight=False, kernel=kernel)
        assert bitwise_equal(got, ref)


# ---- fast mode tolerance ----------------------------------------------------------

@pytest.mark.parametrize("L", [64, 128])
def test_fast_within_tolerance(L):
    px, mats = baseline_small(n_views=48, shrink=2)
    ref, _ = O.reconstruct(px, mats, L)
    got, _ = gpu_recon(px, mats, L, strict=False)
    emax, erms = err_stats(got, ref)
    assert emax <= TOL_MAX and erms <= TOL_RMS, (emax, erms)


# ---- known answers (test_kernel.cpp) ------------------------------------------------

def _single_view(img, A, L, **kw):
    return gpu_recon(img[None], np.asarray(A, np.float64)[None], L, **kw)[0]


def test_zero_image_noop():
    img = np.zeros((64, 64), np.float32)
    A = random_matrix(17, 64, 64)
    vol = _single_view(img, A, 32)
    assert not vol.any()


def test_pixel_centre_hits_accumulate_c_r2():
    # test_kernel.cpp:84-101: u = x-ish, v on a pixel centre, w = 1
    L = 256
    g = O.Grid.cube(L)
    wz136 = g.oz + 136 * g.MM
    A = [1, 0, 0, 0, 1, 0, 0, 0, 0, 127.5, 127.5 - wz136, 1]
    c = 0.8125
    img = np.full((32, 32), c, np.float32)
    for kernel in (0, 1):
        vol = _single_view(img, A, L, kernel=kernel)
        line = vol[136, 130]
        for x in range(128, 141):
            u = np.float32(g.ox + x * g.MM) + np.float32(127.5)
            if u == np.floor(u) and 0 <= u < 31:
                assert line[x] == np.float32(c)
        ref = np.zeros(L, np.float32)
        O.line_update(ref, img, np.asarray(A, np.float32), L, 130, 136, 0, L - 1)
        assert bitwise_equal(line, ref)


def test_fully_outside_contributes_exact_zero():
    # test_kernel.cpp:151-167: u = wx + 5000, far off-detector for every voxel
    img = random_image(32, 32, 55, 0.5, 2.0)
    A = [1, 0, 0, 0, 1, 0, 0, 0, 0, 5000.0, 0.0, 1.0]
    for kernel in (0, 1):
        vol = _single_view(img, A, 16, kernel=kernel)
        assert not vol.any()


def test_partially_outside_matches_guarded_double_oracle():
    # test_kernel.cpp:169-183: the projected line straddles the left image edge
    img = random_image(24, 24, 77, 0.5, 1.5)
    A = [0.125, 0, 0, 0, 0, 0, 0, 0.0, 0, 10.0, 12.3, 1.0]
    L = 32
    vol = _single_view(img, A, L)
    g = O.Grid.cube(L)
    f = np.asarray(A, np.float32).astype(np.float64)
    wy, wz = g.oy + 4 * g.MM, g.oz + 4 * g.MM
    for x in range(L):
        wx = g.ox + x * g.MM
        uw = f[0] * wx + f[3] * wy + f[6] * wz + f[9]
        vw = f[1] * wx + f[4] * wy + f[7] * wz + f[10]
        w = f[2] * wx + f[5] * wy + f[8] * wz + f[11]
        u, v = uw / w, vw / w
        iu, iv = int(np.floor(u)), int(np.floor(v))
        sx, sy = u - iu, v - iv

        def pix(a, b):
            return float(img[b, a]) if 0 <= a < 24 and 0 <= b < 24 else 0.0
        fx = sx * (sy * pix(iu + 1, iv + 1) + (1 - sy) * pix(iu + 1, iv)) + \
            (1 - sx) * (sy * pix(iu, iv + 1) + (1 - sy) * pix(iu, iv))
        ref = fx / (w * w)
        assert abs(vol[4, 4, x] - ref) <= 1e-5 * max(1.0, abs(ref))


# ---- clip statistics ------------------------------------------------------------------

def test_visible_update_count_matches_clip_stats():
    px, mats = baseline_small(n_views=16, shrink=4)
    for L in (32, 64):
        ref = int(O.visible_updates(mats, px.shape[2], px.shape[1], L).sum())
        _, st = gpu_recon(px, mats, L, count_visible=True)
        assert st.visible_updates == ref
        if O.ref_available():
            assert ref == O.ref_clip_total(mats, px.shape[2], px.shape[1], L)


# ---- pipeline / API invariance -----------------------------------------------------

def test_copy_and_async_paths_identical():
    px, mats = baseline_small(n_views=20, shrink=4)
    a, _ = gpu_recon(px, mats, 64, copy=True)
    b, _ = gpu_recon(px, mats, 64, copy=False)
    assert bitwise_equal(a, b)


def test_bp_reconstruct_drop_in():
    # reference C ABI (capi.cpp:109-166) through the GPU
    px, mats = small_stack("spheres3", 4, 48, 40)
    st = bp.Stack.from_arrays(px, mats)
    vol, rs = bp.reconstruct(st, bp.recon_params(16, block_b=1))
    ref, _ = O.reconstruct(px, mats, 16)
    assert bitwise_equal(vol.data, ref)
    assert rs.voxel_updates == 4 * 16 ** 3
    assert rs.writeback_stores == 4 * 16 ** 3
    assert rs.gflops == pytest.approx(31.0 * rs.gups)
    # repeat: cached context, fresh volume
    vol2, _ = bp.reconstruct(st, bp.recon_params(16, block_b=3))
    assert bitwise_equal(vol2.data, ref)


def test_slab_and_virtual_slabs_equal_full():
    px, mats = baseline_small(n_views=24, shrink=4)
    stack = bp.Stack.from_arrays(px, mats)
    full, _ = bp.reconstruct_ex(stack, 64)
    for G in (2, 3, 5):
        got, st = bp.reconstruct_ex(stack, 64, virtual_slabs=G)
        assert bitwise_equal(got, full), G
        assert st.h2d_bytes <= G * px.nbytes
    ref, _ = O.reconstruct(px, mats, 64)
    assert bitwise_equal(full, ref)


def test_explicit_slab_context():
    px, mats = baseline_small(n_views=12, shrink=4)
    ref, _ = O.reconstruct(px, mats, 64, z0=20, z1=41)
    got, st = gpu_recon(px, mats, 64, z_begin=20, z_end=41)
    assert got.shape == (21, 64, 64)
    assert bitwise_equal(got, ref)
    assert st.h2d_bytes < px.nbytes  # row windows trimmed the upload


def test_determinism_repeat():
    px, mats = baseline_small(n_views=16, shrink=4)
    a, _ = gpu_recon(px, mats, 64, strict=False)
    b, _ = gpu_recon(px, mats, 64, strict=False)
    assert bitwise_equal(a, b)


def test_resident_timing_path_matches_streaming():
    px, mats = baseline_small(n_views=40, shrink=4)
    n, isy, isx = px.shape
    with bp.GpuContext(64, isx, isy, ring_batches=2, view_batch=32) as ctx:
        ctx.upload_views(px, mats)
        ms, st = ctx.time_resident(iters=2)
        assert ms > 0 and st.views == 2 * n
        ptr = ctx.volume_device_ptr()
        assert ptr != 0
        vol, _ = ctx.finish()  # no views queued: volume keeps the resident result? (reset)
    ref, _ = O.reconstruct(px, mats, 64)
    got, _ = gpu_recon(px, mats, 64)
    assert bitwise_equal(got, ref)


def test_invalid_geometry_rejected():
    px, mats = small_stack("point", 2, 24, 24)
    bad = mats.copy()
    bad[1] = [1, 0, 0, 0, 1, 0, 0, 0, 0, 0, 0, -1]
    with pytest.raises(bp.BPError) as e:
        gpu_recon(px, bad, 8)
    assert e.value.code == bp.BP_EVERIFY


def test_approx_recip_modes_match_reference_ladder():
    # recip.hpp:14-23 restated on the GPU (simple kernel); PSNR ordering of acceptance C4
    px, mats = small_stack("spheres3", 4, 48, 40)
    st = bp.Stack.from_arrays(px, mats)
    exact, _ = bp.reconstruct(st, bp.recon_params(16))
    nr, _ = bp.reconstruct(st, bp.recon_params(16, recip_mode=bp.BP_RECIP_APPROX12_NR))
    ap, _ = bp.reconstruct(st, bp.recon_params(16, recip_mode=bp.BP_RECIP_APPROX12))
    p_nr, p_12 = nr.psnr(exact), ap.psnr(exact)
    assert p_nr >= 90.0 and p_12 <= p_nr - 20.0 and p_12 > 20.0


@pytest.mark.parametrize("mode", [1, 2])
def test_approx_recip_modes_bitwise_vs_golden(mode):
    import os
    g = np.load(os.path.join(os.path.dirname(__file__), "golden", "recon_recip_16.npz"))
    st = bp.Stack.from_arrays(g["pixels"], g["mats"])
    got, _ = bp.reconstruct(st, bp.recon_params(16, recip_mode=mode))
    assert bitwise_equal(got.data, g["approx12" if mode == 1 else "approx12_nr"])


@pytest.mark.parametrize("mode", [1, 2])
def test_approx_recip_modes_bitwise_vs_reference(mode):
    # recip_approx12 / recip_approx12_nr (recip.hpp:14-23) are restated operation for
    # operation on the GPU (double frexp / rint / ldexp, then the float Newton step), so
    # the whole reconstruction is bitwise the reference's bp::reconstruct with that mode
    if not O.ref_available():
        pytest.skip("oracle/_ref not built")
    px, mats = baseline_small(n_views=12, shrink=8)
    ref, _ = O.ref_reconstruct(px, mats, 32, threads=4, recip=mode)
    got, _ = bp.reconstruct(bp.Stack.from_arrays(px, mats), bp.recon_params(32, recip_mode=mode))
    assert bitwise_equal(got.data, ref), err_stats(got.data, ref)


# ---- clip table / clip_cache (precompute.cpp:51-134, capi.cpp:133-143) ----------

def test_gpu_clip_table_matches_reference_golden():
    import os
    g = np.load(os.path.join(os.path.dirname(__file__), "golden", "clip_ranges_baseline_32.npz"))
    mats = g["mats"]
    st = bp.Stack.from_arrays(np.zeros((mats.shape[0], 120, 156), np.float32), mats)
    ranges, total = bp.clip_table(st, 32)
    assert np.array_equal(ranges, g["ranges"])
    assert total == int(g["total"])


def test_gpu_clip_table_matches_live_reference():
    if not O.ref_available():
        pytest.skip("oracle/_ref not built")
    px, mats = small_stack("spheres3", 5, 48, 40)
    st = bp.Stack.from_arrays(px, mats)
    for L in (20, 33):
        ranges, total = bp.clip_table(st, L)
        ref_r, ref_t = O.ref_clip_table(mats, 48, 40, L)
        assert np.array_equal(ranges, ref_r) and total == ref_t


def test_clip_cache_written_then_reused(tmp_path):
    import os
    px, mats = baseline_small(n_views=10, shrink=8)
    st = bp.Stack.from_arrays(px, mats)
    cache = str(tmp_path / "t.bpct")
    v1, s1 = bp.reconstruct(st, bp.recon_params(24, clip=1, clip_cache=cache))
    assert os.path.exists(cache)
    m1 = os.path.getmtime(cache)
    v2, s2 = bp.reconstruct(st, bp.recon_params(24, clip=1, clip_cache=cache))
    assert os.path.getmtime(cache) == m1                 # reused, not rewritten
    assert bitwise_equal(v1.data, v2.data)
    assert s1.voxel_updates == s2.voxel_updates == int(O.visible_updates(mats, 156, 120, 24).sum())
    assert s1.clip_reduction > 0
    # a table for another grid is rejected (scheduler.cpp:40-42)
    with pytest.raises(bp.BPError) as e:
        bp.reconstruct(st, bp.recon_params(16, clip=1, clip_cache=cache))
    assert e.value.code == bp.BP_EVERIFY


def test_block_b_beyond_kernel_batch_is_clamped_not_rejected():
    # the reference accepts any block_b >= 1; results are batch-invariant (scheduler.cpp:77-100)
    px, mats = baseline_small(n_views=20, shrink=8)
    st = bp.Stack.from_arrays(px, mats)
    a, sa = bp.reconstruct(st, bp.recon_params(24, block_b=500))
    b, _ = bp.reconstruct(st, bp.recon_params(24, block_b=7))
    assert bitwise_equal(a.data, b.data)
    assert sa.writeback_stores == 24 ** 3  # one batch of 20 views


@pytest.mark.parametrize("debug", ["1", "2"])
def test_global_fallback_path_bitwise(debug, monkeypatch):
    # Every (block, view) pair can be forced through the guarded global-memory fallback:
    # bit 0 forces it at the producer, bit 1 at the consumers. The fallback uses the reference
    # clamp and arithmetic (kernel.cpp:53-82) and must stay bitwise.
    px, mats = baseline_small(n_views=10, shrink=8)
    ref, _ = O.reconstruct(px, mats, 32)
    monkeypatch.setenv("BP_DEBUG", debug)
    got, st = gpu_recon(px, mats, 32)
    assert st.fallback_pairs > 0 or debug == "2"
    assert bitwise_equal(got, ref), err_stats(got, ref)


@pytest.mark.parametrize("seed", list(range(8)))
def test_strict_bitwise_random_geometry_fuzz(seed):
    # random single-view geometries (test_support.hpp:32-45) stacked into one scan, random
    # grid offsets and edge lengths (odd L takes the simple kernel): strict mode stays bitwise
    rng = np.random.default_rng(1000 + seed)
    isx, isy = int(rng.integers(24, 200)), int(rng.integers(24, 160))
    n = int(rng.integers(1, 9))
    mats = np.stack([random_matrix(int(rng.integers(0, 1 << 30)), isx, isy) for _ in range(n)])
    px = np.stack([random_image(isx, isy, int(rng.integers(0, 1 << 30)), -1.0, 2.0) for _ in range(n)])
    L = int(rng.choice([16, 31, 48, 64, 96]))
    off = tuple(float(v) for v in rng.uniform(-40, 40, size=3))
    ref, _ = O.reconstruct(px, mats, L, offset=off)
    got, _ = gpu_recon(px, mats, L, offset=off, view_batch=int(rng.integers(1, 9)))
    assert bitwise_equal(got, ref), err_stats(got, ref)


def test_hw_rcp_tiled_fast_mode_within_tolerance():
    # the opt-in BP_RECIP_HW_APPROX tier on the tiled kernel stays inside the north_star bounds
    px, mats = baseline_small(n_views=48, shrink=2)
    ref, _ = O.reconstruct(px, mats, 128)
    n, isy, isx = px.shape
    with bp.GpuContext(128, isx, isy, strict=False, recip_mode=bp.BP_RECIP_HW_APPROX) as ctx:
        for k in range(n):
            ctx.backproject(px[k], mats[k])
        got, st = ctx.finish()
    assert st.tile_pairs > 0  # tiled, not the simple kernel
    emax, erms = err_stats(got, ref)
    assert emax <= TOL_MAX and erms <= TOL_RMS, (emax, erms)
    assert erms > 0  # it is an approximation


def test_recon_stats_per_device_split():
    # RunStats' per-thread min/max (scheduler.hpp:22-30) become per-device min/max; with
    # one device both equal the total, with virtual slabs on one device likewise
    px, mats = baseline_small(n_views=8, shrink=8)
    st = bp.Stack.from_arrays(px, mats)
    _, rs = bp.reconstruct(st, bp.recon_params(32, clip=1))
    assert rs.thread_updates_min == rs.thread_updates_max == rs.voxel_updates
    _, rs0 = bp.reconstruct(st, bp.recon_params(32, clip=0))
    assert rs0.thread_updates_min == rs0.thread_updates_max == rs0.voxel_updates == 8 * 32 ** 3
    out, gs = bp.reconstruct_ex(st, 32, virtual_slabs=3, count_visible=True)
    assert gs.device_updates_min == gs.device_updates_max == gs.visible_updates


def test_multi_device_threads_on_one_gpu():
    # bp_gpu_set_devices([0, 0]): two host worker threads drive two slab contexts
    # concurrently (bp_reconstruct_ex, one thread per listed device); independent kernels
    px, mats = baseline_small(n_views=20, shrink=4)
    stack = bp.Stack.from_arrays(px, mats)
    ref, _ = O.reconstruct(px, mats, 64)
    try:
        bp.set_devices([0, 0])
        got, st = bp.reconstruct_ex(stack, 64, count_visible=True)
        assert bitwise_equal(got, ref)
        assert st.device_updates_min <= st.device_updates_max
        assert st.device_updates_min + st.device_updates_max == st.visible_updates
        vol, rs = bp.reconstruct(stack, bp.recon_params(64, clip=1))
        assert bitwise_equal(vol.data, ref)
        assert rs.thread_updates_min + rs.thread_updates_max == rs.voxel_updates
    finally:
        bp.set_devices([0])


def test_concurrent_bp_reconstruct_calls_from_threads():
    # reentrant across contexts (SURVEY 8b threading row): two host threads call
    # bp_reconstruct at once on different stacks; results equal the serial ones and a
    # failing call's message stays on its own thread (thread-local bp_last_error)
    import threading
    pa, ma = baseline_small(n_views=12, shrink=8, seed=1)
    pb, mb = baseline_small(n_views=12, shrink=8, seed=2)
    sa, sb = bp.Stack.from_arrays(pa, ma), bp.Stack.from_arrays(pb, mb)
    ref_a, _ = bp.reconstruct(sa, bp.recon_params(32))
    ref_b, _ = bp.reconstruct(sb, bp.recon_params(32))
    ra, rb = ref_a.data.copy(), ref_b.data.copy()
    out, errs = {}, {}

    def work(name, st, p):
        try:
            for _ in range(3):
                v, _ = bp.reconstruct(st, p)
                out[name] = v.data.copy()
        except bp.BPError as e:
            errs[name] = (e.code, str(e))

    bad = bp.recon_params(32, lanes=5)  # BP_EINVAL in this thread only
    ts = [threading.Thread(target=work, args=("a", sa, bp.recon_params(32))),
          threading.Thread(target=work, args=("b", sb, bp.recon_params(32))),
          threading.Thread(target=work, args=("c", sa, bad))]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert bitwise_equal(out["a"], ra) and bitwise_equal(out["b"], rb)
    assert errs.get("c", (None,))[0] == bp.BP_EINVAL and "lane" in errs["c"][1]
    assert "a" not in errs and "b" not in errs


@pytest.mark.parametrize("isx,isy,L", [(58, 47, 32), (250, 173, 64), (2048, 64, 128)])
def test_strict_bitwise_odd_and_wide_detectors(isx, isy, L):
    # pitch != isx (2-D H2D copies into a 16-B aligned ring), odd row counts, and a wide
    # detector whose footprints exceed the tile (fallback pairs) -- all bitwise
    s = bp.Stack.generate("spheres3", 5, isx, isy, 750.0, 1200.0, 0.32 * 1248.0 / isx)
    px, mats = s.pixels.copy(), s.matrices.copy()
    ref, _ = O.reconstruct(px, mats, L)
    for kw in (dict(), dict(row_windows=False), dict(view_batch=2)):
        got, st = gpu_recon(px, mats, L, **kw)
        assert bitwise_equal(got, ref), (kw, err_stats(got, ref))


def test_module_config_errors():
    # bp_gpu_load validation: every rejected configuration returns BP_EINVAL with a message
    bad = [dict(view_batch=257), dict(z_begin=10, z_end=5), dict(z_begin=-1, z_end=4),
           dict(recip_mode=7), dict(filter=(750.0, 0.0, 0.3))]
    for kw in bad:
        with pytest.raises(bp.BPError) as e:
            bp.GpuContext(32, 64, 48, **kw)
        assert e.value.code == bp.BP_EINVAL, kw
    # the largest batch is accepted and batch-invariant
    px, mats = baseline_small(n_views=260, shrink=16)
    ref, _ = O.reconstruct(px, mats, 32)
    got, _ = gpu_recon(px, mats, 32, view_batch=256)
    assert bitwise_equal(got, ref)
