"""Edge cases of the streaming module ABI (include/bp_gpu.h), against the C oracle
(bp::reconstruct restated, oracle/bp_oracle.c): an empty reconstruction, a single view,
a batch of one view per launch, a view count hint larger than the stack with nothing
queued, and a context reused across different stacks.  Strict mode must be bitwise.
"""
import numpy as np
import pytest

import paper_1104_5243_b200 as bp
from oracle import oracle as O
from tests.helpers import bitwise_equal, small_stack

pytestmark = pytest.mark.gpu


def test_empty_reconstruction_is_zero():
    for hint in (0, 50):
        with bp.GpuContext(32, 96, 80, device=0, strict=True, views=hint) as c:
            vol, st = c.finish()
        assert st.views == 0 and st.launches == 0
        assert not np.any(vol.view(np.uint32))  # +0 everywhere (the reference's first touch)


def test_single_view_and_batch_of_one():
    px, mats = small_stack("spheres3", 5, 120, 96)
    ref1, _ = O.reconstruct(px[:1], mats[:1], 40)
    ref5, _ = O.reconstruct(px, mats, 40)
    for hint in (0, 1):
        with bp.GpuContext(40, 120, 96, device=0, strict=True, views=hint) as c:
            c.backproject(px[0], mats[0])
            vol, st = c.finish()
        assert st.views == 1 and bitwise_equal(vol, ref1)
    with bp.GpuContext(40, 120, 96, device=0, strict=True, view_batch=1, views=5) as c:
        for k in range(5):
            c.backproject(px[k], mats[k])
        vol, st = c.finish()
    assert st.launches >= 5 and bitwise_equal(vol, ref5)


def test_context_reused_across_stacks():
    # finish() resets the reconstruction: a second, different stack on the same context
    # is not contaminated by the first
    a_px, a_m = small_stack("spheres3", 12, 120, 96)
    b_px, b_m = small_stack("point", 9, 120, 96)
    ref_a, _ = O.reconstruct(a_px, a_m, 48)
    ref_b, _ = O.reconstruct(b_px, b_m, 48)
    with bp.GpuContext(48, 120, 96, device=0, strict=True, view_batch=4, views=12) as c:
        for px, m, ref in ((a_px, a_m, ref_a), (b_px, b_m, ref_b), (a_px, a_m, ref_a)):
            for k in range(px.shape[0]):
                c.backproject(px[k], m[k], copy=False)
            vol, _ = c.finish()
            assert bitwise_equal(vol, ref)


def test_default_view_batch():
    # view_batch <= 0 selects the library default (bp_gpu.h): 32 views per launch, 62 for a
    # whole volume of 1024^3 voxels or more; the result does not depend on the batch
    px, mats = small_stack("spheres3", 70, 120, 96)
    ref, _ = O.reconstruct(px, mats, 40)
    with bp.GpuContext(40, 120, 96, device=0, strict=True, view_batch=0, tail_batches=0) as c:
        for k in range(70):
            c.backproject(px[k], mats[k])
        vol, st = c.finish()
    assert st.launches == 3 and bitwise_equal(vol, ref)  # 32 + 32 + 6
    cfg = bp.GpuConfig()
    bp.lib().bp_gpu_config_init(bp.C.byref(cfg))
    assert cfg.view_batch == 0
    with bp.GpuContext(1024, 120, 96, device=0, strict=False, view_batch=0, tail_batches=0) as c:
        for k in range(70):
            c.backproject(px[k], mats[k])
        _, st = c.finish(readback=False)
    assert st.launches == 2  # 62 + 8


def test_merged_view_major_launches(monkeypatch):
    # BP_MERGE=3: the first batch alone, then three batches per launch (what compute-bound slabs
    # get by default); ascending view order is kept, so strict mode stays bitwise
    px, mats = small_stack("spheres3", 45, 120, 96)
    ref, _ = O.reconstruct(px, mats, 48)
    monkeypatch.setenv("BP_MERGE", "3")
    for hint in (0, 45):
        with bp.GpuContext(48, 120, 96, device=0, strict=True, view_batch=4, tail_batches=0, views=hint) as c:
            for k in range(45):
                c.backproject(px[k], mats[k])
            vol, st = c.finish()
        assert bitwise_equal(vol, ref)
        assert st.launches == 5  # 12 batches: 1 + 3 + 3 + 3 + (2 full + the 1-view remainder)
    with bp.GpuContext(48, 120, 96, device=0, strict=True, view_batch=4, views=45) as c:  # with a band tail
        for k in range(45):
            c.backproject(px[k], mats[k], copy=False)
        vol, st = c.finish()
    assert bitwise_equal(vol, ref)
