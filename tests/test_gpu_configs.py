"""Full-volume parity at BASELINE configs 1, 2 and 3 (496 views of 1248x960, the
seeded BASELINE stack), against the reference's own reconstruction.

* config 1, 128^3: strict mode bitwise and fast mode within the north_star tolerance
  against the C oracle over the whole volume; the oracle itself is checked bitwise
  against the live reference library (oracle/_ref, the unmodified sources) when it
  was built, i.e. bp::reconstruct (proj/src/scheduler.cpp:24-133) with lanes 8,
  block_b 8 and clip on, the configuration BASELINE.md section 3 times;
* config 2, 256^3 (the 16x16x8 kernel): fast mode within tolerance over the whole
  volume (strict bitwise is test_gpu_fullsize.py::test_config2_256_full_volume_strict_bitwise);
* config 3, 512^3 (the headline): strict mode bitwise and fast mode within
  tolerance over the WHOLE volume against the reference library run on every host
  core (about a minute on 16 cores), or against the C oracle when the reference
  library is absent.
Tolerance (north_star): max|d| <= 1e-4 * max|ref|, RMS(d) <= 1e-6 * max|ref|.
"""
import os

import numpy as np
import pytest

import paper_1104_5243_b200 as bp
from oracle import oracle as O
from tests.helpers import TOL_MAX, TOL_RMS, bitwise_equal, err_stats

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def stack():
    return bp.Stack.baseline()


def _gpu(stack, L, strict, view_batch=32):
    with bp.GpuContext(L, 1248, 960, device=0, strict=strict, view_batch=view_batch) as c:
        c.backproject_stack(stack)
        vol, st = c.finish()
    assert st.fallback_pairs == 0 and st.tile_pairs > 0
    return vol


def _reference(stack, L):
    """bp::reconstruct of the reference (lanes 8, block_b 8, clip on, all host threads)
    when oracle/_ref exists, else the C oracle (pinned bitwise to it in test_oracle.py)."""
    if O.ref_available():
        ref, st = O.ref_reconstruct(stack.pixels, stack.matrices, L, threads=os.cpu_count() or 1,
                                    block_b=8, lanes=8, clip=True)
        return ref, "reference"
    ref, _ = O.reconstruct(stack.pixels, stack.matrices, L)
    return ref, "oracle"


def test_config1_128_full_volume(stack):
    L = 128
    ref, _ = O.reconstruct(stack.pixels, stack.matrices, L)
    if O.ref_available():
        live, _ = O.ref_reconstruct(stack.pixels, stack.matrices, L, threads=os.cpu_count() or 1,
                                    block_b=8, lanes=8, clip=True)
        assert bitwise_equal(live, ref)  # the oracle is the reference, bit for bit
    strict = _gpu(stack, L, True)
    assert bitwise_equal(strict, ref), err_stats(strict, ref)
    fast = _gpu(stack, L, False)
    emax, erms = err_stats(fast, ref)
    print(f"config 1 fast vs reference: max {emax:.2e} rms {erms:.2e}")
    assert emax <= TOL_MAX and erms <= TOL_RMS, (emax, erms)


def test_config2_256_fast_full_volume(stack):
    L = 256
    ref, _ = O.reconstruct(stack.pixels, stack.matrices, L)
    fast = _gpu(stack, L, False)
    emax, erms = err_stats(fast, ref)
    print(f"config 2 fast vs reference: max {emax:.2e} rms {erms:.2e}")
    assert emax <= TOL_MAX and erms <= TOL_RMS, (emax, erms)


def test_config3_512_full_volume(stack):
    L = 512
    ref, kind = _reference(stack, L)
    strict = _gpu(stack, L, True)
    assert bitwise_equal(strict, ref), err_stats(strict, ref)
    del strict
    fast = _gpu(stack, L, False, view_batch=248)
    emax, erms = err_stats(fast, ref)
    print(f"config 3 fast vs {kind}: max {emax:.2e} rms {erms:.2e}")
    assert emax <= TOL_MAX and erms <= TOL_RMS, (emax, erms)
