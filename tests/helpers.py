"""Shared fixtures for the parity tests (mirrors proj/tests/test_support.hpp).

random_image / random_matrix / small_stack restate test_support.hpp:22-45,
104-109 with numpy's seeded generator (the mt19937 streams of the reference are
not reproduced; the properties are).
"""
from __future__ import annotations

import numpy as np

import paper_1104_5243_b200 as bp
from oracle import oracle as O


def random_image(isx, isy, seed, lo=0.0, hi=1.0):
    rng = np.random.default_rng(seed)
    return rng.uniform(lo, hi, size=(isy, isx)).astype(np.float32)


def circular(n, sid, sdd, nu, nv, pitch):
    """make_circular_trajectory (geometry.cpp:86-128) via the library's restatement."""
    s = bp.Stack.generate("point", n, nu, nv, sid, sdd, pitch)
    return s.matrices.copy()


def random_matrix(seed, isx, isy):
    """test_support.hpp:32-45: a random valid single-view geometry."""
    rng = np.random.default_rng(seed)
    n = int(rng.integers(3, 65))
    s = rng.uniform(600.0, 900.0)
    d = s * rng.uniform(1.3, 1.8)
    pitch = 420.0 * (d / s) / isx
    mats = circular(n, s, d, isx, isy, pitch)
    return mats[int(rng.integers(0, n))]


def small_stack(phantom, views, isx, isy):
    """test_support.hpp:104-109: same field of view as the full detector."""
    s = bp.Stack.generate(phantom, views, isx, isy, 750.0, 1200.0, 0.32 * 1248.0 / isx)
    return s.pixels.copy(), s.matrices.copy()


def baseline_small(n_views=24, shrink=8, seed=20110428, filter=1):
    """BASELINE-shaped stack scaled down: same FOV, detector / shrink."""
    s = bp.Stack.baseline(n_views=n_views, isx=1248 // shrink, isy=960 // shrink,
                          pitch_mm=0.32 * shrink, seed=seed, filter=filter)
    return s.pixels.copy(), s.matrices.copy()


def err_stats(got, ref):
    """(max|d|/max|ref|, rms(d)/max|ref|) -- the north_star tolerance metrics."""
    got = np.asarray(got, np.float64)
    ref = np.asarray(ref, np.float64)
    peak = np.abs(ref).max()
    d = got - ref
    return float(np.abs(d).max() / peak), float(np.sqrt(np.mean(d * d)) / peak)


def bitwise_equal(a, b):
    a = np.ascontiguousarray(a, np.float32)
    b = np.ascontiguousarray(b, np.float32)
    return a.shape == b.shape and np.array_equal(a.view(np.uint32), b.view(np.uint32))


TOL_MAX = 1e-4   # north_star: max|d| <= 1e-4 * max|ref|
TOL_RMS = 1e-6   # north_star: RMS     <= 1e-6 * max|ref|
