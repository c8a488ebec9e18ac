"""Python front-end of the CPU oracle -- TEST INFRASTRUCTURE ONLY.

Loads oracle/_build/libbp_oracle.so (the C restatement, oracle/bp_oracle.c) and,
when present, oracle/_ref/libbackproject_ref.so (the unmodified reference
sources compiled by oracle/Makefile).  Only tests/, __graft_entry__.smoke() and
bench.py's CPU legs import this module; the product package never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
_ORACLE_SO = os.path.join(HERE, "_build", "libbp_oracle.so")
_REF_SO = os.path.join(HERE, "_ref", "libbackproject_ref.so")
REF_SRC = "/root/reference/proj"


class Grid(C.Structure):
    """bpo_grid == bp::VoxelGrid (proj/src/geometry.hpp:13-23)."""

    _fields_ = [("L", C.c_int), ("MM", C.c_double), ("ox", C.c_double), ("oy", C.c_double),
                ("oz", C.c_double)]

    @staticmethod
    def cube(L: int, dx: float = 0.0, dy: float = 0.0, dz: float = 0.0) -> "Grid":
        # VoxelGrid::cube, proj/src/geometry.cpp:11-19
        MM = 256.0 / L
        off = -0.5 * (L - 1) * MM
        return Grid(L, MM, off + dx, off + dy, off + dz)


def build(ref: bool = True) -> None:
    """Compile the oracle (and the reference when its sources are present)."""
    targets = ["all"]
    if ref and os.path.isdir(REF_SRC):
        targets.append("ref")
    subprocess.run(["make", "-s", "-C", HERE] + targets, check=True)


_lib = None
_ref = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_ORACLE_SO):
            build(ref=False)
        L = C.CDLL(_ORACLE_SO)
        fp = C.POINTER(C.c_float)
        dp = C.POINTER(C.c_double)
        ip = C.POINTER(C.c_int)
        L.bpo_reconstruct.argtypes = [fp, dp, C.c_int, C.c_int, C.c_int, C.POINTER(Grid), C.c_int,
                                      C.c_int, C.c_int, C.c_int, fp, C.POINTER(C.c_uint64)]
        L.bpo_reconstruct_lines.argtypes = [fp, dp, C.c_int, C.c_int, C.c_int, C.POINTER(Grid),
                                            ip, ip, C.c_int, C.c_int, C.c_int, fp]
        L.bpo_visible_updates.argtypes = [dp, C.c_int, C.c_int, C.c_int, C.POINTER(Grid), C.c_int,
                                          C.c_int, C.c_int, C.POINTER(C.c_uint64)]
        L.bpo_line_update.argtypes = [fp, fp, C.c_int, C.c_int, fp, C.POINTER(Grid), C.c_int,
                                      C.c_int, C.c_int, C.c_int, C.c_int]
        L.bpo_line_update.restype = C.c_uint64
        L.bpo_clip_line.argtypes = [fp, C.POINTER(Grid), C.c_int, C.c_int, C.c_int, C.c_int, ip, ip]
        _lib = L
    return _lib


def ref_available() -> bool:
    return os.path.exists(_REF_SO)


def ref():
    """The reference library built from /root/reference (None if not built)."""
    global _ref
    if _ref is None:
        if not os.path.exists(_REF_SO):
            if os.path.isdir(REF_SRC):
                build(ref=True)
            else:
                return None
        R = C.CDLL(_REF_SO)
        fp = C.POINTER(C.c_float)
        dp = C.POINTER(C.c_double)
        ip = C.POINTER(C.c_int)
        d = C.c_double
        i = C.c_int
        R.ref_reconstruct.argtypes = [fp, dp, i, i, i, i, d, d, d, i, i, i, i, i, i, i, fp, dp]
        R.ref_reconstruct_lines.argtypes = [fp, dp, i, i, i, i, d, d, d, ip, ip, i, i, fp]
        R.ref_clip_table.argtypes = [dp, i, i, i, i, d, d, d, C.POINTER(C.c_uint16),
                                     C.POINTER(C.c_uint64)]
        R.ref_make_stack.argtypes = [C.c_char_p, i, i, i, d, d, d, dp, fp]
        R.ref_forward_project.argtypes = [dp, i, dp, i, i, fp]
        R.ref_read_clip_table.argtypes = [C.c_char_p, C.POINTER(C.c_int), C.POINTER(C.c_int),
                                          C.POINTER(C.c_uint16), C.POINTER(C.c_uint64)]
        R.ref_write_clip_table.argtypes = [C.c_char_p, i, i, C.POINTER(C.c_uint16)]
        R.ref_last_error.restype = C.c_char_p
        _ref = R
    return _ref


def _f(a):
    return a.ctypes.data_as(C.POINTER(C.c_float))


def _d(a):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def _i(a):
    return a.ctypes.data_as(C.POINTER(C.c_int))


def _prep(pixels, mats):
    pixels = np.ascontiguousarray(pixels, dtype=np.float32)
    mats = np.ascontiguousarray(mats, dtype=np.float64).reshape(-1, 12)
    n, isy, isx = pixels.shape
    assert mats.shape[0] == n
    return pixels, mats, n, isx, isy


def reconstruct(pixels, mats, L, *, offset=(0.0, 0.0, 0.0), z0=0, z1=None, distance_weight=True,
                threads=None, init=None):
    """C restatement of bp::reconstruct over the z-slab [z0, z1).  Returns (vol, updates)."""
    pixels, mats, n, isx, isy = _prep(pixels, mats)
    z1 = L if z1 is None else z1
    g = Grid.cube(L, *offset)
    out = np.zeros((z1 - z0, L, L), np.float32) if init is None else np.array(init, np.float32)
    upd = C.c_uint64(0)
    threads = threads or os.cpu_count() or 1
    rc = lib().bpo_reconstruct(_f(pixels), _d(mats), n, isx, isy, C.byref(g), z0, z1,
                               int(distance_weight), threads, _f(out), C.byref(upd))
    if rc != 0:
        raise ValueError(f"oracle reconstruct failed ({rc})")
    return out, upd.value


def reconstruct_lines(pixels, mats, L, ys, zs, *, offset=(0.0, 0.0, 0.0), distance_weight=True,
                      threads=None):
    pixels, mats, n, isx, isy = _prep(pixels, mats)
    ys = np.ascontiguousarray(ys, np.int32)
    zs = np.ascontiguousarray(zs, np.int32)
    out = np.zeros((len(ys), L), np.float32)
    g = Grid.cube(L, *offset)
    threads = threads or os.cpu_count() or 1
    rc = lib().bpo_reconstruct_lines(_f(pixels), _d(mats), n, isx, isy, C.byref(g), _i(ys),
                                     _i(zs), len(ys), int(distance_weight), threads, _f(out))
    if rc != 0:
        raise ValueError("oracle lines failed")
    return out


def visible_updates(mats, isx, isy, L, *, offset=(0.0, 0.0, 0.0), z0=0, z1=None, threads=None):
    """Per-view clip_stats totals (precompute.cpp:93-103) over the slab [z0, z1)."""
    mats = np.ascontiguousarray(mats, np.float64).reshape(-1, 12)
    n = mats.shape[0]
    z1 = L if z1 is None else z1
    per = np.zeros(n, np.uint64)
    g = Grid.cube(L, *offset)
    lib().bpo_visible_updates(_d(mats), n, isx, isy, C.byref(g), z0, z1,
                              threads or os.cpu_count() or 1,
                              per.ctypes.data_as(C.POINTER(C.c_uint64)))
    return per


def line_update(line, img, A, L, y, z, x0, x1, *, offset=(0.0, 0.0, 0.0), distance_weight=True):
    """One voxel-line update (kernel.cpp:49-85) in place on `line` (float32[L])."""
    img = np.ascontiguousarray(img, np.float32)
    A = np.ascontiguousarray(A, np.float32)
    g = Grid.cube(L, *offset)
    isy, isx = img.shape
    return lib().bpo_line_update(_f(line), _f(img), isx, isy, _f(A), C.byref(g), y, z, x0, x1,
                                 int(distance_weight))


# ---- reference (oracle/_ref) entry points --------------------------------

def ref_reconstruct(pixels, mats, L, *, offset=(0.0, 0.0, 0.0), threads=1, chunk=1, block_b=1,
                    lanes=1, clip=False, distance_weight=True, recip=0):
    """bp::reconstruct of the reference; recip = RecipMode (geometry.hpp:39): 0 exact, 1 approx12,
    2 approx12_nr."""
    R = ref()
    pixels, mats, n, isx, isy = _prep(pixels, mats)
    out = np.zeros((L, L, L), np.float32)
    st = np.zeros(6, np.float64)
    rc = R.ref_reconstruct(_f(pixels), _d(mats), n, isx, isy, L, *offset, threads, chunk, block_b,
                           lanes, int(clip), int(distance_weight), int(recip), _f(out), _d(st))
    if rc != 0:
        raise ValueError(R.ref_last_error().decode())
    return out, {"seconds": st[0], "voxel_updates": int(st[1]), "gups": st[2],
                 "writeback_stores": int(st[3]), "bytes_copied": int(st[4]),
                 "clip_reduction": st[5]}


def ref_reconstruct_lines(pixels, mats, L, ys, zs, *, offset=(0.0, 0.0, 0.0), distance_weight=True):
    R = ref()
    pixels, mats, n, isx, isy = _prep(pixels, mats)
    ys = np.ascontiguousarray(ys, np.int32)
    zs = np.ascontiguousarray(zs, np.int32)
    out = np.zeros((len(ys), L), np.float32)
    rc = R.ref_reconstruct_lines(_f(pixels), _d(mats), n, isx, isy, L, *offset, _i(ys), _i(zs),
                                 len(ys), int(distance_weight), _f(out))
    if rc != 0:
        raise ValueError(R.ref_last_error().decode())
    return out


def ref_clip_total(mats, isx, isy, L, *, offset=(0.0, 0.0, 0.0)):
    R = ref()
    mats = np.ascontiguousarray(mats, np.float64).reshape(-1, 12)
    tot = C.c_uint64(0)
    rc = R.ref_clip_table(_d(mats), mats.shape[0], isx, isy, L, *offset, None, C.byref(tot))
    if rc != 0:
        raise ValueError(R.ref_last_error().decode())
    return tot.value


def ref_make_stack(phantom, n, isx, isy, sid=750.0, sdd=1200.0, pitch=0.32):
    R = ref()
    mats = np.zeros((n, 12), np.float64)
    px = np.zeros((n, isy, isx), np.float32)
    rc = R.ref_make_stack(phantom.encode(), n, isx, isy, sid, sdd, pitch, _d(mats), _f(px))
    if rc != 0:
        raise ValueError(R.ref_last_error().decode())
    return px, mats


def ref_forward_project(ellipsoids, mat, isx, isy):
    R = ref()
    e = np.ascontiguousarray(ellipsoids, np.float64).reshape(-1, 7)
    m = np.ascontiguousarray(mat, np.float64)
    out = np.zeros((isy, isx), np.float32)
    rc = R.ref_forward_project(_d(e), e.shape[0], _d(m), isx, isy, _f(out))
    if rc != 0:
        raise ValueError(R.ref_last_error().decode())
    return out


def ref_clip_table(mats, isx, isy, L, *, offset=(0.0, 0.0, 0.0)):
    """The reference's build_clip_table ranges (n, L, L, 2) u16 and clip_stats total."""
    R = ref()
    mats = np.ascontiguousarray(mats, np.float64).reshape(-1, 12)
    n = mats.shape[0]
    ranges = np.zeros((n, L, L, 2), np.uint16)
    tot = C.c_uint64(0)
    rc = R.ref_clip_table(_d(mats), n, isx, isy, L, *offset,
                          ranges.ctypes.data_as(C.POINTER(C.c_uint16)), C.byref(tot))
    if rc != 0:
        raise ValueError(R.ref_last_error().decode())
    return ranges, tot.value


def ref_read_clip_table(path):
    """BPCT file through the reference's read_clip_table: (ranges (n, L, L, 2) u16, total)."""
    R = ref()
    L, n = C.c_int(), C.c_int()
    if R.ref_read_clip_table(path.encode(), C.byref(L), C.byref(n), None, None) != 0:
        raise ValueError(R.ref_last_error().decode())
    ranges = np.zeros((n.value, L.value, L.value, 2), np.uint16)
    tot = C.c_uint64(0)
    if R.ref_read_clip_table(path.encode(), None, None,
                             ranges.ctypes.data_as(C.POINTER(C.c_uint16)), C.byref(tot)) != 0:
        raise ValueError(R.ref_last_error().decode())
    return ranges, tot.value


def ref_write_clip_table(path, ranges):
    """BPCT file through the reference's write_clip_table."""
    R = ref()
    r = np.ascontiguousarray(ranges, np.uint16)
    if R.ref_write_clip_table(path.encode(), r.shape[1], r.shape[0],
                              r.ctypes.data_as(C.POINTER(C.c_uint16))) != 0:
        raise ValueError(R.ref_last_error().decode())

