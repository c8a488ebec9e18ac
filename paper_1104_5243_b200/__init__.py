"""paper_1104_5243_b200 -- B200-native voxel-driven FDK backprojection.

Python host mirror of the reference C ABI (proj/include/backproject.h) over the
CUDA library ``libbackproject.so`` built from ``csrc/`` (sm_100a).  Everything
computes on the GPU; when the library or a CUDA device is missing, calls fail
loudly (RuntimeError / BPError) -- there is no CPU fallback.

Reference correspondences:
    Stack / Volume handles   proj/src/capi.cpp:43-107
    reconstruct()            bp_reconstruct, proj/src/capi.cpp:109-166
    GpuContext               load / backproject / finish / unload (BASELINE north_star; bp_gpu.h)
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("BP_LIB_PATH") or os.path.join(HERE, "libbackproject.so")

BP_OK, BP_EINVAL, BP_EIO, BP_EVERIFY, BP_EINTERNAL = 0, 1, 2, 3, 4
BP_RECIP_EXACT, BP_RECIP_APPROX12, BP_RECIP_APPROX12_NR = 0, 1, 2
BP_RECIP_HW_APPROX = 3  # GPU-only extension (include/bp_gpu.h)
BP_EXTRACT_V1_STORE, BP_EXTRACT_V2_SHIFT = 0, 1


class BPError(RuntimeError):
    """Non-zero return code of the C ABI, with bp_last_error()."""

    def __init__(self, code: int, msg: str):
        super().__init__(f"[{ {1: 'BP_EINVAL', 2: 'BP_EIO', 3: 'BP_EVERIFY', 4: 'BP_EINTERNAL'}.get(code, code)}] {msg}")
        self.code = code


# ---- C structs (include/backproject.h, include/bp_gpu.h) -------------------

class GenParams(C.Structure):
    _fields_ = [("phantom", C.c_char_p), ("n_views", C.c_int), ("isx", C.c_int), ("isy", C.c_int),
                ("sid_mm", C.c_double), ("sdd_mm", C.c_double), ("pitch_mm", C.c_double)]


class ReconParams(C.Structure):
    _fields_ = [("l", C.c_uint32), ("threads", C.c_int), ("chunk", C.c_int), ("block_b", C.c_int),
                ("lanes", C.c_int), ("recip_mode", C.c_int), ("extract", C.c_int),
                ("strict_mode", C.c_int), ("distance_weight", C.c_int), ("clip", C.c_int),
                ("numa_domains", C.c_int), ("clip_cache", C.c_char_p)]


class ReconStats(C.Structure):
    _fields_ = [("seconds", C.c_double), ("voxel_updates", C.c_uint64), ("gups", C.c_double),
                ("gflops", C.c_double), ("writeback_stores", C.c_uint64),
                ("bytes_copied", C.c_uint64), ("clip_reduction", C.c_double),
                ("thread_updates_min", C.c_uint64), ("thread_updates_max", C.c_uint64)]


class GpuConfig(C.Structure):
    _fields_ = [("l", C.c_uint32), ("isx", C.c_uint32), ("isy", C.c_uint32),
                ("offset_mm", C.c_double * 3), ("device", C.c_int), ("z_begin", C.c_int),
                ("z_end", C.c_int), ("view_batch", C.c_int), ("ring_batches", C.c_int),
                ("strict_mode", C.c_int), ("distance_weight", C.c_int), ("row_windows", C.c_int),
                ("kernel", C.c_int), ("count_visible", C.c_int), ("profile_launches", C.c_int),
                ("recip_mode", C.c_int), ("device_volume", C.c_void_p), ("filter", C.c_int),
                ("sid_mm", C.c_double), ("sdd_mm", C.c_double), ("pitch_mm", C.c_double),
                ("output_volume", C.c_void_p), ("tail_batches", C.c_int), ("views", C.c_int)]


class GpuStats(C.Structure):
    _fields_ = [("wall_ms", C.c_double), ("device_ms", C.c_double), ("kernel_ms", C.c_double),
                ("h2d_ms", C.c_double), ("d2h_ms", C.c_double), ("views", C.c_uint64),
                ("launches", C.c_uint64), ("nominal_updates", C.c_uint64),
                ("visible_updates", C.c_uint64), ("tile_pairs", C.c_uint64),
                ("skipped_pairs", C.c_uint64), ("fallback_pairs", C.c_uint64),
                ("h2d_bytes", C.c_uint64), ("d2h_bytes", C.c_uint64), ("tile_w", C.c_int),
                ("tile_h", C.c_int), ("block_x", C.c_int), ("block_y", C.c_int),
                ("block_z", C.c_int), ("device_updates_min", C.c_uint64),
                ("device_updates_max", C.c_uint64), ("prep_launches", C.c_uint64)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


class BaselineParams(C.Structure):
    _fields_ = [("seed", C.c_uint64), ("n_views", C.c_int), ("isx", C.c_int), ("isy", C.c_int),
                ("sid_mm", C.c_double), ("sdd_mm", C.c_double), ("pitch_mm", C.c_double),
                ("arc_deg", C.c_double), ("jitter_mm", C.c_double), ("jitter_deg", C.c_double),
                ("n_ellipsoids", C.c_int), ("filter", C.c_int), ("threads", C.c_int)]


class ReconEx(C.Structure):
    _fields_ = [("offset_mm", C.POINTER(C.c_double)), ("n_devices", C.c_int),
                ("virtual_slabs", C.c_int), ("view_batch", C.c_int), ("strict_mode", C.c_int),
                ("distance_weight", C.c_int), ("kernel", C.c_int), ("row_windows", C.c_int),
                ("count_visible", C.c_int), ("recip_mode", C.c_int), ("filter", C.c_int),
                ("sid_mm", C.c_double), ("sdd_mm", C.c_double), ("pitch_mm", C.c_double)]


# Every symbol declared in include/*.h (checked by tests/test_host_abi.py).
EXPORTED = [
    "bp_last_error", "bp_stack_generate", "bp_stack_read", "bp_stack_write", "bp_stack_dims",
    "bp_stack_free", "bp_volume_read", "bp_volume_write", "bp_volume_edge", "bp_volume_data",
    "bp_volume_free", "bp_psnr", "bp_reconstruct", "bp_machine_load", "bp_machine_free",
    "bp_model_report_build", "bp_machine_measure", "bp_model_deviation",
    "bp_gpu_config_init", "bp_gpu_load", "bp_gpu_backproject", "bp_gpu_backproject_async",
    "bp_gpu_finish", "bp_gpu_unload", "bp_gpu_volume_device", "bp_gpu_upload_views",
    "bp_gpu_time_resident", "bp_stack_create", "bp_stack_pixels", "bp_stack_matrices",
    "bp_baseline_params_init", "bp_stack_generate_baseline", "bp_baseline_phantom",
    "bp_volume_create", "bp_volume_data_mut", "bp_gpu_set_devices", "bp_gpu_device_count",
    "bp_partition_slabs", "bp_slab_work", "bp_partition_by_cost", "bp_slab_row_window",
    "bp_recon_ex_init", "bp_reconstruct_ex",
    "bp_selftest_rcp", "bp_build_info", "bp_gpu_read_lines", "bp_device_compare",
    "bp_gpu_clip_table", "bp_gpu_filter_views", "bp_ipc_handle", "bp_ipc_open", "bp_ipc_close",
    "bp_gpu_release_cache", "bp_clip_table_read", "bp_clip_table_write",
]


def build(verbose: bool = False) -> None:
    """Compile libbackproject.so in-tree (nvcc -gencode arch=compute_100a,code=sm_100a)."""
    r = subprocess.run(["make", "-C", HERE, "-j8"], capture_output=not verbose, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"libbackproject build failed:\n{r.stdout}\n{r.stderr}")


_lib = None


def lib():
    """Load libbackproject.so.  Raises if it has not been built (no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(f"{LIB_PATH} missing: run paper_1104_5243_b200.build() "
                           "(the GPU path has no CPU fallback)")
    L = C.CDLL(LIB_PATH)
    vp, ip, dp, fp = C.c_void_p, C.c_int, C.POINTER(C.c_double), C.POINTER(C.c_float)
    pp = C.POINTER(C.c_void_p)
    u32 = C.c_uint32
    sig = {
        "bp_last_error": (C.c_char_p, []),
        "bp_build_info": (C.c_char_p, []),
        "bp_stack_generate": (ip, [C.POINTER(GenParams), pp]),
        "bp_stack_read": (ip, [C.c_char_p, pp]),
        "bp_stack_write": (ip, [vp, C.c_char_p]),
        "bp_stack_dims": (None, [vp, C.POINTER(u32), C.POINTER(u32), C.POINTER(u32)]),
        "bp_stack_free": (None, [vp]),
        "bp_stack_create": (ip, [u32, u32, u32, dp, fp, pp]),
        "bp_stack_pixels": (C.c_void_p, [vp]),
        "bp_stack_matrices": (C.c_void_p, [vp]),
        "bp_volume_read": (ip, [C.c_char_p, pp]),
        "bp_volume_write": (ip, [vp, C.c_char_p]),
        "bp_volume_edge": (u32, [vp]),
        "bp_volume_data": (C.c_void_p, [vp]),
        "bp_volume_data_mut": (C.c_void_p, [vp]),
        "bp_volume_free": (None, [vp]),
        "bp_volume_create": (ip, [u32, pp]),
        "bp_psnr": (ip, [vp, vp, C.c_double, dp]),
        "bp_reconstruct": (ip, [vp, C.POINTER(ReconParams), pp, C.POINTER(ReconStats)]),
        "bp_gpu_config_init": (None, [C.POINTER(GpuConfig)]),
        "bp_gpu_load": (ip, [C.POINTER(GpuConfig), pp]),
        "bp_gpu_backproject": (ip, [vp, fp, dp]),
        "bp_gpu_backproject_async": (ip, [vp, fp, dp]),
        "bp_gpu_finish": (ip, [vp, fp, C.POINTER(GpuStats)]),
        "bp_gpu_unload": (ip, [vp]),
        "bp_gpu_volume_device": (ip, [vp, pp, C.POINTER(ip), C.POINTER(ip)]),
        "bp_gpu_upload_views": (ip, [vp, fp, dp, ip]),
        "bp_gpu_time_resident": (ip, [vp, ip, dp, C.POINTER(GpuStats)]),
        "bp_baseline_params_init": (None, [C.POINTER(BaselineParams)]),
        "bp_stack_generate_baseline": (ip, [C.POINTER(BaselineParams), pp]),
        "bp_baseline_phantom": (ip, [C.POINTER(BaselineParams), dp, ip, C.POINTER(ip)]),
        "bp_gpu_set_devices": (ip, [C.POINTER(ip), ip]),
        "bp_gpu_device_count": (ip, [C.POINTER(ip)]),
        "bp_partition_slabs": (ip, [dp, ip, u32, u32, u32, dp, ip, C.POINTER(ip)]),
        "bp_slab_work": (ip, [dp, ip, u32, u32, u32, dp, dp]),
        "bp_partition_by_cost": (ip, [dp, u32, ip, ip, C.POINTER(ip)]),
        "bp_slab_row_window": (ip, [dp, u32, u32, dp, ip, ip, C.POINTER(ip), C.POINTER(ip)]),
        "bp_recon_ex_init": (None, [C.POINTER(ReconEx)]),
        "bp_reconstruct_ex": (ip, [vp, u32, C.POINTER(ReconEx), fp, C.POINTER(GpuStats)]),
        "bp_selftest_rcp": (ip, [u32, u32, C.POINTER(C.c_uint64)]),
        "bp_gpu_read_lines": (ip, [vp, C.POINTER(ip), C.POINTER(ip), ip, fp]),
        "bp_device_compare": (ip, [vp, vp, C.c_uint64, dp, dp, dp, C.POINTER(C.c_uint64)]),
        "bp_gpu_clip_table": (ip, [vp, u32, dp, C.POINTER(C.c_uint16), C.POINTER(C.c_uint64)]),
        "bp_gpu_filter_views": (ip, [fp, fp, ip, u32, u32, C.c_double, C.c_double, C.c_double, ip]),
        "bp_ipc_handle": (ip, [vp, C.POINTER(C.c_ubyte), C.POINTER(C.c_uint64)]),
        "bp_ipc_open": (ip, [C.POINTER(C.c_ubyte), pp]),
        "bp_ipc_close": (ip, [vp]),
        "bp_gpu_release_cache": (ip, []),
        "bp_clip_table_read": (ip, [C.c_char_p, C.POINTER(u32), C.POINTER(u32),
                                    C.POINTER(C.c_uint16), C.POINTER(C.c_uint64)]),
        "bp_clip_table_write": (ip, [C.c_char_p, u32, u32, C.POINTER(C.c_uint16)]),
    }
    for name, (res, args) in sig.items():
        # an older build (BP_LIB_PATH, compile-time A/B) may lack a newer extension symbol;
        # the default in-tree library must export them all (tests/test_host_abi.py)
        if not hasattr(L, name) and os.environ.get("BP_LIB_PATH"):
            continue
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args
    _lib = L
    return L


def _check(rc: int) -> None:
    if rc != BP_OK:
        raise BPError(rc, lib().bp_last_error().decode())


def last_error() -> str:
    return lib().bp_last_error().decode()


def build_info() -> str:
    return lib().bp_build_info().decode()


def device_count() -> int:
    n = C.c_int(0)
    _check(lib().bp_gpu_device_count(C.byref(n)))
    return n.value


def _f(a):
    return a.ctypes.data_as(C.POINTER(C.c_float))


def _d(a):
    return a.ctypes.data_as(C.POINTER(C.c_double))


# ---- stacks and volumes ------------------------------------------------------

class Stack:
    """Projection stack in library-owned pinned host memory (bp_stack)."""

    def __init__(self, handle):
        self._h = handle

    @classmethod
    def from_arrays(cls, pixels, matrices) -> "Stack":
        pixels = np.ascontiguousarray(pixels, np.float32)
        mats = np.ascontiguousarray(matrices, np.float64).reshape(-1, 12)
        n, isy, isx = pixels.shape
        assert mats.shape[0] == n, "one matrix per view"
        h = C.c_void_p()
        _check(lib().bp_stack_create(isx, isy, n, _d(mats), _f(pixels), C.byref(h)))
        return cls(h)

    @classmethod
    def generate(cls, phantom="spheres3", n_views=8, isx=64, isy=48, sid=0.0, sdd=0.0,
                 pitch=0.0) -> "Stack":
        """bp_stack_generate (reference datagen: circular trajectory + named phantom)."""
        p = GenParams(phantom.encode() if phantom is not None else None, n_views, isx, isy, sid,
                      sdd, pitch)
        h = C.c_void_p()
        _check(lib().bp_stack_generate(C.byref(p), C.byref(h)))
        return cls(h)

    @classmethod
    def baseline(cls, **kw) -> "Stack":
        """Seeded BASELINE.json stack (short scan + jitter, 10 ellipsoids, filtered)."""
        p = baseline_params(**kw)
        h = C.c_void_p()
        _check(lib().bp_stack_generate_baseline(C.byref(p), C.byref(h)))
        return cls(h)

    @classmethod
    def read(cls, path: str) -> "Stack":
        h = C.c_void_p()
        _check(lib().bp_stack_read(path.encode(), C.byref(h)))
        return cls(h)

    def write(self, path: str) -> None:
        _check(lib().bp_stack_write(self._h, path.encode()))

    @property
    def dims(self):
        a, b, c = C.c_uint32(), C.c_uint32(), C.c_uint32()
        lib().bp_stack_dims(self._h, C.byref(a), C.byref(b), C.byref(c))
        return a.value, b.value, c.value  # isx, isy, count

    @property
    def pixels(self) -> np.ndarray:
        """Zero-copy view (count, isy, isx) of the pinned pixel buffer."""
        isx, isy, n = self.dims
        p = lib().bp_stack_pixels(self._h)
        return np.ctypeslib.as_array(C.cast(p, C.POINTER(C.c_float)), shape=(n, isy, isx))

    @property
    def matrices(self) -> np.ndarray:
        isx, isy, n = self.dims
        p = lib().bp_stack_matrices(self._h)
        return np.ctypeslib.as_array(C.cast(p, C.POINTER(C.c_double)), shape=(n, 12))

    def close(self):
        if self._h:
            lib().bp_stack_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Volume:
    def __init__(self, handle):
        self._h = handle

    @classmethod
    def read(cls, path: str) -> "Volume":
        h = C.c_void_p()
        _check(lib().bp_volume_read(path.encode(), C.byref(h)))
        return cls(h)

    @classmethod
    def create(cls, l: int) -> "Volume":
        h = C.c_void_p()
        _check(lib().bp_volume_create(l, C.byref(h)))
        return cls(h)

    def write(self, path: str) -> None:
        _check(lib().bp_volume_write(self._h, path.encode()))

    @property
    def edge(self) -> int:
        return lib().bp_volume_edge(self._h)

    @property
    def data(self) -> np.ndarray:
        """Zero-copy (L, L, L) view, index [z, y, x] (x fastest, kernel.hpp:26-33)."""
        L = self.edge
        p = lib().bp_volume_data_mut(self._h)
        return np.ctypeslib.as_array(C.cast(p, C.POINTER(C.c_float)), shape=(L, L, L))

    def psnr(self, ref: "Volume", peak: float = 0.0) -> float:
        out = C.c_double()
        _check(lib().bp_psnr(self._h, ref._h, peak, C.byref(out)))
        return out.value

    def close(self):
        if self._h:
            lib().bp_volume_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def recon_params(l, threads=1, chunk=1, block_b=32, lanes=1, recip_mode=0, extract=0,
                 strict_mode=1, distance_weight=1, clip=0, numa_domains=1, clip_cache=None):
    return ReconParams(l, threads, chunk, block_b, lanes, recip_mode, extract, strict_mode,
                       distance_weight, clip, numa_domains,
                       clip_cache.encode() if clip_cache else None)


def reconstruct(stack: Stack, params: ReconParams):
    """bp_reconstruct: returns (Volume, ReconStats)."""
    h = C.c_void_p()
    st = ReconStats()
    _check(lib().bp_reconstruct(stack._h, C.byref(params), C.byref(h), C.byref(st)))
    return Volume(h), st


def reconstruct_ex(stack: Stack, l: int, *, offset=(0.0, 0.0, 0.0), n_devices=0,
                   virtual_slabs=0, view_batch=32, strict=True, distance_weight=True, kernel=0,
                   row_windows=True, count_visible=False, recip_mode=0, filter=None, out=None):
    """bp_reconstruct_ex: multi-slab reconstruction into a numpy (L, L, L) array.

    filter=(sid_mm, sdd_mm, pitch_mm) runs the GPU cosine + ramp filter on every
    (raw) view before backprojection."""
    p = ReconEx()
    lib().bp_recon_ex_init(C.byref(p))
    off = (C.c_double * 3)(*offset)
    p.offset_mm = C.cast(off, C.POINTER(C.c_double))
    p.n_devices = n_devices
    p.virtual_slabs = virtual_slabs
    p.view_batch = view_batch
    p.strict_mode = int(strict)
    p.distance_weight = int(distance_weight)
    p.kernel = kernel
    p.row_windows = int(row_windows)
    p.count_visible = int(count_visible)
    p.recip_mode = recip_mode
    if filter is not None:
        p.filter = 1
        p.sid_mm, p.sdd_mm, p.pitch_mm = (float(v) for v in filter)
    if out is None:
        out = np.empty((l, l, l), np.float32)
    st = GpuStats()
    _check(lib().bp_reconstruct_ex(stack._h, l, C.byref(p), _f(out), C.byref(st)))
    return out, st


def baseline_params(**kw) -> BaselineParams:
    p = BaselineParams()
    lib().bp_baseline_params_init(C.byref(p))
    names = {f for f, _ in BaselineParams._fields_}
    for k, v in kw.items():
        if k not in names:
            raise TypeError(f"unknown baseline parameter {k!r} (fields: {sorted(names)})")
        setattr(p, k, v)
    return p


def baseline_phantom(**kw) -> np.ndarray:
    p = baseline_params(**kw)
    buf = np.zeros((64, 7), np.float64)
    n = C.c_int(0)
    _check(lib().bp_baseline_phantom(C.byref(p), _d(buf), 64, C.byref(n)))
    return buf[: n.value].copy()


def partition_slabs(matrices, isx, isy, l, G, offset=(0.0, 0.0, 0.0)) -> np.ndarray:
    mats = np.ascontiguousarray(matrices, np.float64).reshape(-1, 12)
    b = (C.c_int * (G + 1))()
    off = np.asarray(offset, np.float64)
    _check(lib().bp_partition_slabs(_d(mats), mats.shape[0], isx, isy, l, _d(off), G, b))
    return np.array(list(b), np.int64)


def slab_work(matrices, isx, isy, l, offset=(0.0, 0.0, 0.0)) -> np.ndarray:
    """The partitioner's per-slice cost model (include/bp_gpu.h bp_slab_work)."""
    mats = np.ascontiguousarray(matrices, np.float64).reshape(-1, 12)
    w = np.zeros(l, np.float64)
    off = np.asarray(offset, np.float64)
    _check(lib().bp_slab_work(_d(mats), mats.shape[0], isx, isy, l, _d(off), _d(w)))
    return w


def partition_by_cost(slice_cost, G, align=1) -> np.ndarray:
    """Slab bounds balancing a per-slice cost (include/bp_gpu.h bp_partition_by_cost)."""
    c = np.ascontiguousarray(slice_cost, np.float64)
    b = (C.c_int * (G + 1))()
    _check(lib().bp_partition_by_cost(_d(c), c.size, G, align, b))
    return np.array(list(b), np.int64)


def slab_row_window(matrix, isy, l, z_begin, z_end, offset=(0.0, 0.0, 0.0)):
    m = np.ascontiguousarray(matrix, np.float64).reshape(12)
    off = np.asarray(offset, np.float64)
    r0, r1 = C.c_int(), C.c_int()
    _check(lib().bp_slab_row_window(_d(m), isy, l, _d(off), z_begin, z_end, C.byref(r0),
                                    C.byref(r1)))
    return r0.value, r1.value


def clip_table(stack: Stack, l: int, offset=(0.0, 0.0, 0.0)):
    """Exact per-line clip ranges (reference BPCT layout) built on the GPU: (ranges, total)."""
    isx, isy, n = stack.dims
    ranges = np.zeros((n, l, l, 2), np.uint16)
    off = np.asarray(offset, np.float64)
    tot = C.c_uint64(0)
    _check(lib().bp_gpu_clip_table(stack._h, l, _d(off),
                                   ranges.ctypes.data_as(C.POINTER(C.c_uint16)), C.byref(tot)))
    return ranges, tot.value


def filter_views(pixels, sid: float, sdd: float, pitch: float, *, device: int = -1, out=None):
    """bp_gpu_filter_views: FDK cosine weight + Ram-Lak row filter of (n, isy, isx) images on the GPU."""
    px = np.ascontiguousarray(pixels, np.float32)
    if px.ndim == 2:
        px = px[None]
    n, isy, isx = px.shape
    if out is None:
        out = np.empty_like(px)
    _check(lib().bp_gpu_filter_views(_f(px), _f(out), n, isx, isy, C.c_double(sid), C.c_double(sdd),
                                     C.c_double(pitch), device))
    return out


def ipc_handle(device_ptr: int) -> bytes:
    """bp_ipc_handle: a 72-byte token for a device pointer of this process. The token is the 64-byte CUDA
    IPC handle of its allocation plus the pointer's offset inside that allocation."""
    buf = (C.c_ubyte * 64)()
    off = C.c_uint64(0)
    _check(lib().bp_ipc_handle(C.c_void_p(int(device_ptr)), buf, C.byref(off)))
    return bytes(buf) + int(off.value).to_bytes(8, "little")


def ipc_open(token: bytes) -> int:
    """bp_ipc_open: map the allocation behind an ipc_handle() token from another process and return the
    exporter's pointer in this process. Pass the same value to ipc_close()."""
    buf = (C.c_ubyte * 64).from_buffer_copy(token[:64])
    off = int.from_bytes(token[64:72], "little") if len(token) >= 72 else 0
    p = C.c_void_p()
    _check(lib().bp_ipc_open(buf, C.byref(p)))
    _ipc_bases[int(p.value) + off] = int(p.value)
    return int(p.value) + off


_ipc_bases = {}


def ipc_close(device_ptr: int) -> None:
    base = _ipc_bases.pop(int(device_ptr), int(device_ptr))
    _check(lib().bp_ipc_close(C.c_void_p(base)))


def clip_table_read(path: str):
    """BPCT file -> (ranges (count, l, l, 2) u16, clip_stats total)."""
    l, n = C.c_uint32(), C.c_uint32()
    _check(lib().bp_clip_table_read(path.encode(), C.byref(l), C.byref(n), None, None))
    ranges = np.zeros((n.value, l.value, l.value, 2), np.uint16)
    tot = C.c_uint64()
    _check(lib().bp_clip_table_read(path.encode(), None, None,
                                    ranges.ctypes.data_as(C.POINTER(C.c_uint16)), C.byref(tot)))
    return ranges, tot.value


def clip_table_write(path: str, ranges) -> None:
    r = np.ascontiguousarray(ranges, np.uint16)
    n, l = r.shape[0], r.shape[1]
    assert r.shape == (n, l, l, 2)
    _check(lib().bp_clip_table_write(path.encode(), l, n, r.ctypes.data_as(C.POINTER(C.c_uint16))))


def release_cache() -> None:
    """Frees the idle loaded contexts bp_reconstruct keeps between calls."""
    _check(lib().bp_gpu_release_cache())


def set_devices(devs) -> None:
    arr = (C.c_int * len(devs))(*devs)
    _check(lib().bp_gpu_set_devices(arr, len(devs)))


def selftest_rcp(lo_bits: int, hi_bits: int) -> int:
    m = C.c_uint64(0)
    _check(lib().bp_selftest_rcp(lo_bits, hi_bits, C.byref(m)))
    return m.value


# ---- streaming module API ------------------------------------------------------

class GpuContext:
    """load / backproject / finish / unload (include/bp_gpu.h)."""

    def __init__(self, l, isx, isy, *, offset=(0.0, 0.0, 0.0), device=-1, z_begin=0, z_end=0,
                 view_batch=32, ring_batches=0, strict=True, distance_weight=True,
                 row_windows=True, kernel=0, count_visible=False, profile_launches=False,
                 recip_mode=0, device_volume=None, filter=None, output_volume=None,
                 tail_batches=-1, views=0):
        cfg = GpuConfig()
        lib().bp_gpu_config_init(C.byref(cfg))
        cfg.l, cfg.isx, cfg.isy = l, isx, isy
        for i in range(3):
            cfg.offset_mm[i] = offset[i]
        cfg.device = device
        cfg.z_begin, cfg.z_end = z_begin, z_end
        cfg.view_batch, cfg.ring_batches = view_batch, ring_batches
        cfg.strict_mode = int(strict)
        cfg.distance_weight = int(distance_weight)
        cfg.row_windows = int(row_windows)
        cfg.kernel = kernel
        cfg.count_visible = int(count_visible)
        if output_volume is not None:  # device pointer (int): final pass stores here
            cfg.output_volume = C.c_void_p(int(output_volume))
        if filter is not None:  # (sid_mm, sdd_mm, pitch_mm): filter raw views on upload
            cfg.filter = 1
            cfg.sid_mm, cfg.sdd_mm, cfg.pitch_mm = (float(v) for v in filter)
        cfg.profile_launches = int(profile_launches)
        cfg.recip_mode = recip_mode
        cfg.device_volume = device_volume
        cfg.tail_batches = tail_batches
        cfg.views = views  # views per reconstruction, if known: band-ordered tail (bp_gpu.h)
        self.l, self.isx, self.isy = l, isx, isy
        self.z_begin, self.z_end = z_begin, (z_end if z_end > 0 else l)
        h = C.c_void_p()
        _check(lib().bp_gpu_load(C.byref(cfg), C.byref(h)))
        self._h = h

    def backproject(self, image, matrix, copy=True) -> None:
        m = np.ascontiguousarray(matrix, np.float64).reshape(12)
        if copy:
            img = np.ascontiguousarray(image, np.float32)
            _check(lib().bp_gpu_backproject(self._h, _f(img), _d(m)))
        else:
            # zero-copy: the library reads `image` until finish(), so it must be the
            # caller's own float32 C-contiguous buffer (a converted temporary would be
            # freed on return while the upload is still pending)
            if not (isinstance(image, np.ndarray) and image.dtype == np.float32
                    and image.flags.c_contiguous):
                raise ValueError("backproject(copy=False) needs a float32 C-contiguous array "
                                 "that stays alive until finish()")
            if image.size != self.isx * self.isy:
                raise ValueError(f"image has {image.size} pixels, expected {self.isx * self.isy}")
            _check(lib().bp_gpu_backproject_async(self._h, _f(image), _d(m)))

    def backproject_stack(self, stack: Stack) -> None:
        px, mats = stack.pixels, stack.matrices
        for k in range(px.shape[0]):
            _check(lib().bp_gpu_backproject_async(self._h, _f(px[k]), _d(mats[k])))

    def finish(self, out=None, readback=True):
        st = GpuStats()
        if readback:
            nz = self.z_end - self.z_begin
            if out is None:
                out = np.empty((nz, self.l, self.l), np.float32)
            elif not (isinstance(out, np.ndarray) and out.dtype == np.float32
                      and out.flags.c_contiguous and out.flags.writeable
                      and out.size >= nz * self.l * self.l):
                raise ValueError(f"finish(out=...) needs a writeable float32 C-contiguous array "
                                 f"of at least {nz * self.l * self.l} elements")
            _check(lib().bp_gpu_finish(self._h, _f(out), C.byref(st)))
        else:
            _check(lib().bp_gpu_finish(self._h, None, C.byref(st)))
        return out, st

    def upload_views(self, pixels, matrices) -> None:
        px = np.ascontiguousarray(pixels, np.float32)
        m = np.ascontiguousarray(matrices, np.float64).reshape(-1, 12)
        _check(lib().bp_gpu_upload_views(self._h, _f(px), _d(m), m.shape[0]))

    def upload_stack(self, stack: Stack) -> None:
        px, m = stack.pixels, stack.matrices
        _check(lib().bp_gpu_upload_views(self._h, _f(px), _d(m), m.shape[0]))

    def time_resident(self, iters=1):
        ms = C.c_double()
        st = GpuStats()
        _check(lib().bp_gpu_time_resident(self._h, iters, C.byref(ms), C.byref(st)))
        return ms.value, st

    def volume_device_ptr(self) -> int:
        p = C.c_void_p()
        a, b = C.c_int(), C.c_int()
        _check(lib().bp_gpu_volume_device(self._h, C.byref(p), C.byref(a), C.byref(b)))
        return p.value

    def read_lines(self, ys, zs) -> np.ndarray:
        ys = np.ascontiguousarray(ys, np.int32)
        zs = np.ascontiguousarray(zs, np.int32)
        out = np.empty((len(ys), self.l), np.float32)
        _check(lib().bp_gpu_read_lines(self._h, ys.ctypes.data_as(C.POINTER(C.c_int)),
                                       zs.ctypes.data_as(C.POINTER(C.c_int)), len(ys), _f(out)))
        return out

    def compare_with(self, other: "GpuContext"):
        """(max|a-b|, max|b|, rms(a-b), n_bitwise_diff) of the two device slabs."""
        n = (self.z_end - self.z_begin) * self.l * self.l
        mx, mr, ss, nb = C.c_double(), C.c_double(), C.c_double(), C.c_uint64()
        _check(lib().bp_device_compare(C.c_void_p(self.volume_device_ptr()),
                                       C.c_void_p(other.volume_device_ptr()), n, C.byref(mx),
                                       C.byref(mr), C.byref(ss), C.byref(nb)))
        return mx.value, mr.value, (ss.value / n) ** 0.5, nb.value

    def close(self):
        if getattr(self, "_h", None):
            lib().bp_gpu_unload(self._h)
            self._h = None

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
