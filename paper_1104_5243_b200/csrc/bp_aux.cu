// bp_aux.cu -- auxiliary kernels around the backprojection: the exact visible-update
// count and per-line clip ranges (precompute.cpp:19-103), the reciprocal self-test, and
// the on-device volume comparison used by the full-size parity tests.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstring>

#include "bp_device.hpp"
#include "bp_device_math.cuh"

namespace bpg {

// ---------------------------------------------------------------------------
// Exact visible-update count (LineProjector::visible, precompute.cpp:37-46):
// one thread per (view, z, y) line, scanning x from both ends like
// build_clip_table (precompute.cpp:68-80).

__global__ void bp_clip_count_kernel(const __grid_constant__ SlabArgs s,
                                     const __grid_constant__ BatchArgs b) {
    const long long lines = (long long)s.nz * s.L;
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const int k = blockIdx.y;
    unsigned long long vis = 0;
    if (i < lines) {
        const int y = (int)(i % s.L);
        const int z = s.z0 + (int)(i / s.L);
        const float* A = b.A[k];
        float uy, vy, wy_;
        line_consts(A, s.wy[y], s.wz[z], uy, vy, wy_);
        const float hu = (float)s.isx, hv = (float)s.isy;
        auto visible = [&](int x) {
            const float wx = s.wx[x];
            const float w = __fadd_rn(__fmul_rn(A[2], wx), wy_);
            const float r = __frcp_rn(w);
            float u = __fmul_rn(__fadd_rn(__fmul_rn(A[0], wx), uy), r);
            u = (u < -2.0f) ? -2.0f : u;
            u = (hu < u) ? hu : u;
            float v = __fmul_rn(__fadd_rn(__fmul_rn(A[1], wx), vy), r);
            v = (v < -2.0f) ? -2.0f : v;
            v = (hv < v) ? hv : v;
            const int iu = (int)floorf(u), iv = (int)floorf(v);
            return iu >= -1 && iu <= s.isx - 1 && iv >= -1 && iv <= s.isy - 1;
        };
        int f = 0;
        while (f < s.L && !visible(f)) ++f;
        if (f < s.L) {
            int l = s.L - 1;
            while (l > f && !visible(l)) --l;
            vis = (unsigned long long)(l - f + 1);
        }
    }
    // warp reduce then one atomic per warp
    for (int o = 16; o; o >>= 1) vis += __shfl_xor_sync(0xffffffffu, vis, o);
    if ((threadIdx.x & 31) == 0 && vis) atomicAdd(s.counters + 3, vis);
}

// Per-line clip ranges in the reference's BPCT layout (precompute.cpp:51-91,
// precompute.hpp:14-25): ranges[2*((p*L + z)*L + y)] = first, last; empty lines
// are (0xFFFF, 0).  Same exact float replay as bp_clip_count_kernel.
__global__ void bp_clip_ranges_kernel(const __grid_constant__ SlabArgs s,
                                      const __grid_constant__ BatchArgs b, uint16_t* ranges,
                                      int view0) {
    const long long lines = (long long)s.nz * s.L;
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const int k = blockIdx.y;
    if (i >= lines) return;
    const int y = (int)(i % s.L);
    const int z = s.z0 + (int)(i / s.L);
    const float* A = b.A[k];
    float uy, vy, wy_;
    line_consts(A, s.wy[y], s.wz[z], uy, vy, wy_);
    const float hu = (float)s.isx, hv = (float)s.isy;
    auto visible = [&](int x) {
        const float wx = s.wx[x];
        const float w = __fadd_rn(__fmul_rn(A[2], wx), wy_);
        const float r = __frcp_rn(w);
        float u = __fmul_rn(__fadd_rn(__fmul_rn(A[0], wx), uy), r);
        u = (u < -2.0f) ? -2.0f : u;
        u = (hu < u) ? hu : u;
        float v = __fmul_rn(__fadd_rn(__fmul_rn(A[1], wx), vy), r);
        v = (v < -2.0f) ? -2.0f : v;
        v = (hv < v) ? hv : v;
        const int iu = (int)floorf(u), iv = (int)floorf(v);
        return iu >= -1 && iu <= s.isx - 1 && iv >= -1 && iv <= s.isy - 1;
    };
    int f = 0;
    while (f < s.L && !visible(f)) ++f;
    uint16_t first = 0xFFFF, last = 0;
    if (f < s.L) {
        int l = s.L - 1;
        while (l > f && !visible(l)) --l;
        first = (uint16_t)f;
        last = (uint16_t)l;
    }
    const size_t idx = 2 * (((size_t)(view0 + k) * s.L + z) * s.L + y);
    ranges[idx] = first;
    ranges[idx + 1] = last;
}

int launch_clip_ranges(const SlabArgs& s, const BatchArgs& b, uint16_t* ranges, int view0,
                       void* stream) {
    const long long lines = (long long)s.nz * s.L;
    dim3 grid((unsigned)((lines + 255) / 256), (unsigned)b.nviews);
    bp_clip_ranges_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(s, b, ranges, view0);
    return (int)cudaGetLastError();
}

// ---------------------------------------------------------------------------
// Self-test: the paired MUFU+Newton reciprocal against __frcp_rn (== IEEE
// 1.0f/w) over every float bit pattern in [lo_bits, hi_bits).

__global__ void bp_rcp_selftest_kernel(uint32_t lo, uint32_t hi, unsigned long long* bad) {
    unsigned long long nbad = 0;
    for (uint32_t i = lo + 2u * (blockIdx.x * blockDim.x + threadIdx.x); i < hi;
         i += 2u * gridDim.x * blockDim.x) {
        const float a = __uint_as_float(i);
        const float b = __uint_as_float(i + 1 < hi ? i + 1 : i);
        const f2 r = rcp2_rn(f2{a, b});
        nbad += (__float_as_uint(r.x) != __float_as_uint(__frcp_rn(a)));
        nbad += (__float_as_uint(r.y) != __float_as_uint(__frcp_rn(b)));
    }
    for (int o = 16; o; o >>= 1) nbad += __shfl_xor_sync(0xffffffffu, nbad, o);
    if ((threadIdx.x & 31) == 0 && nbad) atomicAdd(bad, nbad);
}

int selftest_rcp(uint32_t lo_bits, uint32_t hi_bits, unsigned long long* mismatches) {
    unsigned long long* d = nullptr;
    cudaError_t e = cudaMalloc(&d, sizeof *d);
    if (e != cudaSuccess) return (int)e;
    cudaMemset(d, 0, sizeof *d);
    bp_rcp_selftest_kernel<<<148 * 8, 256>>>(lo_bits, hi_bits, d);
    e = cudaGetLastError();
    if (e == cudaSuccess) e = cudaMemcpy(mismatches, d, sizeof *d, cudaMemcpyDeviceToHost);
    cudaFree(d);
    return (int)e;
}

// ---------------------------------------------------------------------------
// Diagnostic comparison (full-size property tests without host transfers).

__global__ void bp_compare_kernel(const float* a, const float* b, unsigned long long n,
                                  double* out, unsigned long long* nbit) {
    double mx = 0.0, mr = 0.0, ss = 0.0;
    unsigned long long nb = 0;
    for (unsigned long long i = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; i < n;
         i += (unsigned long long)gridDim.x * blockDim.x) {
        const float x = a[i], y = b[i];
        const double d = (double)x - (double)y;
        mx = fmax(mx, fabs(d));
        mr = fmax(mr, fabs((double)y));
        ss += d * d;
        nb += (__float_as_uint(x) != __float_as_uint(y));
    }
    for (int o = 16; o; o >>= 1) {
        mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        mr = fmax(mr, __shfl_xor_sync(0xffffffffu, mr, o));
        ss += __shfl_xor_sync(0xffffffffu, ss, o);
        nb += __shfl_xor_sync(0xffffffffu, nb, o);
    }
    if ((threadIdx.x & 31) == 0) {
        // max of non-negative doubles via their ordered bit patterns
        atomicMax(reinterpret_cast<unsigned long long*>(out + 0), (unsigned long long)__double_as_longlong(mx));
        atomicMax(reinterpret_cast<unsigned long long*>(out + 1), (unsigned long long)__double_as_longlong(mr));
        atomicAdd(out + 2, ss);
        atomicAdd(nbit, nb);
    }
}

int device_compare(const float* a, const float* b, unsigned long long n, double* res3,
                   unsigned long long* nbit) {
    double* d = nullptr;
    cudaError_t e = cudaMalloc(&d, 4 * sizeof(double));
    if (e != cudaSuccess) return (int)e;
    cudaMemset(d, 0, 4 * sizeof(double));
    bp_compare_kernel<<<148 * 8, 256>>>(a, b, n, d, reinterpret_cast<unsigned long long*>(d + 3));
    e = cudaGetLastError();
    double h[4] = {0, 0, 0, 0};
    if (e == cudaSuccess) e = cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
    cudaFree(d);
    res3[0] = h[0];
    res3[1] = h[1];
    res3[2] = h[2];
    std::memcpy(nbit, &h[3], sizeof *nbit);
    return (int)e;
}

int launch_clip_count(const SlabArgs& s, const BatchArgs& b, void* stream) {
    const long long lines = (long long)s.nz * s.L;
    dim3 grid((unsigned)((lines + 255) / 256), (unsigned)b.nviews);
    bp_clip_count_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(s, b);
    return (int)cudaGetLastError();
}

// ---------------------------------------------------------------------------
// Pair ring for the fast-mode kernel ("pair ring"): pair row e of a
// slot holds, per column c, (p[e-1][c], p[e][c] - p[e-1][c]) with p[-1] = p[isy] = 0,
// the zero border of pad_image (kernel.cpp:32-47).  The fast kernel's vertical lerp
// fma(sy, bl - tl, tl) then needs one 8-byte load per column and no subtraction;
// bl - tl is the same IEEE subtraction the kernel would do, so results are bitwise
// those of the raw-tile fast kernel.  One block per (pair row, view), float4 in,
// 2 x float4 out: HBM-bound (4 + 8 bytes per texel).  128-thread blocks with few
// registers fit beside two resident backprojection CTAs, so the expansion of the
// next batch runs on a low-priority stream under the current batch's kernel.
__global__ void __launch_bounds__(128) bp_expand_kernel(const __grid_constant__ ExpandArgs a) {
    const int e = a.e0 + (int)blockIdx.x;
    const size_t slot = (size_t)a.slot[blockIdx.y];
    const float* img = a.ring + slot * a.isy * a.pitch;
    const float4* up = reinterpret_cast<const float4*>(img + (size_t)(e - 1) * a.pitch);
    const float4* dn = reinterpret_cast<const float4*>(img + (size_t)e * a.pitch);
    float4* out = reinterpret_cast<float4*>(a.ringx + (slot * (a.isy + 1) + e) * a.pitchx);
    const bool has_up = e > 0, has_dn = e < a.isy;
    const int n4 = a.pitch / 4;
    for (int c = threadIdx.x; c < n4; c += blockDim.x) {
        const float4 zero = make_float4(0.f, 0.f, 0.f, 0.f);
        const float4 p = has_up ? __ldg(up + c) : zero;
        const float4 q = has_dn ? __ldg(dn + c) : zero;
        out[2 * c] = make_float4(p.x, __fsub_rn(q.x, p.x), p.y, __fsub_rn(q.y, p.y));
        out[2 * c + 1] = make_float4(p.z, __fsub_rn(q.z, p.z), p.w, __fsub_rn(q.w, p.w));
    }
}

// The same expansion as a small grid (one 128-thread, 32-register block per SM) that
// fits beside two resident backprojection CTAs (2 x 320 threads x 96 registers leave
// exactly 4096 registers and ~2 KB of shared memory per SM): launched just BEFORE a
// batch's backprojection, it builds the next batch's pair rows underneath it.
__global__ void __launch_bounds__(128, 16) bp_expand_small_kernel(const __grid_constant__ ExpandArgs a,
                                                                  int nviews) {
    const int rows = a.isy + 1, n4 = a.pitch / 4;
    const long long units = (long long)nviews * rows;
    for (long long u = blockIdx.x; u < units; u += gridDim.x) {
        const int e = (int)(u % rows);
        const size_t slot = (size_t)a.slot[u / rows];
        const float* img = a.ring + slot * a.isy * a.pitch;
        const float4* up = reinterpret_cast<const float4*>(img + (size_t)(e - 1) * a.pitch);
        const float4* dn = reinterpret_cast<const float4*>(img + (size_t)e * a.pitch);
        float4* out = reinterpret_cast<float4*>(a.ringx + (slot * rows + e) * a.pitchx);
        for (int c = threadIdx.x; c < n4; c += blockDim.x) {
            const float4 zero = make_float4(0.f, 0.f, 0.f, 0.f);
            const float4 p = e > 0 ? __ldg(up + c) : zero;
            const float4 q = e < a.isy ? __ldg(dn + c) : zero;
            out[2 * c] = make_float4(p.x, __fsub_rn(q.x, p.x), p.y, __fsub_rn(q.y, p.y));
            out[2 * c + 1] = make_float4(p.z, __fsub_rn(q.z, p.z), p.w, __fsub_rn(q.w, p.w));
        }
    }
}

int launch_expand_small(const ExpandArgs& a, int n, int blocks, void* stream) {
    if (n < 1) return 0;
    if (a.pitch % 4 || a.pitchx < a.pitch) return (int)cudaErrorInvalidValue;
    static const bool carve = [] {
        return cudaFuncSetAttribute(bp_expand_small_kernel,
                                    cudaFuncAttributePreferredSharedMemoryCarveout, 100) == cudaSuccess;
    }();
    (void)carve;
    bp_expand_small_kernel<<<blocks, 128, 0, (cudaStream_t)stream>>>(a, n);
    return (int)cudaGetLastError();
}

int launch_expand(const ExpandArgs& a, int n, void* stream) {
    if (n < 1) return 0;
    if (a.pitch % 4 || a.pitchx < a.pitch) return (int)cudaErrorInvalidValue;
    if (a.e1 > a.e0 && (a.e0 < 0 || a.e1 > a.isy + 1)) return (int)cudaErrorInvalidValue;
    dim3 grid((unsigned)(a.e1 > a.e0 ? a.e1 - a.e0 : a.isy + 1), (unsigned)n);
    static const bool carve = [] {
        // same shared-memory carveout as the backprojection kernel, so expansion
        // blocks can be co-resident with it on an SM
        return cudaFuncSetAttribute(bp_expand_kernel, cudaFuncAttributePreferredSharedMemoryCarveout,
                                    100) == cudaSuccess;
    }();
    (void)carve;
    bp_expand_kernel<<<grid, 128, 0, (cudaStream_t)stream>>>(a);
    return (int)cudaGetLastError();
}

}  // namespace bpg
