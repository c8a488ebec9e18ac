// bp_filter.cu -- FDK projection preprocessing on the GPU:
// cosine weight + row-wise Ram-Lak ramp filter, applied in place to detector rows
// that are already in HBM (a projection-ring slot or a caller buffer), so raw
// projections never need a host FFT pass.
//
// The math is the host restatement bph::cosine_ramp_filter (bp_host.cpp), which
// follows PAPER.md:104-108:
//   p'(u,v) = tau * IDFT_M( H * DFT_M( sdd / sqrt(sdd^2+du^2+dv^2) * p(.,v) ) )
// with H the real spectrum of the zero-padded Ram-Lak kernel (bph::ramp_spectrum).
//
// One CTA filters one PAIR of detector rows: they are packed as the real and
// imaginary parts of one complex row (H is real, so the two rows stay separate).
// M is the smallest R0 * 2^q >= 2 isx - 1 with R0 in {1, 3, 5} (2560 at isx = 1248); a
// non-power-of-two M adds a leading radix-R0 pass (r0_forward / r0_inverse below).
// The 2^q-point part runs in shared memory as a radix-2 network grouped into
// register passes of up to 4 stages (16 elements per thread):
//   * forward: decimation-in-frequency, natural order in -> bit-reversed out;
//   * multiply by H, pre-permuted to bit-reversed order on the host;
//   * inverse: decimation-in-time, bit-reversed in -> natural order out.
// No permutation pass is needed.  The first forward pass reads the rows straight
// from global memory (applying the cosine weight, zero padding p >= isx) and the
// last inverse pass writes them straight back; the last forward pass, the H
// multiply and the first inverse pass are fused.  Shared-memory positions are
// XOR-swizzled, phys(p) = p ^ ((p >> 4) & 15), which makes every pass
// conflict-free (both the stride-g tuples and the contiguous g = 1 tuples).
//
// Roofline: HBM traffic is one read and one write of each row (8 B per pixel);
// the FFT work (~10 * M * log2 M flops per row pair) and the shared-memory
// passes dominate, and together are a small fraction of the backprojection.
#include <cuda_runtime.h>

#include <cstdint>

#include "bp_device.hpp"

namespace bpg {
namespace {

__device__ __forceinline__ int swz(int p) { return p ^ ((p >> 4) & 15); }

__device__ __forceinline__ float2 cmul(float2 a, float2 w) {
    return make_float2(a.x * w.x - a.y * w.y, a.x * w.y + a.y * w.x);
}
__device__ __forceinline__ float2 cmulc(float2 a, float2 w) {  // a * conj(w)
    return make_float2(a.x * w.x + a.y * w.y, a.y * w.x - a.x * w.y);
}
__device__ __forceinline__ float2 cadd(float2 a, float2 b) { return make_float2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ float2 csub(float2 a, float2 b) { return make_float2(a.x - b.x, a.y - b.y); }

// 16th roots of unity: W16^n = cos16(n) - i sin16(n), n < 8 (compile-time folded)
__host__ __device__ constexpr float cos16(int n) {
    return n == 0 ? 1.0f : n == 1 ? 0.923879532511286756f : n == 2 ? 0.707106781186547524f
         : n == 3 ? 0.382683432365089772f : n == 4 ? 0.0f : n == 5 ? -0.382683432365089772f
         : n == 6 ? -0.707106781186547524f : -0.923879532511286756f;
}
__host__ __device__ constexpr float sin16(int n) { return n <= 4 ? cos16(4 - n) : cos16(n - 4); }

// The twiddle of stage half hs = g*t for tuple element pair offset k = m mod t is
//   W_{2hs}^{j + k g} = alpha_t(j) * W16^(8k/t),  alpha_t(j) = exp(-2 pi i j / (2 g t)),
// so each thread loads r values alpha (one per stage) and multiplies by
// compile-time roots of unity.  MID: the g = 1 pass, where j = 0 and alpha = 1.
template <bool MID, int T, int K>
__device__ __forceinline__ float2 twiddle(const float2 (&alpha)[4]) {
    constexpr int n = 8 * K / T;
    constexpr int s = T == 1 ? 0 : T == 2 ? 1 : T == 4 ? 2 : 3;
    if (MID) return make_float2(cos16(n), -sin16(n));
    if (n == 0) return alpha[s];
    return cmul(alpha[s], make_float2(cos16(n), -sin16(n)));
}

template <int R, bool MID, int T, int M0>
__device__ __forceinline__ void dif_pairs(float2 (&e)[R], const float2 (&alpha)[4]) {
    if constexpr (M0 < R) {
        if constexpr ((M0 & T) == 0) {
            constexpr int K = M0 & (T - 1);
            const float2 a = e[M0], c = e[M0 + T];
            e[M0] = cadd(a, c);
            const float2 d = csub(a, c);
            if constexpr (MID && K == 0)
                e[M0 + T] = d;
            else
                e[M0 + T] = cmul(d, twiddle<MID, T, K>(alpha));
        }
        dif_pairs<R, MID, T, M0 + 1>(e, alpha);
    }
}
template <int R, bool MID, int T, int M0>
__device__ __forceinline__ void dit_pairs(float2 (&e)[R], const float2 (&alpha)[4]) {
    if constexpr (M0 < R) {
        if constexpr ((M0 & T) == 0) {
            constexpr int K = M0 & (T - 1);
            const float2 a = e[M0];
            float2 c;
            if constexpr (MID && K == 0)
                c = e[M0 + T];
            else
                c = cmulc(e[M0 + T], twiddle<MID, T, K>(alpha));
            e[M0] = cadd(a, c);
            e[M0 + T] = csub(a, c);
        }
        dit_pairs<R, MID, T, M0 + 1>(e, alpha);
    }
}
// r radix-2 DIF stages on the tuple e[m] = x[b + j + m*g], halves g*R/2 .. g
template <int R, bool MID, int T = R / 2>
__device__ __forceinline__ void dif_stages(float2 (&e)[R], const float2 (&alpha)[4]) {
    if constexpr (T >= 1) {
        dif_pairs<R, MID, T, 0>(e, alpha);
        dif_stages<R, MID, T / 2>(e, alpha);
    }
}
// r radix-2 DIT stages with conjugate twiddles, halves g .. g*R/2 (stages T < TEND)
template <int R, bool MID, int T = 1, int TEND = R>
__device__ __forceinline__ void dit_stages(float2 (&e)[R], const float2 (&alpha)[4]) {
    if constexpr (T < TEND) {
        dit_pairs<R, MID, T, 0>(e, alpha);
        dit_stages<R, MID, T * 2, TEND>(e, alpha);
    }
}

// Pruned first forward stage: in the pass that reads the rows from HBM, tuple
// elements m >= R/2 sit at p >= M/2 >= isx and are zero, so the largest-half
// butterflies reduce to e[m + R/2] = e[m] * w.
template <int R, int M0 = 0>
__device__ __forceinline__ void dif_first_pruned(float2 (&e)[R], const float2 (&alpha)[4]) {
    if constexpr (M0 < R / 2) {
        e[M0 + R / 2] = cmul(e[M0], twiddle<false, R / 2, M0>(alpha));
        dif_first_pruned<R, M0 + 1>(e, alpha);
    }
}
// Pruned last inverse stage: only outputs p < M/2 (m < R/2) are ever stored.
template <int R, int M0 = 0>
__device__ __forceinline__ void dit_last_pruned(float2 (&e)[R], const float2 (&alpha)[4]) {
    if constexpr (M0 < R / 2) {
        constexpr int T = R / 2;
        const float2 c = cmulc(e[M0 + T], twiddle<false, T, M0>(alpha));
        e[M0] = cadd(e[M0], c);
        dit_last_pruned<R, M0 + 1>(e, alpha);
    }
}

struct RowPair {
    const FilterArgs* a;
    float* r0;
    float* r1;     // nullptr: unpaired last row
    float q0, q1;  // sdd^2 + dv^2 for each row
    float sdd, cu, pitch;
    __device__ float2 load(int p) const {
        if (p >= a->isx) return make_float2(0.f, 0.f);
        // cosine weight sdd / sqrt(sdd^2 + du^2 + dv^2) in fp32 (rel. error ~1e-7,
        // far inside the 2e-5 filter tolerance of tests/test_filter.py)
        const float du = ((float)p - cu) * pitch;
        const float x = r0[p] * (sdd * rsqrtf(fmaf(du, du, q0)));
        const float y = r1 ? r1[p] * (sdd * rsqrtf(fmaf(du, du, q1))) : 0.f;
        return make_float2(x, y);
    }
    __device__ void store(int p, float2 v) const {
        if (p >= a->isx) return;
        r0[p] = v.x;
        if (r1) r1[p] = v.y;
    }
};

// One grouped pass over all tuples.  KIND: 0 forward (DIF), 1 fused middle
// (DIF, * H, DIT; g == 1), 2 inverse (DIT).  FG: the pass reads the rows from HBM
// (first forward pass); TG: it writes them back (last inverse pass).
template <int R, int KIND, bool FG, bool TG>
__device__ void pass(const FilterArgs& a, float2* x, const RowPair& rp, int lg, const float2* tw) {
    constexpr int r = R == 2 ? 1 : R == 4 ? 2 : R == 8 ? 3 : 4;
    // pruning applies when the pass spans the whole row (g * R == M): only then are
    // tuple elements m >= R/2 exactly the positions p >= M/2
    constexpr bool kPruneIn = FG && KIND == 0 && R >= 2;
    constexpr bool kPruneOut = TG && KIND == 2 && R >= 2;
    const int g = 1 << lg;
    const int ntup = a.M >> r;
    for (int t = threadIdx.x; t < ntup; t += blockDim.x) {
        const int j = t & (g - 1);
        const int b = (t >> lg) << (lg + r);
        float2 alpha[4];
        if (KIND != 1) {
#pragma unroll
            for (int s = 0; s < r; ++s) alpha[s] = __ldg(tw + j * r + s);
        }
        float2 e[R];
#pragma unroll
        for (int m = 0; m < R; ++m) {
            const int p = b + j + m * g;
            if (kPruneIn)
                e[m] = m < R / 2 ? rp.load(p) : make_float2(0.f, 0.f);
            else
                e[m] = FG ? rp.load(p) : x[swz(p)];
        }
        if constexpr (KIND == 0) {
            if constexpr (kPruneIn) {
                dif_first_pruned<R>(e, alpha);
                dif_stages<R, false, R / 4>(e, alpha);
            } else {
                dif_stages<R, false>(e, alpha);
            }
        }
        if constexpr (KIND == 1) {
            dif_stages<R, true>(e, alpha);
#pragma unroll
            for (int m = 0; m < R; ++m) {
                const float h = __ldg(a.hperm + b + m);
                e[m].x *= h;
                e[m].y *= h;
            }
            dit_stages<R, true>(e, alpha);
        }
        if constexpr (KIND == 2) {
            if constexpr (kPruneOut) {
                dit_stages<R, false, 1, R / 2>(e, alpha);
                dit_last_pruned<R>(e, alpha);
            } else {
                dit_stages<R, false>(e, alpha);
            }
        }
#pragma unroll
        for (int m = 0; m < R; ++m) {
            const int p = b + j + m * g;
            if (TG) {
                if (!kPruneOut || m < R / 2) rp.store(p, e[m]);
            } else {
                x[swz(p)] = e[m];
            }
        }
    }
}

template <int KIND, bool FG, bool TG>
__device__ void run_pass(int r, const FilterArgs& a, float2* x, const RowPair& rp, int lg,
                         const float2* tw) {
    switch (r) {
        case 1: pass<2, KIND, FG, TG>(a, x, rp, lg, tw); break;
        case 2: pass<4, KIND, FG, TG>(a, x, rp, lg, tw); break;
        case 3: pass<8, KIND, FG, TG>(a, x, rp, lg, tw); break;
        default: pass<16, KIND, FG, TG>(a, x, rp, lg, tw); break;
    }
}

// ---- leading radix-3 / radix-5 pass of a mixed-radix length M = R0 * N2 ----------
// Forward (DIF): for j < N2, y[m'] = W_M^(j m') * sum_m x[j + m N2] W_R0^(m m'), stored at
// m' N2 + j; the N2-point radix-2 passes then run inside each of the R0 blocks, so the
// spectrum lands at sigma(m' N2 + j) = m' + R0 * bitrev(j).  Inverse (DIT): the radix-2
// passes first, then x[j + m N2] = sum_m' W_R0^(-m m') W_M^(-j m') y_m'[j].
template <int R0, bool INV>
__device__ __forceinline__ void dft_small(float2 (&e)[R0]) {
    // conj(W) for the inverse: swap the sign of the "i" rotations
    auto rot = [](float2 b, bool plus) {  // plus: +i*b, else -i*b
        return plus ? make_float2(-b.y, b.x) : make_float2(b.y, -b.x);
    };
    if constexpr (R0 == 3) {
        constexpr float c = -0.5f, sn = 0.866025403784438647f;  // cos, sin(2 pi / 3)
        const float2 t1 = cadd(e[1], e[2]), t2 = csub(e[1], e[2]);
        const float2 y0 = cadd(e[0], t1);
        const float2 a = make_float2(fmaf(c, t1.x, e[0].x), fmaf(c, t1.y, e[0].y));
        const float2 bb = make_float2(sn * t2.x, sn * t2.y);
        e[0] = y0;
        e[1] = cadd(a, rot(bb, INV));
        e[2] = cadd(a, rot(bb, !INV));
    } else {
        constexpr float c1 = 0.309016994374947424f, c2 = -0.809016994374947424f;
        constexpr float s1 = 0.951056516295153572f, s2 = 0.587785252292473129f;
        const float2 t1 = cadd(e[1], e[4]), t2 = cadd(e[2], e[3]);
        const float2 t3 = csub(e[1], e[4]), t4 = csub(e[2], e[3]);
        const float2 y0 = cadd(e[0], cadd(t1, t2));
        const float2 a1 = make_float2(fmaf(c1, t1.x, fmaf(c2, t2.x, e[0].x)),
                                      fmaf(c1, t1.y, fmaf(c2, t2.y, e[0].y)));
        const float2 a2 = make_float2(fmaf(c2, t1.x, fmaf(c1, t2.x, e[0].x)),
                                      fmaf(c2, t1.y, fmaf(c1, t2.y, e[0].y)));
        const float2 b1 = make_float2(fmaf(s1, t3.x, s2 * t4.x), fmaf(s1, t3.y, s2 * t4.y));
        const float2 b2 = make_float2(fmaf(s2, t3.x, -s1 * t4.x), fmaf(s2, t3.y, -s1 * t4.y));
        e[0] = y0;
        e[1] = cadd(a1, rot(b1, INV));
        e[4] = cadd(a1, rot(b1, !INV));
        e[2] = cadd(a2, rot(b2, INV));
        e[3] = cadd(a2, rot(b2, !INV));
    }
}

template <int R0>
__device__ void r0_forward(const FilterArgs& a, float2* x, const RowPair& rp) {
    const int N2 = a.N2;
    for (int j = threadIdx.x; j < N2; j += blockDim.x) {
        float2 e[R0];
#pragma unroll
        for (int m = 0; m < R0; ++m) e[m] = rp.load(j + m * N2);
        dft_small<R0, false>(e);
        x[swz(j)] = e[0];
#pragma unroll
        for (int m = 1; m < R0; ++m) x[swz(m * N2 + j)] = cmul(e[m], __ldg(a.twr + (m - 1) * N2 + j));
    }
}

template <int R0>
__device__ void r0_inverse(const FilterArgs& a, const float2* x, const RowPair& rp) {
    const int N2 = a.N2;
    for (int j = threadIdx.x; j < N2; j += blockDim.x) {
        float2 e[R0];
        e[0] = x[swz(j)];
#pragma unroll
        for (int m = 1; m < R0; ++m) e[m] = cmulc(x[swz(m * N2 + j)], __ldg(a.twr + (m - 1) * N2 + j));
        dft_small<R0, true>(e);
#pragma unroll
        for (int m = 0; m < R0; ++m) rp.store(j + m * N2, e[m]);
    }
}

__device__ __forceinline__ void ramp_filter_body(const FilterArgs& a) {
    extern __shared__ __align__(16) float2 fx[];
    const int y = (int)blockIdx.y;
    const int row0 = a.per_view ? a.vrow0[y] : a.row0;
    const int row1 = a.per_view ? a.vrow1[y] : a.row1;
    const int iv = row0 + 2 * (int)blockIdx.x;
    if (iv >= row1) return;
    float* base = a.img + (long long)(a.per_view ? a.slot[y] : y) * a.view_stride;
    RowPair rp;
    rp.a = &a;
    rp.r0 = base + (long long)iv * a.pitch;
    rp.r1 = iv + 1 < row1 ? rp.r0 + a.pitch : nullptr;
    const double dv0 = ((double)iv - a.cv) * a.pitch_mm, dv1 = ((double)(iv + 1) - a.cv) * a.pitch_mm;
    rp.q0 = (float)(a.sdd * a.sdd + dv0 * dv0);
    rp.q1 = (float)(a.sdd * a.sdd + dv1 * dv1);
    rp.sdd = (float)a.sdd;
    rp.cu = (float)a.cu;
    rp.pitch = (float)a.pitch_mm;

    const int ng = a.ngroups;
    int lm = 0;
    while ((1 << lm) < a.N2) ++lm;
    if (a.R0 > 1) {
        // mixed radix: leading radix-R0 pass from HBM, radix-2 passes inside the R0
        // blocks of N2, the fused middle, the inverse radix-2 passes, then radix-R0 to HBM
        if (a.R0 == 3) r0_forward<3>(a, fx, rp); else r0_forward<5>(a, fx, rp);
        __syncthreads();
        int lg = lm;
        for (int gi = 0; gi < ng - 1; ++gi) {
            lg -= a.r[gi];
            run_pass<0, false, false>(a.r[gi], a, fx, rp, lg, a.tw + a.twoff[gi]);
            __syncthreads();
        }
        run_pass<1, false, false>(a.r[ng - 1], a, fx, rp, 0, nullptr);
        lg = 0;
        for (int gi = ng - 2; gi >= 0; --gi) {
            __syncthreads();
            lg += a.r[gi + 1];
            run_pass<2, false, false>(a.r[gi], a, fx, rp, lg, a.tw + a.twoff[gi]);
        }
        __syncthreads();
        if (a.R0 == 3) r0_inverse<3>(a, fx, rp); else r0_inverse<5>(a, fx, rp);
        return;
    }
    // forward passes; g_i = M >> (r_0 + ... + r_i); the last one (g = 1) is fused
    // with the H multiply and the first inverse pass
    if (ng == 1) {  // M <= 16: one pass from HBM to HBM
        run_pass<1, true, true>(a.r[0], a, fx, rp, 0, nullptr);
        return;
    }
    int lg = lm - a.r[0];
    run_pass<0, true, false>(a.r[0], a, fx, rp, lg, a.tw + a.twoff[0]);
    __syncthreads();
    for (int gi = 1; gi < ng - 1; ++gi) {
        lg -= a.r[gi];
        run_pass<0, false, false>(a.r[gi], a, fx, rp, lg, a.tw + a.twoff[gi]);
        __syncthreads();
    }
    run_pass<1, false, false>(a.r[ng - 1], a, fx, rp, 0, nullptr);
    // remaining inverse passes, g growing back to M >> r_0
    lg = 0;
    for (int gi = ng - 2; gi >= 1; --gi) {
        __syncthreads();
        lg += a.r[gi + 1];
        run_pass<2, false, false>(a.r[gi], a, fx, rp, lg, a.tw + a.twoff[gi]);
    }
    __syncthreads();
    lg += a.r[1];
    run_pass<2, false, true>(a.r[0], a, fx, rp, lg, a.tw + a.twoff[0]);
}

// The M = 2560 launch (160 threads, isx 1248) is latency-bound: capping it at 64 registers
// (6 CTAs per SM, no spills) measured FDK e2e 57.8 -> 56.6 ms at 512^3.
__global__ void __launch_bounds__(160, 6) bp_ramp_filter_kernel_160(const __grid_constant__ FilterArgs a) {
    ramp_filter_body(a);
}
__global__ void __launch_bounds__(256) bp_ramp_filter_kernel(const __grid_constant__ FilterArgs a) {
    ramp_filter_body(a);
}

}  // namespace

int launch_ramp_filter(const FilterArgs& a, int nviews, cudaStream_t stream) {
    const int rows = a.row1 - a.row0;
    if (rows <= 0 || nviews <= 0) return 0;
    const size_t smem = (size_t)a.M * sizeof(float2);
    const int threads = a.M / 16 >= 256 ? 256 : (a.M / 16 >= 32 ? (a.M / 16 + 31) / 32 * 32 : 32);
    auto kern = threads <= 160 ? bp_ramp_filter_kernel_160 : bp_ramp_filter_kernel;
    if (smem > 48 * 1024) {
        const cudaError_t e =
            cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return (int)e;
    }
    dim3 grid((unsigned)((rows + 1) / 2), (unsigned)nviews);
    kern<<<grid, threads, smem, stream>>>(a);
    return (int)cudaGetLastError();
}

}  // namespace bpg
