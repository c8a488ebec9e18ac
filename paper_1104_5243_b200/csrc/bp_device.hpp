// bp_device.hpp -- host/device shared launch structures for the backprojection
// kernels (bp_kernels.cu) and the host pipeline (bp_runtime.cpp).
//
// Reference path replaced: bp::reconstruct's blocked view loop
// (proj/src/scheduler.cpp:77-100) driving bp::line_update_scalar
// (proj/src/kernel.cpp:49-85).  One kernel launch here = one "projection block"
// of the reference (block_b views), with the voxel accumulators held in
// registers across the batch instead of the reference's per-line linebuf.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace bpg {

// Maximum views per kernel launch (register batch).  The per-view matrices
// travel as kernel parameters (constant bank), so the batch is bounded by the
// 32 KB parameter space; 256 x 52 B + extras (13.5 KB) stays below it.  At 512^3 the
// resident run measured +0.6% for 124- over 64-view batches and +0.85% for 248- over
// 124-view batches (fewer volume passes).
constexpr int kMaxBatch = 256;

// One launch = one batch of views against one z-slab of the volume.
struct BatchArgs {
    int nviews;                  // views in this batch (1..kMaxBatch)
    int load_volume;             // 0: first batch, accumulators start at +0
    int slot[kMaxBatch];         // projection slot (ring index) of view k
    float A[kMaxBatch][12];      // narrowed matrices, reference a[] layout (geometry.hpp:25-37)
};

struct SlabArgs {
    float* vol;                  // slab volume [nz][L][L], x fastest (kernel.hpp:26-33)
    float* vol_out;              // final pass only: store the results here instead of vol
                                 // (same layout; may be a peer GPU's memory over NVLink)
    const float* proj;           // projection ring [slots][isy][pitch]
    const float* wx;             // world x of voxel i, float(offset_x + i*MM) (kernel.cpp:62)
    const float* wy;
    const float* wz;             // indexed by GLOBAL z
    unsigned long long* counters;  // [0]=tile pairs [1]=skipped pairs [2]=fallback pairs
    int L;                       // voxels per edge
    int z0;                      // first global z of the slab
    int nz;                      // slab depth
    int isx, isy;                // detector size
    int pitch;                   // row pitch of a projection slot, floats (multiple of 4)
    int nbx, nby, nbz;           // voxel blocks of the tiled kernel
    int debug;                   // BP_DEBUG bits (diagnostics only)
};

// Launchers (bp_kernels.cu).  All asynchronous on `stream`.
enum KernelKind : int { kKernelAuto = 0, kKernelSimple = 1 };

struct TileShape {
    int bx, by, bz;              // voxel block
    int tw, th;                  // tile pitch (texels; % 4 == 0, % 2 for dy) and ring rows (% 8 == 0)
    int stages;
    int threads;                 // consumer + producer threads per CTA
    int smem_bytes;
    int dy;                      // 1: fast-mode kernel over the pair ring (p, p_down - p),
                                 //    8-byte texels ("pair ring")
    int xp;                      // x-pairs per thread; 0: the shape's default variant
};

// Picks the tiled-kernel variant for edge length L (returns false if the
// tiled kernel cannot serve this L, e.g. odd L).
bool tile_shape_for(int L, TileShape* out);

// Encodes the TMA descriptor over the projection ring (CUtensorMap, 128 B).
// Returns 0 on success.
int encode_ring_tmap(void* tmap128, const float* ring, int isx, int isy, int pitch, int slots,
                     const TileShape& ts, char* err, int errlen);

// Same over the pair ring [slots][isy + 1][pitchx] float2 (8-byte texels): pair row e
// holds (p[e-1][c], p[e][c] - p[e-1][c]) with zero rows at e-1 = -1 and e = isy.
int encode_pair_tmap(void* tmap128, const float2* ringx, int isx, int isy, int pitchx, int slots,
                     const TileShape& ts, char* err, int errlen);

// Builds pair rows [0, isy] of n ring slots from the raw float ring (bp_aux.cu).
struct ExpandArgs {
    const float* ring;
    float2* ringx;
    int isx, isy, pitch, pitchx;  // pitch, pitchx: multiples of 4 (floats / float2)
    int e0, e1;                   // pair rows [e0, e1) (launch_expand); e1 <= e0: all, 0..isy
    int slot[kMaxBatch];
};
int launch_expand(const ExpandArgs& a, int n, void* stream);
// Same result from `blocks` co-resident 128-thread blocks (one per SM), for running
// under a backprojection launch.
int launch_expand_small(const ExpandArgs& a, int n, int blocks, void* stream);

// True when a pair-ring (dy) variant exists for this block shape.
bool has_pair_variant(const TileShape& ts);

int launch_tiled(const void* tmap128, const SlabArgs& s, const BatchArgs& b,
                 const TileShape& ts, bool strict, bool distance_weight, bool hw_rcp, void* stream);

// recip: 0 exact (recip.hpp:12), 1 approx12 (recip.hpp:14-18), 2 approx12_nr (recip.hpp:20-23)
int launch_simple(const SlabArgs& s, const BatchArgs& b, bool distance_weight, int recip,
                  void* stream);

int smem_bytes_for(const TileShape& ts);
// Largest ring (rows) with `ctas` CTAs per SM, at least min_rows.
int ring_rows_for_shape(const TileShape& ts, int min_rows, int ctas);

// Bitwise check of the kernel's paired reciprocal against __frcp_rn over the
// float bit patterns [lo_bits, hi_bits).  Synchronous.
int selftest_rcp(uint32_t lo_bits, uint32_t hi_bits, unsigned long long* mismatches);

// max|a-b|, max|b|, sum (a-b)^2 into res3; bitwise-different count into nbit.
int device_compare(const float* a, const float* b, unsigned long long n, double* res3,
                   unsigned long long* nbit);

// Reference BPCT clip ranges for views [view0, view0 + b.nviews) of a full-volume
// table (u16 pairs, precompute.hpp:14-25).
int launch_clip_ranges(const SlabArgs& s, const BatchArgs& b, uint16_t* ranges, int view0,
                       void* stream);

// Exact visible-update count (clip_stats semantics, precompute.cpp:93-103)
// for views [0,n) of the batch: adds into counters[3].
int launch_clip_count(const SlabArgs& s, const BatchArgs& b, void* stream);

// ---- FDK preprocessing: cosine weight + Ram-Lak row filter (bp_filter.cu) ----
constexpr int kMaxFilterM = 16384;  // FFT length; isx <= 8192
struct FilterArgs {
    float* img;             // view y: img + (per_view ? slot[y] : y) * view_stride
    long long view_stride;  // floats
    int pitch;              // floats per detector row
    int isx, row0, row1;    // rows [row0, row1) are filtered in place (per_view == 0)
    int per_view;           // nonzero: slot / vrow0 / vrow1 per blockIdx.y
    int slot[kMaxBatch];
    int vrow0[kMaxBatch], vrow1[kMaxBatch];
    int M, ngroups;         // FFT length (power of two >= 2*isx); register passes
    int r[8];               // radix-2 stages per pass, leading pass first (sum = log2 M)
    int twoff[8];           // pass i: twiddle table at tw + twoff[i], r[i] float2 per j < g_i
    const float2* tw;       // alpha_{i,j,s} = exp(-2 pi i j / (2 g_i 2^s)), s < r[i]
    const float* hperm;     // tau/M * H[sigma(p)], sigma = the forward network's output order
    double sdd, cu, cv, pitch_mm;
    // mixed radix: M = R0 * N2 (R0 in {3, 5}, N2 = 2^q); R0 == 1: pure radix-2 (N2 = M)
    int R0, N2;
    const float2* twr;      // W_M^(j m') for m' in [1, R0), j < N2: twr[(m'-1) N2 + j]
};
int launch_ramp_filter(const FilterArgs& a, int nviews, cudaStream_t stream);

}  // namespace bpg
