// bp_host.hpp -- host-side data model of the B200 backprojection library.
//
// Mirrors the reference data model (proj/src/geometry.hpp, datagen.hpp,
// kernel.hpp:26-33) with GPU-friendly storage: stacks and volumes live in
// pinned host memory from a size-keyed pool so H2D/D2H run at full PCIe rate.
#pragma once

#include <array>
#include <complex>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

namespace bph {

// ---- error taxonomy (proj/src/errors.hpp:9-30) -------------------------
struct config_error : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct io_error : std::runtime_error {
    explicit io_error(const std::string& m, long long off = -1)
        : std::runtime_error(off >= 0 ? m + " (at byte " + std::to_string(off) + ")" : m) {}
};
struct validation_error : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct device_error : std::runtime_error {  // CUDA failures -> BP_EINTERNAL
    using std::runtime_error::runtime_error;
};

// ---- pinned host memory pool -------------------------------------------
// Page-locked buffers (cudaHostAlloc) recycled by size so that repeated
// bp_reconstruct calls do not pay the pinning cost.  Falls back to aligned
// pageable memory when no CUDA driver is present (CPU-only hosts can still
// build stacks / read files).
void* pinned_alloc(size_t bytes);
void pinned_free(void* p);

// memcpy split over a persistent fork-join pool of host threads (the caller takes a
// share): the copy-semantics staging of bp_gpu_backproject and the readback into a
// pageable host volume.  One copy runs at a time (callers queue); small copies stay
// on the calling thread.
void parallel_memcpy(void* dst, const void* src, size_t bytes);
// true when p is ordinary pageable host memory (not page-locked, not device memory)
bool is_pageable(const void* p);
bool pinned_is_device_pinned(const void* p);
void pinned_trim();

template <class T>
struct PinnedArray {
    T* p = nullptr;
    size_t n = 0;
    PinnedArray() = default;
    explicit PinnedArray(size_t count) : n(count) {
        p = static_cast<T*>(pinned_alloc(count > 0 ? count * sizeof(T) : sizeof(T)));
    }
    PinnedArray(const PinnedArray&) = delete;
    PinnedArray& operator=(const PinnedArray&) = delete;
    PinnedArray(PinnedArray&& o) noexcept : p(o.p), n(o.n) { o.p = nullptr; o.n = 0; }
    PinnedArray& operator=(PinnedArray&& o) noexcept {
        if (this != &o) { reset(); p = o.p; n = o.n; o.p = nullptr; o.n = 0; }
        return *this;
    }
    ~PinnedArray() { reset(); }
    void reset() { if (p) pinned_free(p); p = nullptr; n = 0; }
    T* data() { return p; }
    const T* data() const { return p; }
    size_t size() const { return n; }
};

// ---- geometry (proj/src/geometry.hpp:13-37, geometry.cpp:11-25, 130-144) ----
struct Grid {
    int L = 0;
    double MM = 0.0;
    double ox = 0.0, oy = 0.0, oz = 0.0;
    static Grid cube(int L, double dx = 0.0, double dy = 0.0, double dz = 0.0);
    double wx(int i) const { return ox + i * MM; }
    double wy(int i) const { return oy + i * MM; }
    double wz(int i) const { return oz + i * MM; }
};

using Mat = std::array<double, 12>;  // column-interleaved a[] layout (geometry.hpp:25-32)

std::array<float, 12> narrowed(const Mat& a);
// throws validation_error when w <= 0 at a grid corner
void validate_matrix_for_grid(const Mat& a, const Grid& g);
// world-coordinate table float(o + i*MM) for i in [0, n) (kernel.cpp:53-54, 62)
std::vector<float> world_table(double origin, double MM, int n);

// Detector rows [r0, r1) that the voxel box [x0,x1]x[y0,y1]x[z0,z1] (voxel
// indices, inclusive) can read through the kernel's 2x2 footprint, with a
// guard band; clipped to [0, isy).  Returns r0 == r1 when the box misses the
// detector (no rows needed).  Falls back to the full detector for degenerate
// projections.
void row_window(const Mat& a, const Grid& g, int x0, int x1, int y0, int y1, int z0, int z1,
                int isy, int* r0, int* r1);

// Work-balanced contiguous z-slabs: boundaries b[0]=0 < ... <
// b[G]=L such that the estimated visible work per slab is as even as possible.
// The work estimate samples voxels on a coarse lattice and views with a stride
// (a contiguous analogue of the reference's cyclic z scheduling,
// scheduler.cpp:12-22).  Deterministic.
// Contiguous slab bounds (G+1) balancing a per-slice cost, bounds on multiples of align.
std::vector<int> partition_by_cost(const std::vector<double>& work, int G, int align);
std::vector<int> partition_slabs(const std::vector<Mat>& mats, int isx, int isy, const Grid& g,
                                 int G, std::vector<double>* work_out = nullptr);

// Round-robin chunk partition of the reference (scheduler.cpp:12-22) -- kept
// for API parity with partition_slices.
std::vector<std::vector<int>> partition_slices(int L, int threads, int chunk);

// ---- stacks / volumes -------------------------------------------------------
struct Stack {
    int isx = 0, isy = 0;
    std::vector<Mat> mats;
    PinnedArray<float> pixels;  // count * isy * isx, row-major per image
    int count() const { return (int)mats.size(); }
    const float* image(int k) const { return pixels.data() + (size_t)k * isy * isx; }
    float* image(int k) { return pixels.data() + (size_t)k * isy * isx; }
};

struct Volume {
    Grid grid;
    PinnedArray<float> vox;  // L^3, x fastest
    explicit Volume(const Grid& g) : grid(g), vox((size_t)g.L * g.L * g.L) {}
};

// ---- datagen (proj/src/datagen.cpp, restated; harness input, off the hot path) ---
struct Ellipsoid {
    double cx, cy, cz, ax, ay, az, density;
};
std::vector<Ellipsoid> named_phantom(const std::string& name);  // datagen.cpp:64-78
std::vector<Mat> circular_trajectory(int n, double sid, double sdd, int nu, int nv,
                                     double pitch);  // geometry.cpp:86-128
void forward_project(const std::vector<Ellipsoid>& ph, const Mat& a, int isx, int isy,
                     float* out);  // datagen.cpp:80-96

struct BaselineSpec {
    uint64_t seed = 20110428;
    int n_views = 496;
    int isx = 1248, isy = 960;
    double sid = 750.0, sdd = 1200.0, pitch = 0.32;
    double arc_deg = -1.0;         // <0: 200 deg + fan angle
    double jitter_mm = 0.5, jitter_deg = 0.1;
    int n_ellipsoids = 10;
    int filter = 1;                // cosine weight + row ramp filter
    int threads = 0;               // 0 = hardware concurrency
};
std::vector<Mat> baseline_trajectory(const BaselineSpec& s);
std::vector<Ellipsoid> baseline_phantom(const BaselineSpec& s);
Stack make_baseline_stack(const BaselineSpec& s);
// FDK projection preprocessing: cosine weight sdd / sqrt(sdd^2 + du^2 + dv^2)
// and a row-wise Ram-Lak ramp filter by zero-padded FFT (double precision).
void cosine_ramp_filter(float* img, int isx, int isy, double sid, double sdd, double pitch);
// The ramp filter's frequency response: M = smallest power of two >= 2*isx,
// tau = pitch*sid/sdd, H[k] = DFT_M(h)[k] (real; h is real and even), and the
// forward twiddles exp(-2 pi i k / M), k < M/2.
struct RampSpectrum {
    int M = 0;
    double tau = 0.0;
    std::vector<double> H;
    std::vector<std::complex<double>> tw;
};
RampSpectrum ramp_spectrum(int isx, double sid, double sdd, double pitch);

// ---- file formats (datagen.hpp:49-57, precompute.hpp:41-43) ----------------
void write_stack(const std::string& path, const Stack& s);
Stack read_stack(const std::string& path);
void write_volume(const std::string& path, const Volume& v);
Volume read_volume(const std::string& path);

// BPCT clip cache (precompute.hpp:14-43): "BPCT", u32 L, u32 count, count*L^2 (u16 first, u16 last)
struct ClipTable {
    int L = 0, n_views = 0;
    std::vector<uint16_t> ranges;
    uint64_t total_updates() const;  // clip_stats (precompute.cpp:93-103)
};
void write_clip_table(const std::string& path, const ClipTable& t);
ClipTable read_clip_table(const std::string& path);

double psnr(const float* v, const float* ref, size_t n, double peak);  // psnr.hpp:14-29

}  // namespace bph
