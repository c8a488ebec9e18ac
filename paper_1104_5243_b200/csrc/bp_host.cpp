// bp_host.cpp -- host data model, datagen, file formats, partitioner.
// See bp_host.hpp for the reference correspondences.
#include "bp_host.hpp"

#include <cuda_runtime.h>

#include <algorithm>
#if defined(__SSE2__)
#include <emmintrin.h>
#endif
#include <atomic>
#include <chrono>
#include <cmath>
#include <complex>
#include <condition_variable>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <map>
#include <mutex>
#include <thread>
#include <unordered_map>

namespace bph {

// ============================================================================
// pinned pool

namespace {
struct PoolState {
    std::mutex mu;
    std::multimap<size_t, void*> free_list;             // size -> buffer
    std::unordered_map<void*, std::pair<size_t, bool>> live;  // buffer -> (size, pinned)
    size_t cached = 0;
    int cuda_ok = -1;
};
PoolState& pool() {
    static PoolState* p = new PoolState();  // intentionally leaked: outlives static dtors
    return *p;
}
bool cuda_usable(PoolState& P) {
    if (P.cuda_ok < 0) {
        int n = 0;
        P.cuda_ok = (cudaGetDeviceCount(&n) == cudaSuccess && n > 0) ? 1 : 0;
        if (!P.cuda_ok) cudaGetLastError();
    }
    return P.cuda_ok == 1;
}
constexpr size_t kPoolCacheLimit = (size_t)16 << 30;
}  // namespace

namespace {

// Copy with non-temporal (streaming) stores: the destination (pinned staging that a DMA
// reads next, or the caller's volume) is not re-read by this thread, and streaming
// stores skip the read-for-ownership of every destination line -- a third of the memory
// traffic of a cached memcpy, which matters while a full-rate H2D reads the same DRAM.
void stream_copy(char* dst, const char* src, size_t n) {
#if defined(__SSE2__)
    // head: up to 16-byte alignment of the destination
    const size_t head = std::min(n, (size_t)((16 - ((uintptr_t)dst & 15)) & 15));
    std::memcpy(dst, src, head);
    dst += head;
    src += head;
    n -= head;
    size_t i = 0;
    for (; i + 64 <= n; i += 64) {
        const __m128i a = _mm_loadu_si128(reinterpret_cast<const __m128i*>(src + i));
        const __m128i b = _mm_loadu_si128(reinterpret_cast<const __m128i*>(src + i + 16));
        const __m128i c = _mm_loadu_si128(reinterpret_cast<const __m128i*>(src + i + 32));
        const __m128i d = _mm_loadu_si128(reinterpret_cast<const __m128i*>(src + i + 48));
        _mm_stream_si128(reinterpret_cast<__m128i*>(dst + i), a);
        _mm_stream_si128(reinterpret_cast<__m128i*>(dst + i + 16), b);
        _mm_stream_si128(reinterpret_cast<__m128i*>(dst + i + 32), c);
        _mm_stream_si128(reinterpret_cast<__m128i*>(dst + i + 48), d);
    }
    _mm_sfence();  // streaming stores are weakly ordered: drain before the job completes
    std::memcpy(dst + i, src + i, n - i);
#else
    std::memcpy(dst, src, n);
#endif
}

// Fork-join pool for the staging copies of copy-semantics uploads and the pageable
// readback: a job is a byte range split in equal parts, part 0 copied by the caller.
// Jobs arrive back to back (one ~4.8 MB view every ~80 us during a reconstruction), so
// idle workers spin on the job counter for up to 2 ms before sleeping on a
// condition variable, and the caller spins on the completion count: a condition-variable
// wake-up per job (tens of us for 7 workers) held the per-view copy to ~22 GB/s on the
// box, against ~60 GB/s for 8 memcpy threads running beside a full-rate H2D
// (tools/host_memcpy_probe.cpp).
class CopyPool {
public:
    CopyPool() {
        const unsigned hc = std::max(1u, std::thread::hardware_concurrency());
        // 12 copy threads on the 16-core box: 8 -> 12 measured e2e_copy 68.0 -> 61.9 ms
        // (14 and 16 no better; the H2D reading the staging shares the same DRAM)
        nworkers_ = (int)std::min(11u, hc > 2 ? hc * 3 / 4 - 1 : 0u);
        // A/B knobs: worker count, spin time before sleeping (0 = sleep at once)
        if (const char* e = std::getenv("BP_COPY_THREADS")) nworkers_ = std::max(0, std::atoi(e) - 1);
        if (const char* e = std::getenv("BP_COPY_SPIN_US")) spin_us_ = std::max(0, std::atoi(e));
        for (int i = 0; i < nworkers_; ++i) th_.emplace_back([this, i] { run(i + 1); });
    }
    ~CopyPool() {
        {
            std::lock_guard<std::mutex> g(mu_);
            stop_.store(true);
            gen_.fetch_add(1, std::memory_order_release);
        }
        cv_.notify_all();
        for (auto& t : th_) t.join();
    }
    void copy(void* dst, const void* src, size_t bytes) {
        if (nworkers_ == 0 || bytes < ((size_t)1 << 20)) {
            std::memcpy(dst, src, bytes);
            return;
        }
        std::lock_guard<std::mutex> one(job_mu_);  // one job at a time
        dst_ = static_cast<char*>(dst);
        src_ = static_cast<const char*>(src);
        bytes_ = bytes;
        pending_.store(nworkers_, std::memory_order_relaxed);
        {
            // under mu_ so that a worker between its last spin check and cv wait sees it
            std::lock_guard<std::mutex> g(mu_);
            gen_.fetch_add(1, std::memory_order_release);
        }
        cv_.notify_all();
        part(0);
        while (pending_.load(std::memory_order_acquire) > 0) {
        }
    }

private:
    int spin_us_ = 2000;
    void part(int i) {
        const int parts = nworkers_ + 1;
        // 4 KB-aligned split points
        auto at = [&](int k) { return std::min(bytes_, ((bytes_ * (size_t)k / parts) + 4095) & ~(size_t)4095); };
        const size_t a = i == 0 ? 0 : at(i), b = i == parts - 1 ? bytes_ : at(i + 1);
        if (b > a) stream_copy(dst_ + a, src_ + a, b - a);
    }
    void run(int i) {
        uint64_t seen = 0;
        for (;;) {
            const auto t0 = std::chrono::steady_clock::now();
            unsigned spins = 0;
            while (gen_.load(std::memory_order_acquire) == seen) {
                if ((++spins & 255u) == 0 &&
                    std::chrono::steady_clock::now() - t0 > std::chrono::microseconds(spin_us_)) {
                    std::unique_lock<std::mutex> g(mu_);
                    cv_.wait(g, [&] { return gen_.load(std::memory_order_acquire) != seen; });
                }
            }
            seen = gen_.load(std::memory_order_acquire);
            if (stop_.load()) return;
            part(i);
            pending_.fetch_sub(1, std::memory_order_acq_rel);
        }
    }
    int nworkers_ = 0;
    std::vector<std::thread> th_;
    std::mutex mu_, job_mu_;
    std::condition_variable cv_;
    std::atomic<uint64_t> gen_{0};
    std::atomic<bool> stop_{false};
    std::atomic<int> pending_{0};
    char* dst_ = nullptr;
    const char* src_ = nullptr;
    size_t bytes_ = 0;
};

CopyPool& copy_pool() {
    static CopyPool* p = new CopyPool();  // never destroyed: workers may outlive statics
    return *p;
}

}  // namespace

void parallel_memcpy(void* dst, const void* src, size_t bytes) { copy_pool().copy(dst, src, bytes); }

bool is_pageable(const void* p) {
    cudaPointerAttributes a{};
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return true;
    }
    return a.type == cudaMemoryTypeUnregistered;
}

void* pinned_alloc(size_t bytes) {
    auto& P = pool();
    std::lock_guard<std::mutex> g(P.mu);
    auto it = P.free_list.find(bytes);
    if (it != P.free_list.end()) {
        void* p = it->second;
        P.free_list.erase(it);
        P.cached -= bytes;
        P.live[p].first = bytes;
        return p;
    }
    void* p = nullptr;
    bool pinned = false;
    if (cuda_usable(P) && cudaHostAlloc(&p, bytes, cudaHostAllocPortable) == cudaSuccess) {
        pinned = true;
    } else {
        cudaGetLastError();
        p = std::aligned_alloc(4096, (bytes + 4095) & ~(size_t)4095);
        if (!p) throw std::bad_alloc();
    }
    P.live[p] = {bytes, pinned};
    return p;
}

void pinned_free(void* p) {
    if (!p) return;
    auto& P = pool();
    std::lock_guard<std::mutex> g(P.mu);
    auto it = P.live.find(p);
    if (it == P.live.end()) return;
    size_t bytes = it->second.first;
    bool pinned = it->second.second;
    if (pinned && P.cached + bytes <= kPoolCacheLimit) {
        P.free_list.emplace(bytes, p);
        P.cached += bytes;
        return;
    }
    P.live.erase(it);
    if (pinned)
        cudaFreeHost(p);
    else
        std::free(p);
}

bool pinned_is_device_pinned(const void* p) {
    auto& P = pool();
    std::lock_guard<std::mutex> g(P.mu);
    auto it = P.live.find(const_cast<void*>(p));
    return it != P.live.end() && it->second.second;
}

void pinned_trim() {
    auto& P = pool();
    std::lock_guard<std::mutex> g(P.mu);
    for (auto& kv : P.free_list) {
        auto it = P.live.find(kv.second);
        bool pinned = it != P.live.end() && it->second.second;
        if (it != P.live.end()) P.live.erase(it);
        if (pinned)
            cudaFreeHost(kv.second);
        else
            std::free(kv.second);
    }
    P.free_list.clear();
    P.cached = 0;
}

// ============================================================================
// geometry

Grid Grid::cube(int L, double dx, double dy, double dz) {
    if (L < 1) throw config_error("grid edge must be >= 1 voxel");
    Grid g;
    g.L = L;
    g.MM = 256.0 / L;
    const double off = -0.5 * (L - 1) * g.MM;
    g.ox = off + dx;
    g.oy = off + dy;
    g.oz = off + dz;
    return g;
}

std::array<float, 12> narrowed(const Mat& a) {
    std::array<float, 12> f;
    for (int i = 0; i < 12; ++i) f[i] = static_cast<float>(a[i]);
    return f;
}

void validate_matrix_for_grid(const Mat& a, const Grid& g) {
    const double lo[3] = {g.ox, g.oy, g.oz};
    const double hi[3] = {g.wx(g.L - 1), g.wy(g.L - 1), g.wz(g.L - 1)};
    for (int i = 0; i < 8; ++i) {
        const double x = (i & 1) ? hi[0] : lo[0];
        const double y = (i & 2) ? hi[1] : lo[1];
        const double z = (i & 4) ? hi[2] : lo[2];
        const double w = a[2] * x + a[5] * y + a[8] * z + a[11];
        if (!(w > 0.0)) {
            char buf[160];
            std::snprintf(buf, sizeof buf, "matrix has w <= 0 at grid corner (%g, %g, %g) mm", x, y,
                          z);
            throw validation_error(buf);
        }
    }
}

std::vector<float> world_table(double origin, double MM, int n) {
    std::vector<float> t((size_t)n);
    for (int i = 0; i < n; ++i) t[(size_t)i] = static_cast<float>(origin + i * MM);
    return t;
}

void row_window(const Mat& a, const Grid& g, int x0, int x1, int y0, int y1, int z0, int z1,
                int isy, int* r0, int* r1) {
    // The same corner rule as the kernel's producer (bp_kernels.cu): extrema of
    // the linear-fractional map over the box are at its vertices; the kernel's
    // per-block rectangle [floor(min)-1, floor(max)+2] is contained in this
    // slab rectangle, widened by one more guard row.
    double umin = 1e300, umax = -1e300, vmin = 1e300, vmax = -1e300, wmin = 1e300;
    const auto f = narrowed(a);
    for (int i = 0; i < 8; ++i) {
        const double x = (double)static_cast<float>(g.wx((i & 1) ? x1 : x0));
        const double y = (double)static_cast<float>(g.wy((i & 2) ? y1 : y0));
        const double z = (double)static_cast<float>(g.wz((i & 4) ? z1 : z0));
        const double uw = (double)f[0] * x + (double)f[3] * y + (double)f[6] * z + (double)f[9];
        const double vw = (double)f[1] * x + (double)f[4] * y + (double)f[7] * z + (double)f[10];
        const double w = (double)f[2] * x + (double)f[5] * y + (double)f[8] * z + (double)f[11];
        wmin = std::min(wmin, w);
        umin = std::min(umin, uw / w);
        umax = std::max(umax, uw / w);
        vmin = std::min(vmin, vw / w);
        vmax = std::max(vmax, vw / w);
    }
    const double lim = 1048576.0;
    if (!(wmin > 0x1p-60) || !(std::fabs(vmin) < lim) || !(std::fabs(vmax) < lim) ||
        !(std::fabs(umin) < lim) || !(std::fabs(umax) < lim)) {
        *r0 = 0;
        *r1 = isy;
        return;
    }
    const long long lo = (long long)std::floor(vmin) - 2;
    const long long hi = (long long)std::floor(vmax) + 3;  // inclusive
    long long a0 = std::max<long long>(lo, 0), a1 = std::min<long long>(hi + 1, isy);
    if (a1 < a0) a1 = a0;
    *r0 = (int)a0;
    *r1 = (int)a1;
}

std::vector<int> partition_by_cost(const std::vector<double>& work, int G, int align) {
    const int L = (int)work.size();
    if (G < 1) throw config_error("slab count must be >= 1");
    if (G > L) throw config_error("more slabs than z-slices");
    align = std::max(1, align);
    std::vector<double> cum((size_t)L + 1, 0.0);
    for (int z = 0; z < L; ++z) {
        if (!(work[(size_t)z] >= 0)) throw config_error("slice cost must be >= 0");
        cum[(size_t)z + 1] = cum[(size_t)z] + work[(size_t)z];
    }
    const double total = cum[(size_t)L];
    std::vector<int> b((size_t)G + 1, 0);
    b[0] = 0;
    b[(size_t)G] = L;
    for (int i = 1; i < G; ++i) {
        const double target = total * i / G;
        int z = (int)(std::lower_bound(cum.begin(), cum.end(), target) - cum.begin());
        // pick the closer of z-1, z
        if (z > 0 && std::fabs(cum[(size_t)z - 1] - target) < std::fabs(cum[(size_t)z] - target)) --z;
        z = (int)std::lround((double)z / align) * align;
        z = std::max(z, b[(size_t)i - 1] + 1);
        z = std::min(z, L - (G - i));
        b[(size_t)i] = z;
    }
    return b;
}

std::vector<int> partition_slabs(const std::vector<Mat>& mats, int isx, int isy, const Grid& g,
                                 int G, std::vector<double>* work_out) {
    const int L = g.L;
    if (G < 1) throw config_error("slab count must be >= 1");
    if (G > L) throw config_error("more slabs than z-slices");
    // Cost model = the tiled kernel's work, not visible voxels: per layer of voxel
    // blocks (the block shapes of tile_shape_for, bp_kernels.cu), the number of
    // (block, view) pairs that survive the producer's cull -- the block's 8 corners
    // projected, footprint [floor(min) - 1, floor(max) + 2] against the detector --
    // times the block's voxels, plus a per-pair overhead (the per-view header, line
    // constants and barrier, ~6% of a block's voxel work) and a per-
    // slice volume read-modify-write term.  A culled pair costs cull_cost of a computed one.
    // Views are strided (every 4th of 496); the counts are exact for those views.
    const int BX = L >= 512 ? 32 : 16, BY = L >= 512 ? 32 : (L >= 256 ? 16 : 8),
              BZ = L >= 256 ? 8 : 4;
    const int nbx = (L + BX - 1) / BX, nby = (L + BY - 1) / BY, nbz = (L + BZ - 1) / BZ;
    const int vstride = std::max<int>(1, (int)mats.size() / 128);
    std::vector<std::array<double, 12>> fm;
    for (size_t k = 0; k < mats.size(); k += (size_t)vstride) fm.push_back(mats[k]);
    std::vector<double> layer((size_t)nbz, 0.0);
    // a culled pair is not free: its share of the CTA's launch, volume pass and 32-view cull
    // passes, as a fraction of a computed pair (calibrated on the 8-way split of the 2048^3
    // + 60 mm grid, whose outer slabs are mostly culled pairs: DESIGN.md 7)
    double cull_cost = 0.07;
    if (const char* e = std::getenv("BP_CULL_COST")) cull_cost = std::atof(e);
    auto worker = [&](int t, int T) {
        for (int bz = t; bz < nbz; bz += T) {
            const double wz[2] = {g.wz(bz * BZ), g.wz(bz * BZ + BZ - 1)};
            double pairs = 0;
            for (const auto& A : fm)
                for (int by = 0; by < nby; ++by) {
                    const double wy[2] = {g.wy(by * BY), g.wy(by * BY + BY - 1)};
                    for (int bx = 0; bx < nbx; ++bx) {
                        const double wx[2] = {g.wx(bx * BX), g.wx(bx * BX + BX - 1)};
                        double umin = 1e30, umax = -1e30, vmin = 1e30, vmax = -1e30;
                        bool sane = true;
                        for (int c = 0; c < 8; ++c) {
                            const double X = wx[c & 1], Y = wy[(c >> 1) & 1], Z = wz[c >> 2];
                            const double w = A[2] * X + A[5] * Y + A[8] * Z + A[11];
                            if (!(w > 0)) { sane = false; break; }
                            const double u = (A[0] * X + A[3] * Y + A[6] * Z + A[9]) / w;
                            const double v = (A[1] * X + A[4] * Y + A[7] * Z + A[10]) / w;
                            umin = std::min(umin, u); umax = std::max(umax, u);
                            vmin = std::min(vmin, v); vmax = std::max(vmax, v);
                        }
                        if (sane && (std::floor(umax) + 2 < 0 || std::floor(umin) - 1 > isx - 1 ||
                                     std::floor(vmax) + 2 < 0 || std::floor(vmin) - 1 > isy - 1)) {
                            pairs += cull_cost;  // culled: the producer's cull and the CTA's fixed work
                            continue;
                        }
                        pairs += 1;
                    }
                }
            layer[(size_t)bz] = pairs;
        }
    };
    {
        int T = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
        std::vector<std::thread> th;
        for (int t = 0; t < T; ++t) th.emplace_back(worker, t, T);
        for (auto& x : th) x.join();
    }
    // per-slice cost in voxel-update units (per view)
    const double per_pair = (double)BX * BY * 1.06;       // one slice of a block, + overhead
    const double rmw = (double)nbx * BX * nby * BY * 0.02;  // volume read/write per slice
    std::vector<double> work((size_t)L, 0.0);
    for (int z = 0; z < L; ++z) work[(size_t)z] = layer[(size_t)(z / BZ)] * per_pair + rmw + 1e-3;
    // slab bounds on block-layer boundaries when the slabs are thick enough
    const int align = (L / G >= 4 * BZ) ? BZ : 1;
    std::vector<int> b = partition_by_cost(work, G, align);
    if (work_out) *work_out = work;
    return b;
}

std::vector<std::vector<int>> partition_slices(int L, int threads, int chunk) {
    if (threads < 1) throw config_error("threads must be >= 1");
    if (chunk < 1) throw config_error("chunk must be >= 1");
    std::vector<std::vector<int>> out((size_t)threads);
    const int nc = (L + chunk - 1) / chunk;
    for (int c = 0; c < nc; ++c)
        for (int z = c * chunk; z < std::min((c + 1) * chunk, L); ++z)
            out[(size_t)(c % threads)].push_back(z);
    return out;
}

// ============================================================================
// datagen

namespace {

void unit(double v[3]) {
    const double n = std::sqrt(v[0] * v[0] + v[1] * v[1] + v[2] * v[2]);
    v[0] /= n;
    v[1] /= n;
    v[2] /= n;
}

// chord of the ray o + t d (|d| = 1) through an axis-aligned ellipsoid
double chord_len(const Ellipsoid& e, const double o[3], const double d[3]) {
    const double p[3] = {(o[0] - e.cx) / e.ax, (o[1] - e.cy) / e.ay, (o[2] - e.cz) / e.az};
    const double q[3] = {d[0] / e.ax, d[1] / e.ay, d[2] / e.az};
    const double A = q[0] * q[0] + q[1] * q[1] + q[2] * q[2];
    const double B = p[0] * q[0] + p[1] * q[1] + p[2] * q[2];
    const double Cc = p[0] * p[0] + p[1] * p[1] + p[2] * p[2] - 1.0;
    const double disc = B * B - A * Cc;
    return disc > 0.0 ? 2.0 * std::sqrt(disc) / A : 0.0;
}

// left 3x3 block M (rows u, v, w) of the a[] layout and its inverse
void left3(const Mat& a, double m[3][3]) {
    for (int i = 0; i < 3; ++i) {
        m[0][i] = a[(size_t)(3 * i)];
        m[1][i] = a[(size_t)(3 * i + 1)];
        m[2][i] = a[(size_t)(3 * i + 2)];
    }
}

bool inv3(const double m[3][3], double inv[3][3]) {
    const double det = m[0][0] * (m[1][1] * m[2][2] - m[1][2] * m[2][1]) -
                       m[0][1] * (m[1][0] * m[2][2] - m[1][2] * m[2][0]) +
                       m[0][2] * (m[1][0] * m[2][1] - m[1][1] * m[2][0]);
    double sc = 0;
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) sc = std::max(sc, std::fabs(m[i][j]));
    if (std::fabs(det) <= 1e-14 * sc * sc * sc) return false;
    inv[0][0] = (m[1][1] * m[2][2] - m[1][2] * m[2][1]) / det;
    inv[0][1] = (m[0][2] * m[2][1] - m[0][1] * m[2][2]) / det;
    inv[0][2] = (m[0][1] * m[1][2] - m[0][2] * m[1][1]) / det;
    inv[1][0] = (m[1][2] * m[2][0] - m[1][0] * m[2][2]) / det;
    inv[1][1] = (m[0][0] * m[2][2] - m[0][2] * m[2][0]) / det;
    inv[1][2] = (m[0][2] * m[1][0] - m[0][0] * m[1][2]) / det;
    inv[2][0] = (m[1][0] * m[2][1] - m[1][1] * m[2][0]) / det;
    inv[2][1] = (m[0][1] * m[2][0] - m[0][0] * m[2][1]) / det;
    inv[2][2] = (m[0][0] * m[1][1] - m[0][1] * m[1][0]) / det;
    return true;
}

struct Rng {  // splitmix64: portable, seedable
    uint64_t s;
    explicit Rng(uint64_t seed) : s(seed) {}
    uint64_t next() {
        uint64_t z = (s += 0x9E3779B97F4A7C15ull);
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
        z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
        return z ^ (z >> 31);
    }
    double uni() { return (double)(next() >> 11) * 0x1p-53; }
    double uni(double lo, double hi) { return lo + (hi - lo) * uni(); }
};

Mat make_camera(const double S[3], const double eu[3], const double ev[3], const double ez[3],
                double fpx, double cu, double cv) {
    double rows[3][3];
    for (int i = 0; i < 3; ++i) {
        rows[0][i] = fpx * eu[i] + cu * ez[i];
        rows[1][i] = fpx * ev[i] + cv * ez[i];
        rows[2][i] = ez[i];
    }
    Mat a{};
    for (int i = 0; i < 3; ++i) {
        a[(size_t)(3 * i)] = rows[0][i];
        a[(size_t)(3 * i + 1)] = rows[1][i];
        a[(size_t)(3 * i + 2)] = rows[2][i];
    }
    for (int r = 0; r < 3; ++r)
        a[(size_t)(9 + r)] = -(rows[r][0] * S[0] + rows[r][1] * S[1] + rows[r][2] * S[2]);
    return a;
}

template <class F>
void parallel_for(int n, int threads, F&& f) {
    int T = threads > 0 ? threads : (int)std::max(1u, std::thread::hardware_concurrency());
    T = std::max(1, std::min(T, n));
    std::vector<std::thread> th;
    for (int t = 0; t < T; ++t)
        th.emplace_back([&, t] {
            for (int i = t; i < n; i += T) f(i);
        });
    for (auto& x : th) x.join();
}

}  // namespace

std::vector<Ellipsoid> named_phantom(const std::string& name) {
    if (name == "spheres3")
        return {{0, 0, 0, 80, 80, 80, 1.0}, {30, 0, 10, 12, 12, 12, 0.5}, {-30, 0, -10, 12, 12, 12, -0.5}};
    if (name == "shell") return {{0, 0, 0, 90, 90, 90, 1.0}, {0, 0, 0, 60, 60, 60, -1.0}};
    if (name == "point") return {{0, 0, 0, 0.5, 0.5, 0.5, 1.0}};
    throw config_error("unknown phantom '" + name + "' (spheres3, shell, point)");
}

std::vector<Mat> circular_trajectory(int n, double sid, double sdd, int nu, int nv, double pitch) {
    if (n < 1) throw config_error("need at least one view");
    if (!(sid > 0.0 && sid < sdd)) throw config_error("require 0 < sid < sdd");
    if (nu < 2 || nv < 2) throw config_error("detector must be at least 2x2 pixels");
    if (!(pitch > 0.0)) throw config_error("pixel pitch must be positive");
    std::vector<Mat> out;
    out.reserve((size_t)n);
    const double cu = 0.5 * (nu - 1), cv = 0.5 * (nv - 1), fpx = sdd / pitch;
    for (int k = 0; k < n; ++k) {
        const double th = 2.0 * M_PI * k / n;
        const double c = std::cos(th), s = std::sin(th);
        const double S[3] = {sid * c, sid * s, 0.0};
        const double ez[3] = {-c, -s, 0.0}, eu[3] = {-s, c, 0.0}, ev[3] = {0.0, 0.0, 1.0};
        out.push_back(make_camera(S, eu, ev, ez, fpx, cu, cv));
    }
    return out;
}

void forward_project(const std::vector<Ellipsoid>& ph, const Mat& a, int isx, int isy, float* out) {
    double m[3][3], inv[3][3];
    left3(a, m);
    if (!inv3(m, inv)) throw validation_error("degenerate projection matrix");
    const double p4[3] = {a[9], a[10], a[11]};
    double C[3];
    for (int r = 0; r < 3; ++r) C[r] = -(inv[r][0] * p4[0] + inv[r][1] * p4[1] + inv[r][2] * p4[2]);
    for (int iv = 0; iv < isy; ++iv)
        for (int iu = 0; iu < isx; ++iu) {
            double d[3] = {inv[0][0] * iu + inv[0][1] * iv + inv[0][2],
                           inv[1][0] * iu + inv[1][1] * iv + inv[1][2],
                           inv[2][0] * iu + inv[2][1] * iv + inv[2][2]};
            unit(d);
            double sum = 0.0;
            for (const auto& e : ph) sum += e.density * chord_len(e, C, d);
            out[(size_t)iv * isx + iu] = static_cast<float>(sum);
        }
}

std::vector<Mat> baseline_trajectory(const BaselineSpec& s) {
    if (s.n_views < 1) throw config_error("need at least one view");
    Rng rng(s.seed ^ 0x7472616A6563ull);
    const double half_w = 0.5 * s.isx * s.pitch;
    const double fan = 2.0 * std::atan(half_w / s.sdd);
    const double arc = s.arc_deg >= 0 ? s.arc_deg * M_PI / 180.0 : 200.0 * M_PI / 180.0 + fan;
    const double cu = 0.5 * (s.isx - 1), cv = 0.5 * (s.isy - 1), fpx = s.sdd / s.pitch;
    std::vector<Mat> out;
    out.reserve((size_t)s.n_views);
    for (int k = 0; k < s.n_views; ++k) {
        const double th = s.n_views > 1 ? arc * k / (s.n_views - 1) : 0.0;
        const double c = std::cos(th), sn = std::sin(th);
        double S[3] = {s.sid * c, s.sid * sn, 0.0};
        double ez[3] = {-c, -sn, 0.0}, eu[3] = {-sn, c, 0.0}, ev[3] = {0.0, 0.0, 1.0};
        // seeded jitter: source translation +-jitter_mm, detector frame rotation +-jitter_deg
        for (double& x : S) x += rng.uni(-s.jitter_mm, s.jitter_mm);
        const double ax = rng.uni(-1, 1) * s.jitter_deg * M_PI / 180.0;
        const double ay = rng.uni(-1, 1) * s.jitter_deg * M_PI / 180.0;
        const double az = rng.uni(-1, 1) * s.jitter_deg * M_PI / 180.0;
        const double cx = std::cos(ax), sx = std::sin(ax), cy = std::cos(ay), sy = std::sin(ay),
                     cz = std::cos(az), sz = std::sin(az);
        const double R[3][3] = {{cy * cz, -cy * sz, sy},
                                {sx * sy * cz + cx * sz, -sx * sy * sz + cx * cz, -sx * cy},
                                {-cx * sy * cz + sx * sz, cx * sy * sz + sx * cz, cx * cy}};
        auto rot = [&](double v[3]) {
            double r[3];
            for (int i = 0; i < 3; ++i) r[i] = R[i][0] * v[0] + R[i][1] * v[1] + R[i][2] * v[2];
            v[0] = r[0];
            v[1] = r[1];
            v[2] = r[2];
        };
        rot(eu);
        rot(ev);
        rot(ez);
        out.push_back(make_camera(S, eu, ev, ez, fpx, cu, cv));
    }
    return out;
}

std::vector<Ellipsoid> baseline_phantom(const BaselineSpec& s) {
    Rng rng(s.seed ^ 0x7068616E746Full);
    std::vector<Ellipsoid> e;
    for (int i = 0; i < s.n_ellipsoids; ++i) {
        Ellipsoid x;
        x.cx = rng.uni(-70, 70);
        x.cy = rng.uni(-70, 70);
        x.cz = rng.uni(-50, 50);
        x.ax = rng.uni(10, 100);
        x.ay = rng.uni(10, 100);
        x.az = rng.uni(10, 100);
        x.density = rng.uni(-1, 2);
        e.push_back(x);
    }
    return e;
}

namespace {
// iterative radix-2 complex FFT, in place (n power of two).  Complex products
// are written out by hand (std::complex's operator* goes through __muldc3).
void fft(std::vector<std::complex<double>>& a, bool inverse,
         const std::vector<std::complex<double>>& tw) {
    const size_t n = a.size();
    double* d = reinterpret_cast<double*>(a.data());
    for (size_t i = 1, j = 0; i < n; ++i) {
        size_t bit = n >> 1;
        for (; j & bit; bit >>= 1) j ^= bit;
        j ^= bit;
        if (i < j) std::swap(a[i], a[j]);
    }
    const double sgn = inverse ? -1.0 : 1.0;
    for (size_t len = 2; len <= n; len <<= 1) {
        const size_t step = n / len, half = len / 2;
        for (size_t i = 0; i < n; i += len)
            for (size_t k = 0; k < half; ++k) {
                const double wr = tw[k * step].real(), wi = sgn * tw[k * step].imag();
                double* u = d + 2 * (i + k);
                double* v = d + 2 * (i + k + half);
                const double vr = v[0] * wr - v[1] * wi, vi = v[0] * wi + v[1] * wr;
                v[0] = u[0] - vr;
                v[1] = u[1] - vi;
                u[0] += vr;
                u[1] += vi;
            }
    }
    if (inverse) {
        const double s = 1.0 / (double)n;
        for (size_t i = 0; i < 2 * n; ++i) d[i] *= s;
    }
}
}  // namespace

RampSpectrum ramp_spectrum(int isx, double sid, double sdd, double pitch) {
    // Ram-Lak kernel sampled at the isocentre pitch tau (Kak & Slaney ch. 3,
    // eq. 61), zero-padded to M >= 2*isx so the circular convolution is linear
    // on the isx outputs; h is real and even, so its spectrum is real.
    if (isx < 2) throw config_error("detector must be at least 2 pixels wide");
    if (!(sid > 0) || !(sdd > 0) || !(pitch > 0)) throw config_error("filter geometry must be positive");
    RampSpectrum r;
    size_t M = 1;
    while (M < (size_t)2 * isx) M <<= 1;
    r.M = (int)M;
    r.tau = pitch * sid / sdd;  // detector sampling at the isocentre
    const double tau = r.tau;
    std::vector<std::complex<double>> tw(M / 2);
    for (size_t k = 0; k < M / 2; ++k) tw[k] = std::polar(1.0, -2.0 * M_PI * (double)k / (double)M);
    std::vector<std::complex<double>> h(M, 0.0);
    for (long n = -(isx - 1); n <= isx - 1; ++n) {
        double v;
        if (n == 0)
            v = 1.0 / (4.0 * tau * tau);
        else if (n & 1)
            v = -1.0 / (M_PI * M_PI * (double)n * (double)n * tau * tau);
        else
            v = 0.0;
        h[(size_t)((n + (long)M) % (long)M)] = v;
    }
    fft(h, false, tw);
    r.H.resize(M);
    for (size_t k = 0; k < M; ++k) r.H[k] = h[k].real();
    r.tw = std::move(tw);
    return r;
}

void cosine_ramp_filter(float* img, int isx, int isy, double sid, double sdd, double pitch) {
    // FDK preprocessing: cosine weight, then a row-wise
    // Ram-Lak ramp filter applied by zero-padded FFT convolution.
    const RampSpectrum rs = ramp_spectrum(isx, sid, sdd, pitch);
    const size_t M = (size_t)rs.M;
    const double tau = rs.tau;
    const double cu = 0.5 * (isx - 1), cv = 0.5 * (isy - 1);
    // Two real rows per complex FFT: h is real and even, so its spectrum is
    // real and filtering (a + i b) yields (a*h) + i (b*h) exactly.
    std::vector<std::complex<double>> row(M);
    auto weighted = [&](int iv, int iu) {
        const double du = (iu - cu) * pitch, dv = (iv - cv) * pitch;
        return (double)img[(size_t)iv * isx + iu] * sdd / std::sqrt(sdd * sdd + du * du + dv * dv);
    };
    for (int iv = 0; iv < isy; iv += 2) {
        const bool pair = iv + 1 < isy;
        for (size_t i = 0; i < M; ++i) row[i] = 0.0;
        for (int iu = 0; iu < isx; ++iu)
            row[(size_t)iu] = std::complex<double>(weighted(iv, iu), pair ? weighted(iv + 1, iu) : 0.0);
        fft(row, false, rs.tw);
        for (size_t i = 0; i < M; ++i) row[i] *= rs.H[i];
        fft(row, true, rs.tw);
        float* r0 = img + (size_t)iv * isx;
        for (int iu = 0; iu < isx; ++iu) r0[iu] = static_cast<float>(row[(size_t)iu].real() * tau);
        if (pair) {
            float* r1 = img + (size_t)(iv + 1) * isx;
            for (int iu = 0; iu < isx; ++iu) r1[iu] = static_cast<float>(row[(size_t)iu].imag() * tau);
        }
    }
}

Stack make_baseline_stack(const BaselineSpec& s) {
    if (s.isx < 2 || s.isy < 2) throw config_error("detector must be at least 2x2 pixels");
    Stack st;
    st.isx = s.isx;
    st.isy = s.isy;
    st.mats = baseline_trajectory(s);
    const auto ph = baseline_phantom(s);
    st.pixels = PinnedArray<float>((size_t)s.n_views * s.isx * s.isy);
    parallel_for(s.n_views, s.threads, [&](int k) {
        float* img = st.image(k);
        forward_project(ph, st.mats[(size_t)k], s.isx, s.isy, img);
        if (s.filter) cosine_ramp_filter(img, s.isx, s.isy, s.sid, s.sdd, s.pitch);
    });
    return st;
}

// ============================================================================
// file formats

namespace {
template <class T>
void put(std::ofstream& f, const T& v) {
    f.write(reinterpret_cast<const char*>(&v), sizeof v);
}
void read_exact(std::ifstream& f, char* dst, std::streamsize n, const char* what,
                const std::string& path) {
    const long long pos = (long long)f.tellg();
    f.read(dst, n);
    if (!f) throw io_error("truncated " + std::string(what) + " in " + path, pos + (long long)f.gcount());
}
template <class T>
T get(std::ifstream& f, const char* what, const std::string& path) {
    T v;
    read_exact(f, reinterpret_cast<char*>(&v), sizeof v, what, path);
    return v;
}
void magic(std::ifstream& f, const char* m, const std::string& path) {
    char b[4];
    f.read(b, 4);
    if (!f || std::memcmp(b, m, 4) != 0)
        throw io_error("bad magic in " + path + " (expected " + m + ")", 0);
}
}  // namespace

void write_stack(const std::string& path, const Stack& s) {
    std::ofstream f(path, std::ios::binary);
    if (!f) throw io_error("cannot open " + path + " for writing");
    f.write("BPST", 4);
    put(f, (uint32_t)s.isx);
    put(f, (uint32_t)s.isy);
    put(f, (uint32_t)s.count());
    for (const auto& m : s.mats) f.write(reinterpret_cast<const char*>(m.data()), 12 * sizeof(double));
    f.write(reinterpret_cast<const char*>(s.pixels.data()),
            (std::streamsize)((size_t)s.count() * s.isx * s.isy * sizeof(float)));
    if (!f) throw io_error("write failed for " + path);
}

Stack read_stack(const std::string& path) {
    std::ifstream f(path, std::ios::binary);
    if (!f) throw io_error("cannot open " + path);
    magic(f, "BPST", path);
    const uint32_t isx = get<uint32_t>(f, "ISX", path), isy = get<uint32_t>(f, "ISY", path),
                   n = get<uint32_t>(f, "count", path);
    if (isx < 2 || isy < 2 || n < 1 || (uint64_t)isx * isy * n > ((uint64_t)1 << 33))
        throw io_error("implausible stack dimensions in " + path, 4);
    Stack s;
    s.isx = (int)isx;
    s.isy = (int)isy;
    s.mats.resize(n);
    for (auto& m : s.mats)
        read_exact(f, reinterpret_cast<char*>(m.data()), 12 * sizeof(double), "matrix block", path);
    s.pixels = PinnedArray<float>((size_t)n * isx * isy);
    read_exact(f, reinterpret_cast<char*>(s.pixels.data()),
               (std::streamsize)((size_t)n * isx * isy * sizeof(float)), "pixel payload", path);
    return s;
}

void write_volume(const std::string& path, const Volume& v) {
    std::ofstream f(path, std::ios::binary);
    if (!f) throw io_error("cannot open " + path + " for writing");
    f.write("BPVL", 4);
    put(f, (uint32_t)v.grid.L);
    f.write(reinterpret_cast<const char*>(v.vox.data()),
            (std::streamsize)(v.vox.size() * sizeof(float)));
    if (!f) throw io_error("write failed for " + path);
}

Volume read_volume(const std::string& path) {
    std::ifstream f(path, std::ios::binary);
    if (!f) throw io_error("cannot open " + path);
    magic(f, "BPVL", path);
    const uint32_t L = get<uint32_t>(f, "L", path);
    if (L < 1 || L > 4096) throw io_error("implausible volume edge in " + path, 4);
    Volume v(Grid::cube((int)L));
    read_exact(f, reinterpret_cast<char*>(v.vox.data()),
               (std::streamsize)(v.vox.size() * sizeof(float)), "voxel payload", path);
    return v;
}

uint64_t ClipTable::total_updates() const {
    uint64_t t = 0;
    for (size_t i = 0; i + 1 < ranges.size(); i += 2)
        if (ranges[i] != 0xFFFF) t += (uint64_t)(ranges[i + 1] - ranges[i] + 1);
    return t;
}

void write_clip_table(const std::string& path, const ClipTable& t) {
    std::ofstream f(path, std::ios::binary);
    if (!f) throw io_error("cannot open " + path + " for writing");
    f.write("BPCT", 4);
    put(f, (uint32_t)t.L);
    put(f, (uint32_t)t.n_views);
    f.write(reinterpret_cast<const char*>(t.ranges.data()),
            (std::streamsize)(t.ranges.size() * sizeof(uint16_t)));
    if (!f) throw io_error("write failed for " + path);
}

ClipTable read_clip_table(const std::string& path) {
    std::ifstream f(path, std::ios::binary);
    if (!f) throw io_error("cannot open " + path);
    magic(f, "BPCT", path);
    const uint32_t l = get<uint32_t>(f, "L", path), n = get<uint32_t>(f, "count", path);
    if (l < 1 || l > 65535 || n < 1) throw io_error("implausible clip table header in " + path, 4);
    ClipTable t;
    t.L = (int)l;
    t.n_views = (int)n;
    t.ranges.resize((size_t)2 * n * l * l);
    read_exact(f, reinterpret_cast<char*>(t.ranges.data()),
               (std::streamsize)(t.ranges.size() * sizeof(uint16_t)), "clip table", path);
    return t;
}

double psnr(const float* v, const float* ref, size_t n, double peak) {
    double mse = 0.0;
    for (size_t i = 0; i < n; ++i) {
        const double d = (double)v[i] - (double)ref[i];
        mse += d * d;
    }
    mse /= (double)n;
    if (peak <= 0.0) {
        float m = 0.0f;
        for (size_t i = 0; i < n; ++i) m = std::max(m, ref[i]);
        peak = m;
    }
    if (mse == 0.0) return INFINITY;
    return 10.0 * std::log10(peak * peak / mse);
}

}  // namespace bph
