// bp_capi.cpp -- extern "C" surface: include/backproject.h (reference-compatible)
// and include/bp_gpu.h (streaming module ABI).
//
// Error behaviour follows proj/src/capi.cpp:18-39: exceptions never cross the
// ABI; config_error -> BP_EINVAL, io_error -> BP_EIO, validation_error ->
// BP_EVERIFY, everything else (CUDA failures included) -> BP_EINTERNAL, with a
// thread-local message in bp_last_error().
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <list>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <thread>
#include <tuple>
#include <vector>

#include "../../include/backproject.h"
#include "../../include/bp_gpu.h"
#include "bp_host.hpp"
#include "bp_runtime.hpp"

namespace {

thread_local std::string g_last_error;

int fail(int code, const std::string& msg) {
    g_last_error = msg;
    return code;
}

template <typename Fn>
int guarded(Fn&& fn) {
    try {
        fn();
        return BP_OK;
    } catch (const bph::config_error& e) {
        return fail(BP_EINVAL, e.what());
    } catch (const bph::io_error& e) {
        return fail(BP_EIO, e.what());
    } catch (const bph::validation_error& e) {
        return fail(BP_EVERIFY, e.what());
    } catch (const std::exception& e) {
        return fail(BP_EINTERNAL, e.what());
    }
}

// ---- persistent device contexts ("loaded module") -------------------------
// bp_reconstruct keeps one SlabContext per (device, geometry, slab, options)
// alive between calls so that repeated reconstructions pay neither cudaMalloc
// of the volume / projection ring nor stream creation.
using CtxKey = std::tuple<int, uint32_t, uint32_t, uint32_t, double, double, double, int, int, int,
                          int, int, int, int, int, int, int, double, double, double, int>;

// Idle contexts, most recently released first.  Bounded by entry count and by the
// device memory they hold (BP_CTX_CACHE_MB, default 16 GiB), least recently used
// evicted first; an allocation failure in acquire() drains the cache and retries
// once; bp_gpu_release_cache() drains it on request.
struct CtxCache {
    std::mutex mu;
    std::list<std::pair<CtxKey, std::unique_ptr<bpr::SlabContext>>> idle;
    size_t bytes = 0;
};
CtxCache& cache() {
    static CtxCache* c = new CtxCache();
    return *c;
}
constexpr size_t kCacheEntries = 8;
size_t cache_cap_bytes() {
    static const size_t cap = [] {
        size_t mb = (size_t)16 << 10;
        if (const char* e = std::getenv("BP_CTX_CACHE_MB")) mb = (size_t)std::max(0L, std::atol(e));
        return mb << 20;
    }();
    return cap;
}

CtxKey key_of(const bp_gpu_config& c) {
    return CtxKey{c.device,        c.l,           c.isx,         c.isy,        c.offset_mm[0],
                  c.offset_mm[1],  c.offset_mm[2], c.z_begin,     c.z_end,      c.view_batch,
                  c.strict_mode,   c.distance_weight, c.row_windows, c.kernel, c.count_visible,
                  c.recip_mode,    c.filter,      c.sid_mm,      c.sdd_mm,     c.pitch_mm,
                  c.views};
}

// Removes every idle context (of `device`, or all when device < 0); the contexts are
// destroyed after the lock is dropped.
void drain_cache(int device) {
    std::vector<std::unique_ptr<bpr::SlabContext>> dead;
    {
        auto& C = cache();
        std::lock_guard<std::mutex> g(C.mu);
        for (auto it = C.idle.begin(); it != C.idle.end();) {
            if (device < 0 || it->second->device() == device) {
                C.bytes -= it->second->device_bytes();
                dead.push_back(std::move(it->second));
                it = C.idle.erase(it);
            } else {
                ++it;
            }
        }
    }
}

std::unique_ptr<bpr::SlabContext> acquire(const bp_gpu_config& c) {
    {
        auto& C = cache();
        std::lock_guard<std::mutex> g(C.mu);
        const CtxKey k = key_of(c);
        for (auto it = C.idle.begin(); it != C.idle.end(); ++it)
            if (it->first == k) {
                auto p = std::move(it->second);
                C.bytes -= p->device_bytes();
                C.idle.erase(it);
                return p;
            }
    }
    try {
        return std::make_unique<bpr::SlabContext>(c);
    } catch (const bph::device_error&) {
        // possibly out of device memory because of idle contexts: drop them, retry once
        drain_cache(-1);
        return std::make_unique<bpr::SlabContext>(c);
    }
}

void release(std::unique_ptr<bpr::SlabContext> p) {
    std::vector<std::unique_ptr<bpr::SlabContext>> dead;
    {
        auto& C = cache();
        std::lock_guard<std::mutex> g(C.mu);
        const size_t b = p->device_bytes();
        if (b > cache_cap_bytes()) return;  // too large to keep idle (destroyed on return)
        C.bytes += b;
        C.idle.emplace_front(key_of(p->config()), std::move(p));
        while (C.idle.size() > kCacheEntries || C.bytes > cache_cap_bytes()) {
            C.bytes -= C.idle.back().second->device_bytes();
            dead.push_back(std::move(C.idle.back().second));
            C.idle.pop_back();
        }
    }
}

std::mutex g_dev_mu;
std::vector<int> g_devices = {0};

}  // namespace

struct bp_stack {
    bph::Stack s;
};
struct bp_volume {
    bph::Volume v;
};
struct bp_gpu_ctx {
    std::unique_ptr<bpr::SlabContext> c;
};
struct bp_machine {
    int unused;
};

extern "C" {

const char* bp_last_error(void) { return g_last_error.c_str(); }

const char* bp_build_info(void) {
    return "paper_1104_5243_b200 libbackproject: sm_100a tiled TMA backprojection "
           "(packed FP32x2, strict/fast), built " __DATE__ " " __TIME__;
}

// ---- stacks ---------------------------------------------------------------

int bp_stack_generate(const bp_gen_params* p, bp_stack** out) {
    if (!p || !out) return fail(BP_EINVAL, "null argument");
    return guarded([&] {
        const double sid = p->sid_mm > 0 ? p->sid_mm : 750.0;
        const double sdd = p->sdd_mm > 0 ? p->sdd_mm : 1200.0;
        const double pitch = p->pitch_mm > 0 ? p->pitch_mm : 0.32;
        const auto ph = bph::named_phantom(p->phantom ? p->phantom : "spheres3");
        auto mats = bph::circular_trajectory(p->n_views, sid, sdd, p->isx, p->isy, pitch);
        auto st = std::make_unique<bp_stack>();
        st->s.isx = p->isx;
        st->s.isy = p->isy;
        st->s.mats = std::move(mats);
        st->s.pixels = bph::PinnedArray<float>((size_t)p->n_views * p->isx * p->isy);
        const int n = p->n_views;
        const int T = std::max(1, std::min<int>(n, (int)std::thread::hardware_concurrency()));
        std::vector<std::thread> th;
        for (int t = 0; t < T; ++t)
            th.emplace_back([&, t] {
                for (int k = t; k < n; k += T)
                    bph::forward_project(ph, st->s.mats[(size_t)k], p->isx, p->isy, st->s.image(k));
            });
        for (auto& x : th) x.join();
        *out = st.release();
    });
}

int bp_stack_read(const char* path, bp_stack** out) {
    if (!path || !out) return fail(BP_EINVAL, "null argument");
    return guarded([&] { *out = new bp_stack{bph::read_stack(path)}; });
}

int bp_stack_write(const bp_stack* s, const char* path) {
    if (!s || !path) return fail(BP_EINVAL, "null argument");
    return guarded([&] { bph::write_stack(path, s->s); });
}

void bp_stack_dims(const bp_stack* s, uint32_t* isx, uint32_t* isy, uint32_t* count) {
    if (!s) return;
    if (isx) *isx = (uint32_t)s->s.isx;
    if (isy) *isy = (uint32_t)s->s.isy;
    if (count) *count = (uint32_t)s->s.count();
}

void bp_stack_free(bp_stack* s) { delete s; }

int bp_stack_create(uint32_t isx, uint32_t isy, uint32_t count, const double* matrices,
                    const float* pixels, bp_stack** out) {
    if (!out) return fail(BP_EINVAL, "null argument");
    return guarded([&] {
        if (isx < 2 || isy < 2) throw bph::config_error("detector must be at least 2x2 pixels");
        if (count < 1) throw bph::config_error("need at least one view");
        auto st = std::make_unique<bp_stack>();
        st->s.isx = (int)isx;
        st->s.isy = (int)isy;
        st->s.mats.resize(count);
        if (matrices)
            for (uint32_t k = 0; k < count; ++k)
                std::memcpy(st->s.mats[k].data(), matrices + 12 * (size_t)k, 12 * sizeof(double));
        st->s.pixels = bph::PinnedArray<float>((size_t)count * isx * isy);
        if (pixels)
            std::memcpy(st->s.pixels.data(), pixels, (size_t)count * isx * isy * sizeof(float));
        else
            std::memset(st->s.pixels.data(), 0, (size_t)count * isx * isy * sizeof(float));
        *out = st.release();
    });
}

float* bp_stack_pixels(bp_stack* s) { return s ? s->s.pixels.data() : nullptr; }
double* bp_stack_matrices(bp_stack* s) {
    return s && !s->s.mats.empty() ? s->s.mats[0].data() : nullptr;
}

void bp_baseline_params_init(bp_baseline_params* p) {
    if (!p) return;
    bph::BaselineSpec d;
    p->seed = d.seed;
    p->n_views = d.n_views;
    p->isx = d.isx;
    p->isy = d.isy;
    p->sid_mm = d.sid;
    p->sdd_mm = d.sdd;
    p->pitch_mm = d.pitch;
    p->arc_deg = d.arc_deg;
    p->jitter_mm = d.jitter_mm;
    p->jitter_deg = d.jitter_deg;
    p->n_ellipsoids = d.n_ellipsoids;
    p->filter = d.filter;
    p->threads = d.threads;
}

static bph::BaselineSpec spec_of(const bp_baseline_params* p) {
    bph::BaselineSpec s;
    s.seed = p->seed;
    s.n_views = p->n_views;
    s.isx = p->isx;
    s.isy = p->isy;
    s.sid = p->sid_mm;
    s.sdd = p->sdd_mm;
    s.pitch = p->pitch_mm;
    s.arc_deg = p->arc_deg;
    s.jitter_mm = p->jitter_mm;
    s.jitter_deg = p->jitter_deg;
    s.n_ellipsoids = p->n_ellipsoids;
    s.filter = p->filter;
    s.threads = p->threads;
    return s;
}

int bp_stack_generate_baseline(const bp_baseline_params* p, bp_stack** out) {
    if (!p || !out) return fail(BP_EINVAL, "null argument");
    return guarded([&] { *out = new bp_stack{bph::make_baseline_stack(spec_of(p))}; });
}

int bp_baseline_phantom(const bp_baseline_params* p, double* ell, int max_n, int* n) {
    if (!p || !n) return fail(BP_EINVAL, "null argument");
    return guarded([&] {
        const auto e = bph::baseline_phantom(spec_of(p));
        *n = (int)e.size();
        for (int i = 0; i < std::min<int>(max_n, (int)e.size()); ++i) {
            const auto& x = e[(size_t)i];
            const double v[7] = {x.cx, x.cy, x.cz, x.ax, x.ay, x.az, x.density};
            std::memcpy(ell + 7 * i, v, sizeof v);
        }
    });
}

// ---- volumes --------------------------------------------------------------

int bp_volume_read(const char* path, bp_volume** out) {
    if (!path || !out) return fail(BP_EINVAL, "null argument");
    return guarded([&] { *out = new bp_volume{bph::read_volume(path)}; });
}

int bp_volume_write(const bp_volume* v, const char* path) {
    if (!v || !path) return fail(BP_EINVAL, "null argument");
    return guarded([&] { bph::write_volume(path, v->v); });
}

uint32_t bp_volume_edge(const bp_volume* v) { return v ? (uint32_t)v->v.grid.L : 0; }
const float* bp_volume_data(const bp_volume* v) { return v ? v->v.vox.data() : nullptr; }
float* bp_volume_data_mut(bp_volume* v) { return v ? v->v.vox.data() : nullptr; }
void bp_volume_free(bp_volume* v) { delete v; }

int bp_volume_create(uint32_t l, bp_volume** out) {
    if (!out) return fail(BP_EINVAL, "null argument");
    return guarded([&] {
        auto v = std::make_unique<bp_volume>(bp_volume{bph::Volume(bph::Grid::cube((int)l))});
        std::memset(v->v.vox.data(), 0, v->v.vox.size() * sizeof(float));
        *out = v.release();
    });
}

int bp_psnr(const bp_volume* vol, const bp_volume* ref, double peak, double* out_db) {
    if (!vol || !ref || !out_db) return fail(BP_EINVAL, "null argument");
    return guarded([&] {
        if (vol->v.grid.L != ref->v.grid.L) throw bph::validation_error("volume dimensions differ");
        *out_db = bph::psnr(vol->v.vox.data(), ref->v.vox.data(), vol->v.vox.size(), peak);
    });
}

// ---- streaming module ABI -----------------------------------------------------

void bp_gpu_config_init(bp_gpu_config* c) {
    if (!c) return;
    std::memset(c, 0, sizeof *c);
    c->device = -1;
    c->view_batch = 0;    /* library default: 32; 62 for whole volumes of 1024^3 or more */
    c->ring_batches = 0;  /* library default: 8 batches (tail deferral needs >= 8) */
    c->strict_mode = 1;
    c->distance_weight = 1;
    c->row_windows = 1;
    c->tail_batches = -1;
}

int bp_gpu_load(const bp_gpu_config* cfg, bp_gpu_ctx** out) {
    if (!cfg || !out) return fail(BP_EINVAL, "null argument");
    return guarded([&] {
        if (cfg->recip_mode < BP_RECIP_EXACT || cfg->recip_mode > BP_RECIP_HW_APPROX)
            throw bph::config_error("recip_mode out of range");
        auto c = std::make_unique<bp_gpu_ctx>();
        c->c = std::make_unique<bpr::SlabContext>(*cfg);
        *out = c.release();
    });
}

int bp_gpu_backproject(bp_gpu_ctx* ctx, const float* image, const double matrix[12]) {
    if (!ctx || !image || !matrix) return fail(BP_EINVAL, "null argument");
    return guarded([&] { ctx->c->backproject(image, matrix, true); });
}

int bp_gpu_backproject_async(bp_gpu_ctx* ctx, const float* image, const double matrix[12]) {
    if (!ctx || !image || !matrix) return fail(BP_EINVAL, "null argument");
    return guarded([&] { ctx->c->backproject(image, matrix, false); });
}

int bp_gpu_finish(bp_gpu_ctx* ctx, float* host_volume, bp_gpu_stats* stats) {
    if (!ctx) return fail(BP_EINVAL, "null argument");
    return guarded([&] { ctx->c->finish(host_volume, stats); });
}

int bp_gpu_unload(bp_gpu_ctx* ctx) {
    if (!ctx) return fail(BP_EINVAL, "null argument");
    return guarded([&] { delete ctx; });
}

int bp_gpu_release_cache(void) {
    return guarded([&] { drain_cache(-1); });
}

int bp_gpu_volume_device(bp_gpu_ctx* ctx, float** dptr, int* z_begin, int* z_end) {
    if (!ctx) return fail(BP_EINVAL, "null argument");
    if (dptr) *dptr = ctx->c->device_volume();
    if (z_begin) *z_begin = ctx->c->z_begin();
    if (z_end) *z_end = ctx->c->z_end();
    return BP_OK;
}

int bp_gpu_read_lines(bp_gpu_ctx* ctx, const int* ys, const int* zs, int n, float* out) {
    if (!ctx) return fail(BP_EINVAL, "null argument");
    return guarded([&] { ctx->c->read_lines(ys, zs, n, out); });
}

int bp_gpu_clip_table(const bp_stack* s, uint32_t l, const double offset_mm[3], uint16_t* ranges,
                      uint64_t* total) {
    if (!s) return fail(BP_EINVAL, "null argument");
    return guarded([&] {
        if (s->s.count() < 1) throw bph::validation_error("empty projection stack");
        bp_gpu_config c;
        bp_gpu_config_init(&c);
        c.l = l;
        c.isx = (uint32_t)s->s.isx;
        c.isy = (uint32_t)s->s.isy;
        for (int i = 0; i < 3; ++i) c.offset_mm[i] = offset_mm ? offset_mm[i] : 0.0;
        c.view_batch = 1;
        c.ring_batches = 1;
        bpr::SlabContext ctx(c);
        ctx.clip_table(s->s.mats[0].data(), s->s.count(), ranges, total);
    });
}

int bp_clip_table_read(const char* path, uint32_t* l, uint32_t* count, uint16_t* ranges,
                       uint64_t* total) {
    if (!path) return fail(BP_EINVAL, "null argument");
    return guarded([&] {
        const auto t = bph::read_clip_table(path);
        if (l) *l = (uint32_t)t.L;
        if (count) *count = (uint32_t)t.n_views;
        if (ranges) std::memcpy(ranges, t.ranges.data(), t.ranges.size() * sizeof(uint16_t));
        if (total) *total = t.total_updates();
    });
}

int bp_clip_table_write(const char* path, uint32_t l, uint32_t count, const uint16_t* ranges) {
    if (!path || !ranges) return fail(BP_EINVAL, "null argument");
    return guarded([&] {
        if (l < 1 || l > 65535 || count < 1) throw bph::config_error("clip table dimensions out of range");
        bph::ClipTable t;
        t.L = (int)l;
        t.n_views = (int)count;
        t.ranges.assign(ranges, ranges + (size_t)2 * count * l * l);
        bph::write_clip_table(path, t);
    });
}

int bp_gpu_filter_views(const float* in, float* out, int count, uint32_t isx, uint32_t isy,
                        double sid_mm, double sdd_mm, double pitch_mm, int device) {
    if (!in || !out || count < 1) return fail(BP_EINVAL, "null argument");
    return guarded([&] {
        if (isx < 2 || isy < 2) throw bph::config_error("detector must be at least 2x2 pixels");
        int ndev = 0;
        if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev < 1) {
            cudaGetLastError();
            throw bph::device_error("no CUDA device available (the GPU path has no CPU fallback)");
        }
        if (device >= ndev) throw bph::config_error("device ordinal out of range");
        if (device >= 0) bpr::check(cudaSetDevice(device), "cudaSetDevice");
        bpr::RampFilter f((int)isx, (int)isy, sid_mm, sdd_mm, pitch_mm);
        const size_t img = (size_t)isx * isy;
        const int chunk = (int)std::max<size_t>(1, std::min<size_t>((size_t)count, ((size_t)256 << 20) / (img * 4)));
        float* d = nullptr;
        bpr::check(cudaMalloc(&d, (size_t)chunk * img * sizeof(float)), "cudaMalloc(filter views)");
        std::unique_ptr<float, decltype(&cudaFree)> hold(d, &cudaFree);
        for (int k0 = 0; k0 < count; k0 += chunk) {
            const int n = std::min(chunk, count - k0);
            bpr::check(cudaMemcpy(d, in + (size_t)k0 * img, (size_t)n * img * sizeof(float),
                                  cudaMemcpyHostToDevice), "H2D");
            f.apply(d, (long long)img, (int)isx, n, 0, (int)isy, nullptr);
            bpr::check(cudaMemcpy(out + (size_t)k0 * img, d, (size_t)n * img * sizeof(float),
                                  cudaMemcpyDeviceToHost), "D2H");
        }
    });
}

int bp_ipc_handle(const void* device_ptr, unsigned char handle[64], uint64_t* offset) {
    if (!device_ptr || !handle) return fail(BP_EINVAL, "null argument");
    return guarded([&] {
        // IPC maps whole allocations: report where device_ptr sits inside its allocation
        // (a caching allocator may hand out sub-ranges), via cuMemGetAddressRange
        using RangeFn = CUresult (*)(CUdeviceptr*, size_t*, CUdeviceptr);
        static RangeFn range = nullptr;
        if (!range) {
            void* fp = nullptr;
            cudaDriverEntryPointQueryResult q;
            if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &fp, cudaEnableDefault, &q) !=
                    cudaSuccess ||
                q != cudaDriverEntryPointSuccess)
                throw bph::device_error("cuMemGetAddressRange entry point unavailable");
            range = reinterpret_cast<RangeFn>(fp);
        }
        CUdeviceptr base = 0;
        size_t size = 0;
        if (range(&base, &size, reinterpret_cast<CUdeviceptr>(device_ptr)) != CUDA_SUCCESS)
            throw bph::device_error("cuMemGetAddressRange failed (not a device allocation?)");
        cudaIpcMemHandle_t h;
        bpr::check(cudaIpcGetMemHandle(&h, reinterpret_cast<void*>(base)), "cudaIpcGetMemHandle");
        static_assert(sizeof h == 64, "CUDA IPC handles are 64 bytes");
        std::memcpy(handle, &h, sizeof h);
        if (offset) *offset = (uint64_t)(reinterpret_cast<CUdeviceptr>(device_ptr) - base);
    });
}

int bp_ipc_open(const unsigned char handle[64], void** device_ptr) {
    if (!handle || !device_ptr) return fail(BP_EINVAL, "null argument");
    return guarded([&] {
        cudaIpcMemHandle_t h;
        std::memcpy(&h, handle, sizeof h);
        void* p = nullptr;
        bpr::check(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess), "cudaIpcOpenMemHandle");
        *device_ptr = p;
    });
}

int bp_ipc_close(void* device_ptr) {
    if (!device_ptr) return fail(BP_EINVAL, "null argument");
    return guarded([&] { bpr::check(cudaIpcCloseMemHandle(device_ptr), "cudaIpcCloseMemHandle"); });
}

int bp_device_compare(const float* d_a, const float* d_b, uint64_t n, double* max_abs_diff,
                      double* max_abs_ref, double* sum_sq_diff, uint64_t* n_bit_diff) {
    if (!d_a || !d_b) return fail(BP_EINVAL, "null argument");
    return guarded([&] {
        double r[3];
        unsigned long long nb = 0;
        bpr::check((cudaError_t)bpg::device_compare(d_a, d_b, n, r, &nb), "device compare");
        if (max_abs_diff) *max_abs_diff = r[0];
        if (max_abs_ref) *max_abs_ref = r[1];
        if (sum_sq_diff) *sum_sq_diff = r[2];
        if (n_bit_diff) *n_bit_diff = nb;
    });
}

int bp_gpu_upload_views(bp_gpu_ctx* ctx, const float* pixels, const double* matrices, int count) {
    if (!ctx || !pixels || !matrices) return fail(BP_EINVAL, "null argument");
    return guarded([&] { ctx->c->upload_views(pixels, matrices, count); });
}

int bp_gpu_time_resident(bp_gpu_ctx* ctx, int iters, double* device_ms, bp_gpu_stats* stats) {
    if (!ctx) return fail(BP_EINVAL, "null argument");
    return guarded([&] {
        const double ms = ctx->c->time_resident(iters, stats);
        if (device_ms) *device_ms = ms;
    });
}

// ---- multi-GPU / partition -----------------------------------------------------

int bp_gpu_set_devices(const int* devices, int n) {
    if (!devices || n < 1) return fail(BP_EINVAL, "need at least one device");
    std::lock_guard<std::mutex> g(g_dev_mu);
    g_devices.assign(devices, devices + n);
    return BP_OK;
}

int bp_gpu_device_count(int* n) {
    if (!n) return fail(BP_EINVAL, "null argument");
    int c = 0;
    if (cudaGetDeviceCount(&c) != cudaSuccess) {
        cudaGetLastError();
        c = 0;
    }
    *n = c;
    return BP_OK;
}

int bp_partition_slabs(const double* matrices, int count, uint32_t isx, uint32_t isy, uint32_t l,
                       const double offset_mm[3], int G, int* bounds) {
    if (!matrices || !bounds || count < 1) return fail(BP_EINVAL, "null argument");
    return guarded([&] {
        std::vector<bph::Mat> m((size_t)count);
        for (int k = 0; k < count; ++k) std::memcpy(m[(size_t)k].data(), matrices + 12 * k, 96);
        const double* o = offset_mm;
        auto g = bph::Grid::cube((int)l, o ? o[0] : 0, o ? o[1] : 0, o ? o[2] : 0);
        auto b = bph::partition_slabs(m, (int)isx, (int)isy, g, G);
        std::copy(b.begin(), b.end(), bounds);
    });
}

int bp_slab_work(const double* matrices, int count, uint32_t isx, uint32_t isy, uint32_t l,
                 const double offset_mm[3], double* work) {
    if (!matrices || !work || count < 1) return fail(BP_EINVAL, "null argument");
    return guarded([&] {
        std::vector<bph::Mat> m((size_t)count);
        for (int k = 0; k < count; ++k) std::memcpy(m[(size_t)k].data(), matrices + 12 * k, 96);
        const double* o = offset_mm;
        auto g = bph::Grid::cube((int)l, o ? o[0] : 0, o ? o[1] : 0, o ? o[2] : 0);
        std::vector<double> w;
        bph::partition_slabs(m, (int)isx, (int)isy, g, 1, &w);
        std::copy(w.begin(), w.end(), work);
    });
}

int bp_partition_by_cost(const double* slice_cost, uint32_t l, int G, int align, int* bounds) {
    if (!slice_cost || !bounds) return fail(BP_EINVAL, "null argument");
    return guarded([&] {
        std::vector<double> c(slice_cost, slice_cost + l);
        auto b = bph::partition_by_cost(c, G, align);
        std::copy(b.begin(), b.end(), bounds);
    });
}

int bp_slab_row_window(const double matrix[12], uint32_t isy, uint32_t l, const double offset_mm[3],
                       int z_begin, int z_end, int* r0, int* r1) {
    if (!matrix || !r0 || !r1) return fail(BP_EINVAL, "null argument");
    return guarded([&] {
        const double* o = offset_mm;
        auto g = bph::Grid::cube((int)l, o ? o[0] : 0, o ? o[1] : 0, o ? o[2] : 0);
        if (z_begin < 0 || z_end > (int)l || z_begin >= z_end)
            throw bph::config_error("slab out of range");
        bph::Mat m;
        std::memcpy(m.data(), matrix, 96);
        bph::row_window(m, g, 0, (int)l - 1, 0, (int)l - 1, z_begin, z_end - 1, (int)isy, r0, r1);
    });
}

void bp_recon_ex_init(bp_recon_ex* p) {
    if (!p) return;
    std::memset(p, 0, sizeof *p);
    p->view_batch = 0;  /* library default (bp_gpu_config.view_batch) */
    p->strict_mode = 1;
    p->distance_weight = 1;
    p->row_windows = 1;
}

int bp_reconstruct_ex(const bp_stack* s, uint32_t l, const bp_recon_ex* p, float* host_volume,
                      bp_gpu_stats* stats) {
    if (!s || !p || !host_volume) return fail(BP_EINVAL, "null argument");
    return guarded([&] {
        if (l < 1) throw bph::config_error("grid edge must be >= 1 voxel");
        if (s->s.count() < 1) throw bph::validation_error("empty projection stack");
        std::vector<int> devs;
        {
            std::lock_guard<std::mutex> g(g_dev_mu);
            devs = g_devices;
        }
        if (p->n_devices > 0) devs.resize(std::min<size_t>(devs.size(), (size_t)p->n_devices));
        if (p->n_devices > (int)devs.size())
            for (int d = (int)devs.size(); d < p->n_devices; ++d) devs.push_back(d);
        const int D = (int)devs.size();
        const int G = std::max(D, p->virtual_slabs);
        const double off[3] = {p->offset_mm ? p->offset_mm[0] : 0.0,
                               p->offset_mm ? p->offset_mm[1] : 0.0,
                               p->offset_mm ? p->offset_mm[2] : 0.0};
        const auto grid = bph::Grid::cube((int)l, off[0], off[1], off[2]);
        // reference: every matrix is validated before any work (scheduler.cpp:35)
        for (const auto& m : s->s.mats) bph::validate_matrix_for_grid(m, grid);
        std::vector<int> bounds = {0, (int)l};
        if (G > 1) bounds = bph::partition_slabs(s->s.mats, s->s.isx, s->s.isy, grid, G);
        std::vector<bp_gpu_stats> per((size_t)G);
        std::vector<std::string> errs((size_t)D);
        std::vector<int> codes((size_t)D, BP_OK);
        auto worker = [&](int d) {
            codes[(size_t)d] = guarded([&] {
                for (int g = d; g < G; g += D) {
                    bp_gpu_config c;
                    bp_gpu_config_init(&c);
                    c.l = l;
                    c.isx = (uint32_t)s->s.isx;
                    c.isy = (uint32_t)s->s.isy;
                    std::memcpy(c.offset_mm, off, sizeof off);
                    c.device = devs[(size_t)d];
                    c.z_begin = bounds[(size_t)g];
                    c.z_end = bounds[(size_t)g + 1];
                    c.view_batch = p->view_batch > 0 ? p->view_batch : 0;
                    c.strict_mode = p->strict_mode;
                    c.distance_weight = p->distance_weight;
                    c.row_windows = p->row_windows;
                    c.kernel = p->kernel;
                    c.count_visible = p->count_visible;
                    c.recip_mode = p->recip_mode;
                    c.filter = p->filter;
                    c.sid_mm = p->sid_mm;
                    c.sdd_mm = p->sdd_mm;
                    c.pitch_mm = p->pitch_mm;
                    c.views = s->s.count();  // the whole stack is at hand: band-ordered tail
                    auto ctx = acquire(c);
                    for (int k = 0; k < s->s.count(); ++k)
                        ctx->backproject(s->s.image(k), s->s.mats[(size_t)k].data(), false);
                    ctx->finish(host_volume + (size_t)c.z_begin * l * l, &per[(size_t)g]);
                    release(std::move(ctx));
                }
            });
            if (codes[(size_t)d] != BP_OK) errs[(size_t)d] = g_last_error;
        };
        if (D == 1) {
            worker(0);
        } else {
            std::vector<std::thread> th;
            for (int d = 0; d < D; ++d) th.emplace_back(worker, d);
            for (auto& t : th) t.join();
        }
        for (int d = 0; d < D; ++d)
            if (codes[(size_t)d] != BP_OK) {
                const int c = codes[(size_t)d];
                const std::string m = "device " + std::to_string(devs[(size_t)d]) + ": " + errs[(size_t)d];
                if (c == BP_EINVAL) throw bph::config_error(m);
                if (c == BP_EVERIFY) throw bph::validation_error(m);
                if (c == BP_EIO) throw bph::io_error(m);
                throw bph::device_error(m);
            }
        if (stats) {
            bp_gpu_stats t{};
            for (const auto& x : per) {
                t.wall_ms = std::max(t.wall_ms, x.wall_ms);
                t.device_ms = std::max(t.device_ms, x.device_ms);
                t.kernel_ms += x.kernel_ms;
                t.h2d_ms = std::max(t.h2d_ms, x.h2d_ms);
                t.d2h_ms = std::max(t.d2h_ms, x.d2h_ms);
                t.views = x.views;
                t.launches += x.launches;
                t.prep_launches += x.prep_launches;
                t.nominal_updates += x.nominal_updates;
                t.visible_updates += x.visible_updates;
                t.tile_pairs += x.tile_pairs;
                t.skipped_pairs += x.skipped_pairs;
                t.fallback_pairs += x.fallback_pairs;
                t.h2d_bytes += x.h2d_bytes;
                t.d2h_bytes += x.d2h_bytes;
                t.tile_w = std::max(t.tile_w, x.tile_w);
                t.tile_h = std::max(t.tile_h, x.tile_h);
                t.block_x = x.block_x;
                t.block_y = x.block_y;
                t.block_z = x.block_z;
            }
            std::vector<uint64_t> dev((size_t)D, 0);
            for (int g = 0; g < G; ++g)
                dev[(size_t)(g % D)] += p->count_visible ? per[(size_t)g].visible_updates
                                                         : per[(size_t)g].nominal_updates;
            t.device_updates_min = *std::min_element(dev.begin(), dev.end());
            t.device_updates_max = *std::max_element(dev.begin(), dev.end());
            *stats = t;
        }
    });
}

// ---- reference one-shot entry point ------------------------------------------------

int bp_reconstruct(const bp_stack* s, const bp_recon_params* p, bp_volume** out,
                   bp_recon_stats* stats) {
    if (!s || !p || !out) return fail(BP_EINVAL, "null argument");
    return guarded([&] {
        // parameter mapping and validation of capi.cpp:113-130 / scheduler.cpp:31-34
        if (p->recip_mode < BP_RECIP_EXACT || p->recip_mode > BP_RECIP_APPROX12_NR)
            throw bph::config_error("recip_mode out of range");
        if (p->extract != BP_EXTRACT_V1_STORE && p->extract != BP_EXTRACT_V2_SHIFT)
            throw bph::config_error("extract out of range");
        const int threads = p->threads;
        const int chunk = p->chunk > 0 ? p->chunk : 1;
        const int block_b = p->block_b > 0 ? p->block_b : 32;
        const int lanes = p->lanes > 0 ? p->lanes : 1;
        const int numa = p->numa_domains > 0 ? p->numa_domains : 1;
        auto grid = bph::Grid::cube((int)p->l);
        if (s->s.count() < 1) throw bph::validation_error("empty projection stack");
        if (threads < 1 || chunk < 1 || block_b < 1 || numa < 1)
            throw bph::config_error("threads, chunk, block_b and numa_domains must be >= 1");
        if (lanes != 1 && lanes != 4 && lanes != 8)
            throw bph::config_error("lane width must be 1, 4 or 8");
        // block_b is the register batch (views per launch). Any value is accepted like
        // the reference's; beyond the kernel's parameter-space batch it is clamped,
        // which cannot change results (ascending view order per voxel is invariant)
        const int gpu_b = std::min(block_b, bpg::kMaxBatch);

        auto vol = std::make_unique<bp_volume>(bp_volume{bph::Volume(grid)});
        bp_recon_ex ex;
        bp_recon_ex_init(&ex);
        ex.view_batch = gpu_b;
        ex.strict_mode = p->strict_mode != 0 ? 1 : 0;
        ex.distance_weight = p->distance_weight != 0 ? 1 : 0;
        ex.count_visible = p->clip != 0 ? 1 : 0;
        ex.recip_mode = p->recip_mode;
        // clip cache (capi.cpp:133-143): read the BPCT table if it exists, else build
        // it (exactly, on the GPU) and write it.  The GPU clips on the fly; the table
        // supplies the clip_stats the reference reports.
        bool have_table = false;
        uint64_t table_total = 0;
        // every matrix against the grid first (w > 0 at the 8 corners, geometry.cpp:130-144):
        // BP_EVERIFY before any clip-table work, as the reference's validation precedes its
        // precompute (scheduler.cpp:31-35)
        for (const auto& m : s->s.mats) bph::validate_matrix_for_grid(m, grid);
        if (p->clip && p->clip_cache) {
            std::ifstream probe(p->clip_cache, std::ios::binary);
            if (probe.good()) {
                probe.close();
                auto t = bph::read_clip_table(p->clip_cache);
                if (t.L != (int)p->l || t.n_views != s->s.count())
                    throw bph::validation_error("clip table does not match grid/stack dimensions");
                table_total = t.total_updates();
            } else {
                bph::ClipTable t;
                t.L = (int)p->l;
                t.n_views = s->s.count();
                t.ranges.resize((size_t)2 * t.n_views * p->l * p->l);
                const int rc = bp_gpu_clip_table(s, p->l, nullptr, t.ranges.data(), &table_total);
                if (rc != BP_OK) {
                    const std::string m = g_last_error;
                    if (rc == BP_EINVAL) throw bph::config_error(m);
                    if (rc == BP_EVERIFY) throw bph::validation_error(m);
                    if (rc == BP_EIO) throw bph::io_error(m);
                    throw bph::device_error(m);
                }
                bph::write_clip_table(p->clip_cache, t);
            }
            have_table = true;
            ex.count_visible = 0;
        }
        bp_gpu_stats gs{};
        const double t0 = bpr::now_ms();
        const int rc = bp_reconstruct_ex(s, p->l, &ex, vol->v.vox.data(), &gs);
        if (have_table) gs.visible_updates = table_total;
        if (rc != BP_OK) {
            const std::string m = g_last_error;
            if (rc == BP_EINVAL) throw bph::config_error(m);
            if (rc == BP_EVERIFY) throw bph::validation_error(m);
            if (rc == BP_EIO) throw bph::io_error(m);
            throw bph::device_error(m);
        }
        const double secs = (bpr::now_ms() - t0) / 1e3;
        *out = vol.release();
        if (stats) {
            *stats = {};
            const uint64_t L3 = (uint64_t)p->l * p->l * p->l;
            const uint64_t n = (uint64_t)s->s.count();
            stats->seconds = secs;
            stats->voxel_updates = p->clip ? gs.visible_updates : n * L3;
            stats->gups = secs > 0 ? stats->voxel_updates / secs / 1e9 : 0.0;
            stats->gflops = secs > 0 ? 31.0 * stats->voxel_updates / secs / 1e9 : 0.0;
            stats->writeback_stores = (n + gpu_b - 1) / gpu_b * L3;
            stats->bytes_copied = gs.h2d_bytes;
            stats->clip_reduction = p->clip ? 1.0 - (double)gs.visible_updates / (double)(n * L3) : 0.0;
            // per-device split of the updates, the GPU analogue of the reference's
            // per-thread min/max (scheduler.hpp:22-30); a cached clip table gives only
            // the total, so the split is then unknown and the total is reported
            const bool split = !(p->clip && have_table);
            stats->thread_updates_min = split ? gs.device_updates_min : stats->voxel_updates;
            stats->thread_updates_max = split ? gs.device_updates_max : stats->voxel_updates;
        }
    });
}

int bp_selftest_rcp(uint32_t lo_bits, uint32_t hi_bits, uint64_t* mismatches) {
    if (!mismatches) return fail(BP_EINVAL, "null argument");
    return guarded([&] {
        unsigned long long m = 0;
        bpr::check((cudaError_t)bpg::selftest_rcp(lo_bits, hi_bits, &m), "rcp selftest");
        *mismatches = m;
    });
}

// ---- performance model: out of scope ------------------------------

static const char* kModelOut =
    "the analytic CPU performance model (proj/src/perfmodel.cpp) is out of scope of the B200 build";

int bp_machine_load(const char*, bp_machine** out) {
    if (out) *out = nullptr;
    return fail(BP_EINVAL, kModelOut);
}
void bp_machine_free(bp_machine* m) { delete m; }
int bp_model_report_build(const bp_machine*, bp_model_report*) { return fail(BP_EINVAL, kModelOut); }
int bp_machine_measure(bp_machine*, size_t, int, double) { return fail(BP_EINVAL, kModelOut); }
int bp_model_deviation(const bp_machine*, double, double*) { return fail(BP_EINVAL, kModelOut); }

}  // extern "C"
