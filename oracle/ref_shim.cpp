// ref_shim.cpp -- TEST INFRASTRUCTURE ONLY (see oracle/bp_oracle.c header).
//
// A thin extern "C" shim, compiled together with the reference's own sources
// where they lie under /root/reference/proj/src (oracle/Makefile), so that the
// Python tests and bench.py's reference arm can drive the UNMODIFIED reference
// internals through ctypes:
//   - bp::reconstruct with an arbitrary VoxelGrid offset (the C ABI
//     only takes L, config 5 needs offset_x += 60)   scheduler.cpp:24-133
//   - pad_image + line_update_scalar per sampled line  kernel.cpp:32-85
//   - build_clip_table / clip_stats                                    precompute.cpp:51-103
//   - make_circular_trajectory + make_stack for datagen pinning        geometry.cpp:86-128, datagen.cpp:80-108
//   - the BPCT clip-cache reader / writer (format interop tests)        precompute.cpp:105-134
// No reference source is copied; this file only calls it.
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>
#include <vector>

#include "datagen.hpp"
#include "geometry.hpp"
#include "kernel.hpp"
#include "precompute.hpp"
#include "scheduler.hpp"

namespace {
thread_local std::string g_err;

bp::ProjectionStack wrap(const float* pixels, const double* mats, int n, int isx, int isy) {
    bp::ProjectionStack s;
    s.isx = isx;
    s.isy = isy;
    s.matrices.resize(n);
    for (int k = 0; k < n; ++k) std::memcpy(s.matrices[k].a.data(), mats + 12 * k, 12 * sizeof(double));
    s.pixels.assign(pixels, pixels + (size_t)n * isx * isy);
    return s;
}

bp::VoxelGrid grid_of(int L, double dx, double dy, double dz) {
    auto g = bp::VoxelGrid::cube(L);
    g.offset_x += dx;
    g.offset_y += dy;
    g.offset_z += dz;
    return g;
}
}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

// stats_out[0]=seconds, [1]=voxel_updates, [2]=gups, [3]=writeback, [4]=bytes_copied, [5]=clip_reduction
int ref_reconstruct(const float* pixels, const double* mats, int n, int isx, int isy, int L,
                    double dx, double dy, double dz, int threads, int chunk, int block_b,
                    int lanes, int clip, int distance_weight, int recip, float* out,
                    double* stats_out) {
    try {
        auto s = wrap(pixels, mats, n, isx, isy);
        auto g = grid_of(L, dx, dy, dz);
        bp::RunConfig cfg;
        cfg.threads = threads;
        cfg.chunk = chunk;
        cfg.block_b = block_b;
        cfg.kernel.lanes = lanes;
        cfg.kernel.distance_weight = distance_weight != 0;
        cfg.kernel.recip = static_cast<bp::RecipMode>(recip);  // geometry.hpp:39
        cfg.clip = clip != 0;
        bp::RunStats st;
        auto vol = bp::reconstruct(s, g, cfg, &st);
        std::memcpy(out, vol.vox.data(), vol.vox.size() * sizeof(float));
        if (stats_out) {
            stats_out[0] = st.seconds;
            stats_out[1] = (double)st.voxel_updates;
            stats_out[2] = st.gups;
            stats_out[3] = (double)st.writeback_stores;
            stats_out[4] = (double)st.bytes_copied;
            stats_out[5] = st.clip_reduction;
        }
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}

// Sampled lines: out[i*L .. i*L+L) accumulates all views in ascending order.
int ref_reconstruct_lines(const float* pixels, const double* mats, int n, int isx, int isy, int L,
                          double dx, double dy, double dz, const int* ys, const int* zs,
                          int nlines, int distance_weight, float* out) {
    try {
        auto g = grid_of(L, dx, dy, dz);
        bp::KernelConfig kc;
        kc.distance_weight = distance_weight != 0;
        for (int k = 0; k < n; ++k) {
            bp::ProjectionMatrix M;
            std::memcpy(M.a.data(), mats + 12 * k, 12 * sizeof(double));
            auto A = M.narrowed();
            auto img = bp::pad_image(pixels + (size_t)k * isx * isy, isx, isy, 1);
            for (int i = 0; i < nlines; ++i)
                bp::line_update_scalar(out + (size_t)i * L, img, A.data(), g, ys[i], zs[i], 0,
                                       L - 1, kc);
        }
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}

// Clip table ranges (2*n*L*L u16) and total visible updates.
int ref_clip_table(const double* mats, int n, int isx, int isy, int L, double dx, double dy,
                   double dz, uint16_t* ranges, uint64_t* total) {
    try {
        auto g = grid_of(L, dx, dy, dz);
        std::vector<bp::ProjectionMatrix> ms(n);
        for (int k = 0; k < n; ++k) std::memcpy(ms[k].a.data(), mats + 12 * k, 12 * sizeof(double));
        auto t = bp::build_clip_table(g, ms, isx, isy);
        if (ranges) std::memcpy(ranges, t.ranges.data(), t.ranges.size() * sizeof(uint16_t));
        if (total) *total = bp::clip_stats(t).total_updates;
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}

// Reference datagen: circular trajectory + named phantom stack.
int ref_make_stack(const char* phantom, int n, int isx, int isy, double sid, double sdd,
                   double pitch, double* mats_out, float* pixels_out) {
    try {
        auto ph = bp::make_phantom(phantom);
        auto ms = bp::make_circular_trajectory(n, sid, sdd, isx, isy, pitch);
        auto s = bp::make_stack(ph, ms, isx, isy);
        for (int k = 0; k < n; ++k) std::memcpy(mats_out + 12 * k, ms[k].a.data(), 12 * sizeof(double));
        std::memcpy(pixels_out, s.pixels.data(), s.pixels.size() * sizeof(float));
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}

// Forward projection of an arbitrary ellipsoid phantom (e: n_ell*7 doubles
// cx,cy,cz,ax,ay,az,density) through one matrix.
int ref_forward_project(const double* ell, int n_ell, const double* mat, int isx, int isy,
                        float* out) {
    try {
        bp::Phantom ph;
        for (int i = 0; i < n_ell; ++i) {
            const double* e = ell + 7 * i;
            ph.ellipsoids.push_back({e[0], e[1], e[2], e[3], e[4], e[5], e[6]});
        }
        bp::ProjectionMatrix M;
        std::memcpy(M.a.data(), mat, 12 * sizeof(double));
        bp::forward_project(ph, M, isx, isy, out);
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}

// BPCT cache file through the reference's own reader: dims first (ranges may be NULL),
// then the ranges (2*n*L*L u16) and clip_stats total.
int ref_read_clip_table(const char* path, int* L, int* n, uint16_t* ranges, uint64_t* total) {
    try {
        auto t = bp::read_clip_table(path);
        if (L) *L = t.L;
        if (n) *n = t.n_views;
        if (ranges) std::memcpy(ranges, t.ranges.data(), t.ranges.size() * sizeof(uint16_t));
        if (total) *total = bp::clip_stats(t).total_updates;
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}

// ... and through the reference's own writer.
int ref_write_clip_table(const char* path, int L, int n, const uint16_t* ranges) {
    try {
        bp::ClipTable t;
        t.L = L;
        t.n_views = n;
        t.ranges.assign(ranges, ranges + (size_t)2 * n * L * L);
        bp::write_clip_table(path, t);
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}

}  // extern "C"
