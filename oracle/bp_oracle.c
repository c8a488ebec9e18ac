/*
 * bp_oracle.c -- CPU restatement of the reference backprojection path.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker for the CUDA
 * product in paper_1104_5243_b200/.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load it.  The product
 * never links, loads or falls back to it.
 *
 * It restates, in plain C (compiled with -ffp-contract=off exactly like the
 * reference, proj/CMakeLists.txt:13), the float pipeline of
 *   - bp::line_update_scalar          proj/src/kernel.cpp:49-85
 *   - bp::bilinear                    proj/src/kernel.hpp:47-51
 *   - clamp_coord                     proj/src/kernel.cpp:28
 *   - recip_exact                     proj/src/recip.hpp:12
 *   - VoxelGrid::cube / world_*       proj/src/geometry.cpp:11-19, geometry.hpp:20-22
 *   - ProjectionMatrix::narrowed      proj/src/geometry.cpp:21-25
 *   - validate_matrix_for_grid        proj/src/geometry.cpp:130-144
 *   - bp::reconstruct (per-voxel ascending view order)  proj/src/scheduler.cpp:24-133
 *   - LineProjector::visible / build_clip_table / clip_stats
 *                                     proj/src/precompute.cpp:19-103
 * The padded image of pad_image (kernel.cpp:32-47) is replaced by guarded reads
 * that return 0 outside the detector, which is the same value the zero border
 * supplies for every index the clamp [-2, ISX] x [-2, ISY] can produce.
 *
 * Parity is pinned two ways (tests/test_oracle.py): against the reference's
 * own library built from /root/reference by oracle/Makefile (oracle/_ref/,
 * bitwise), and against golden fixtures generated from that library and
 * committed under tests/golden/ (tests/golden/make_golden.py).
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef struct bpo_grid {
    int L;
    double MM;
    double ox, oy, oz;
} bpo_grid;

/* VoxelGrid::cube, geometry.cpp:11-19 */
void bpo_grid_cube(int L, bpo_grid* g) {
    g->L = L;
    g->MM = 256.0 / L;
    double off = -0.5 * (L - 1) * g->MM;
    g->ox = g->oy = g->oz = off;
}

static inline float world_f(double off, double MM, int i) { return (float)(off + i * MM); }

/* ProjectionMatrix::narrowed, geometry.cpp:21-25 */
void bpo_narrow(const double* a, float* f) {
    for (int i = 0; i < 12; ++i) f[i] = (float)a[i];
}

/* validate_matrix_for_grid, geometry.cpp:130-144: returns 0 if w > 0 at all 8 corners */
int bpo_validate(const double* a, const bpo_grid* g) {
    double lo[3] = {g->ox, g->oy, g->oz};
    double hi[3] = {g->ox + (g->L - 1) * g->MM, g->oy + (g->L - 1) * g->MM,
                    g->oz + (g->L - 1) * g->MM};
    for (int i = 0; i < 8; ++i) {
        double wx = (i & 1) ? hi[0] : lo[0];
        double wy = (i & 2) ? hi[1] : lo[1];
        double wz = (i & 4) ? hi[2] : lo[2];
        double w = a[2] * wx + a[5] * wy + a[8] * wz + a[11];
        if (!(w > 0.0)) return -1;
    }
    return 0;
}

static inline float pix(const float* img, int isx, int isy, int iu, int iv) {
    return (iu >= 0 && iu < isx && iv >= 0 && iv < isy) ? img[(size_t)iv * isx + iu] : 0.0f;
}

static inline float clamp_coord(float c, float hi) {
    /* std::min(std::max(c, -2.0f), hi) with std:: argument order semantics */
    float m = (c < -2.0f) ? -2.0f : c;
    return (hi < m) ? hi : m;
}

/* line_update_scalar, kernel.cpp:49-85 (exact reciprocal, strict arithmetic) */
uint64_t bpo_line_update(float* line, const float* img, int isx, int isy, const float* A,
                         const bpo_grid* g, int y, int z, int x0, int x1, int distance_weight) {
    if (x1 < x0) return 0;
    const float wy = world_f(g->oy, g->MM, y);
    const float wz = world_f(g->oz, g->MM, z);
    const float hi_u = (float)isx;
    const float hi_v = (float)isy;
    const float uy = A[3] * wy + A[6] * wz + A[9];
    const float vy = A[4] * wy + A[7] * wz + A[10];
    const float wy_ = A[5] * wy + A[8] * wz + A[11];
    for (int x = x0; x <= x1; ++x) {
        const float wx = world_f(g->ox, g->MM, x);
        float uw = A[0] * wx + uy;
        float vw = A[1] * wx + vy;
        float w = A[2] * wx + wy_;
        float r = 1.0f / w;
        float u = clamp_coord(uw * r, hi_u);
        float v = clamp_coord(vw * r, hi_v);
        int iu = (int)floorf(u);
        int iv = (int)floorf(v);
        float scalx = u - (float)iu;
        float scaly = v - (float)iv;
        float valtl = pix(img, isx, isy, iu, iv);
        float valtr = pix(img, isx, isy, iu + 1, iv);
        float valbl = pix(img, isx, isy, iu, iv + 1);
        float valbr = pix(img, isx, isy, iu + 1, iv + 1);
        /* bilinear, kernel.hpp:47-51 */
        float vall = scaly * valbl + (1.0f - scaly) * valtl;
        float valr = scaly * valbr + (1.0f - scaly) * valtr;
        float fx = scalx * valr + (1.0f - scalx) * vall;
        line[x] += distance_weight ? fx * (r * r) : fx;
    }
    return (uint64_t)(x1 - x0 + 1);
}

/* LineProjector::visible, precompute.cpp:37-46 */
static inline int visible(const float* A, float uy, float vy, float wy_, float wx, float hi_u,
                          float hi_v) {
    float w = A[2] * wx + wy_;
    float r = 1.0f / w;
    float u = clamp_coord((A[0] * wx + uy) * r, hi_u);
    float v = clamp_coord((A[1] * wx + vy) * r, hi_v);
    int iu = (int)floorf(u);
    int iv = (int)floorf(v);
    return iu >= -1 && iu <= (int)hi_u - 1 && iv >= -1 && iv <= (int)hi_v - 1;
}

/* build_clip_table scan for one line, precompute.cpp:64-80.  Returns 0 for an
 * empty line, else 1 with [*first,*last]. */
int bpo_clip_line(const float* A, const bpo_grid* g, int isx, int isy, int y, int z, int* first,
                  int* last) {
    const int L = g->L;
    const float wy = world_f(g->oy, g->MM, y);
    const float wz = world_f(g->oz, g->MM, z);
    const float uy = A[3] * wy + A[6] * wz + A[9];
    const float vy = A[4] * wy + A[7] * wz + A[10];
    const float wy_ = A[5] * wy + A[8] * wz + A[11];
    const float hu = (float)isx, hv = (float)isy;
    int f = 0;
    while (f < L && !visible(A, uy, vy, wy_, world_f(g->ox, g->MM, f), hu, hv)) ++f;
    if (f == L) return 0;
    int l = L - 1;
    while (l > f && !visible(A, uy, vy, wy_, world_f(g->ox, g->MM, l), hu, hv)) --l;
    *first = f;
    *last = l;
    return 1;
}

/* ---- threaded drivers ------------------------------------------------- */

typedef struct job {
    const float* pixels;
    const double* mats;
    int nviews, isx, isy;
    const bpo_grid* g;
    int z0, z1;
    int distance_weight;
    int nthreads, tid;
    float* out;
    const int* ys;
    const int* zs;
    int nlines;
    uint64_t updates;
    uint64_t* per_view_visible; /* for clip stats: [nviews] per thread slot */
} job;

static void* recon_worker(void* arg) {
    job* j = (job*)arg;
    const int L = j->g->L;
    float* Af = (float*)malloc(sizeof(float) * 12 * (size_t)j->nviews);
    for (int k = 0; k < j->nviews; ++k) bpo_narrow(j->mats + 12 * k, Af + 12 * k);
    const size_t img_px = (size_t)j->isx * j->isy;
    /* z-slices round-robin over threads (partition_slices with chunk 1,
     * scheduler.cpp:12-22); per voxel, views are applied in ascending order.
     * Views are taken in blocks of 8 around the thread's lines (the reference's
     * projection blocking, scheduler.cpp:77-100), so a block's images stay
     * cache-resident; per-line view order is unchanged, hence bitwise the same. */
    const int VB = 8;
    for (int k0 = 0; k0 < j->nviews; k0 += VB) {
        const int k1 = k0 + VB < j->nviews ? k0 + VB : j->nviews;
        for (int z = j->z0 + j->tid; z < j->z1; z += j->nthreads) {
            for (int y = 0; y < L; ++y) {
                float* line = j->out + ((size_t)(z - j->z0) * L + y) * L;
                for (int k = k0; k < k1; ++k)
                    j->updates += bpo_line_update(line, j->pixels + img_px * k, j->isx, j->isy,
                                                  Af + 12 * k, j->g, y, z, 0, L - 1,
                                                  j->distance_weight);
            }
        }
    }
    free(Af);
    return NULL;
}

static void* lines_worker(void* arg) {
    job* j = (job*)arg;
    const int L = j->g->L;
    float* Af = (float*)malloc(sizeof(float) * 12 * (size_t)j->nviews);
    for (int k = 0; k < j->nviews; ++k) bpo_narrow(j->mats + 12 * k, Af + 12 * k);
    const size_t img_px = (size_t)j->isx * j->isy;
    for (int i = j->tid; i < j->nlines; i += j->nthreads) {
        float* line = j->out + (size_t)i * L;
        for (int k = 0; k < j->nviews; ++k)
            j->updates += bpo_line_update(line, j->pixels + img_px * k, j->isx, j->isy,
                                          Af + 12 * k, j->g, j->ys[i], j->zs[i], 0, L - 1,
                                          j->distance_weight);
    }
    free(Af);
    return NULL;
}

static void* clip_worker(void* arg) {
    job* j = (job*)arg;
    const int L = j->g->L;
    float A[12];
    for (int k = j->tid; k < j->nviews; k += j->nthreads) {
        bpo_narrow(j->mats + 12 * k, A);
        uint64_t vis = 0;
        for (int z = j->z0; z < j->z1; ++z)
            for (int y = 0; y < L; ++y) {
                int f, l;
                if (bpo_clip_line(A, j->g, j->isx, j->isy, y, z, &f, &l)) vis += (uint64_t)(l - f + 1);
            }
        j->per_view_visible[k] = vis;
    }
    return NULL;
}

static int run_threads(job* proto, void* (*fn)(void*), int threads, uint64_t* updates) {
    if (threads < 1) threads = 1;
    job* jobs = (job*)calloc((size_t)threads, sizeof(job));
    pthread_t* th = (pthread_t*)calloc((size_t)threads, sizeof(pthread_t));
    for (int t = 0; t < threads; ++t) {
        jobs[t] = *proto;
        jobs[t].nthreads = threads;
        jobs[t].tid = t;
        jobs[t].updates = 0;
        pthread_create(&th[t], NULL, fn, &jobs[t]);
    }
    uint64_t total = 0;
    for (int t = 0; t < threads; ++t) {
        pthread_join(th[t], NULL);
        total += jobs[t].updates;
    }
    if (updates) *updates = total;
    free(jobs);
    free(th);
    return 0;
}

/* Full (or z-slab) reconstruction, out = (z1-z0)*L*L floats, x fastest.
 * Caller zero-fills or pre-loads `out`; contributions are added in ascending
 * view order exactly as bp::reconstruct does (scheduler.cpp:77-97). */
int bpo_reconstruct(const float* pixels, const double* mats, int nviews, int isx, int isy,
                    const bpo_grid* g, int z0, int z1, int distance_weight, int threads,
                    float* out, uint64_t* updates) {
    if (nviews < 1 || isx < 2 || isy < 2 || z0 < 0 || z1 > g->L || z0 > z1) return -1;
    for (int k = 0; k < nviews; ++k)
        if (bpo_validate(mats + 12 * k, g) != 0) return -3;
    job p;
    memset(&p, 0, sizeof p);
    p.pixels = pixels;
    p.mats = mats;
    p.nviews = nviews;
    p.isx = isx;
    p.isy = isy;
    p.g = g;
    p.z0 = z0;
    p.z1 = z1;
    p.distance_weight = distance_weight;
    p.out = out;
    return run_threads(&p, recon_worker, threads, updates);
}

/* Sampled-line oracle: out = nlines*L floats, caller-initialised. */
int bpo_reconstruct_lines(const float* pixels, const double* mats, int nviews, int isx, int isy,
                          const bpo_grid* g, const int* ys, const int* zs, int nlines,
                          int distance_weight, int threads, float* out) {
    if (nviews < 1 || isx < 2 || isy < 2) return -1;
    job p;
    memset(&p, 0, sizeof p);
    p.pixels = pixels;
    p.mats = mats;
    p.nviews = nviews;
    p.isx = isx;
    p.isy = isy;
    p.g = g;
    p.ys = ys;
    p.zs = zs;
    p.nlines = nlines;
    p.distance_weight = distance_weight;
    p.out = out;
    return run_threads(&p, lines_worker, threads, NULL);
}

/* clip_stats total (precompute.cpp:93-103) per view over slab [z0,z1). */
int bpo_visible_updates(const double* mats, int nviews, int isx, int isy, const bpo_grid* g,
                        int z0, int z1, int threads, uint64_t* per_view) {
    job p;
    memset(&p, 0, sizeof p);
    p.mats = mats;
    p.nviews = nviews;
    p.isx = isx;
    p.isy = isy;
    p.g = g;
    p.z0 = z0;
    p.z1 = z1;
    p.per_view_visible = per_view;
    return run_threads(&p, clip_worker, threads, NULL);
}
