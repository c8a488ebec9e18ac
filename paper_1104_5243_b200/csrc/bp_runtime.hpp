// bp_runtime.hpp -- per-GPU slab context: the streamed upload pipeline, the
// batched kernel launches and the volume readback.
//
// Replaces the reference driver bp::reconstruct (proj/src/scheduler.cpp:24-133):
//   * validation of every matrix against the grid (scheduler.cpp:35) happens per
//     view as it arrives;
//   * the serial, in-timed-region pad_image copies (scheduler.cpp:110-120) become
//     asynchronous row-windowed H2D copies on a copy stream, overlapped with the
//     kernel of the previous batch through a ring of device projection slots;
//   * the std::thread pool + barriers (scheduler.cpp:65-106) become one kernel
//     launch per view batch on a compute stream;
//   * first-touch zeroing (scheduler.cpp:74) disappears: the first batch of a
//     reconstruction writes its accumulators without reading the volume.
#pragma once

#include <cuda_runtime.h>

#include <array>
#include <cstdint>
#include <memory>
#include <vector>

#include "../../include/bp_gpu.h"
#include "bp_device.hpp"
#include "bp_host.hpp"

namespace bpr {

void check(cudaError_t e, const char* what);

// Device-resident FDK preprocessing plan (bp_filter.cu): twiddles and the
// bit-reversed ramp spectrum for one detector width and geometry.
class RampFilter {
public:
    RampFilter(int isx, int isy, double sid, double sdd, double pitch);  // on the current device
    ~RampFilter();
    RampFilter(const RampFilter&) = delete;
    RampFilter& operator=(const RampFilter&) = delete;
    // filter rows [r0, r1) of nviews images in place (row pitch and view stride in floats)
    void apply(float* d_img, long long view_stride, int pitch, int nviews, int r0, int r1,
               cudaStream_t s) const;
    // one launch over a ring batch: view i at slot slots[i], rows [r0s[i], r1s[i])
    void apply_batch(float* d_ring, long long view_stride, int pitch, int n, const int* slots,
                     const int* r0s, const int* r1s, cudaStream_t s) const;
    int fft_length() const { return base_.M; }

private:
    bpg::FilterArgs base_{};
    float2* d_tw_ = nullptr;
    float* d_h_ = nullptr;
};

class SlabContext {
public:
    explicit SlabContext(const bp_gpu_config& cfg);
    ~SlabContext();
    SlabContext(const SlabContext&) = delete;
    SlabContext& operator=(const SlabContext&) = delete;

    // one view, ascending call order; copy=true stages the rows in pinned memory
    void backproject(const float* image, const double* A, bool copy);
    // drain, optional readback (nz*L*L floats), stats, reset for the next recon
    void finish(float* host_volume, bp_gpu_stats* st);
    void upload_views(const float* pixels, const double* mats, int count);
    void read_lines(const int* ys, const int* zs, int n, float* out);
    // exact per-line clip ranges (BPCT layout) for `count` matrices over the whole grid
    void clip_table(const double* mats, int count, uint16_t* host_ranges, uint64_t* total);
    double time_resident(int iters, bp_gpu_stats* st);

    float* device_volume() const { return d_vol_; }
    // where the finished volume lives: cfg.output_volume if set, else the slab buffer
    float* result() const { return out_vol_ ? out_vol_ : d_vol_; }
    int z_begin() const { return z0_; }
    int z_end() const { return z1_; }
    int device() const { return dev_; }
    const bp_gpu_config& config() const { return cfg_; }
    // device memory this context holds (volume if owned, rings, tables)
    size_t device_bytes() const;
    void bind() const;

private:
    void init();
    void release_all() noexcept;  // frees whatever has been allocated (destructor, failed init)
    struct Pending {
        bpg::BatchArgs b;
        int rg;          // ring group holding the batch's projections
        uint64_t index;  // batch index within the reconstruction
        std::array<int, bpg::kMaxBatch> fr0, fr1;  // rows to filter per view (cfg_.filter)
        bool filtered = false;
        bool expanded = false;
        bool band = false;  // its views' uploads are withheld (band tail, cfg_.views)
        cudaEvent_t ready = nullptr;  // the batch's inputs are final (uploaded + prepared)
    };
    // FDK filter and pair-ring expansion of a batch on the low-priority prep stream,
    // issued when the batch is queued so they run under earlier batches' kernels
    void prepare(Pending& p);
    // pair rows of the batch's slots; small: the co-resident small grid (under a kernel)
    void expand(const bpg::BatchArgs& b, cudaStream_t st, bool small = false);
    void flush();
    void choose_tile(const bpg::BatchArgs& b);
    // launch over slab-local z range [zc0, zc1) (default: the whole slab)
    void launch(const bpg::BatchArgs& b, int zc0 = 0, int zc1 = -1, bool final_pass = false);
    void launch_pending_front(bool final_pass = false);
    void launch_pending_group(int n, bool final_pass = false);
    void launch_ready();
    void reset_recon();
    void issue_run();  // pending coalesced H2D copy
    // band tail (cfg_.views > 0): a batch whose uploads were withheld gets
    // them view-major (when it must be launched before finish); or finish issues the whole
    // tail in detector-row bands, z-chunks outside in, each chunk read back as it completes
    void upload_withheld(Pending& p);
    void band_tail(float* host_volume, std::vector<std::pair<size_t, size_t>>& chunks);
    void copy_rows(const Pending& p, int r0, int r1);  // rows [r0, r1) of a band batch's views
    void mark_t0();  // first compute-stream work of a reconstruction

    bp_gpu_config cfg_;
    int dev_ = 0;
    bph::Grid grid_;
    int L_ = 0, z0_ = 0, z1_ = 0, nz_ = 0, isx_ = 0, isy_ = 0, pitch_ = 0;
    int B_ = 32, R_ = 3, slots_ = 0;
    bool own_vol_ = true;
    float* d_vol_ = nullptr;
    float* out_vol_ = nullptr;  // optional final-pass destination (may be peer memory)
    float* d_ring_ = nullptr;
    float* d_wx_ = nullptr;
    float* d_wy_ = nullptr;
    float* d_wz_ = nullptr;
    unsigned long long* d_cnt_ = nullptr;
    float* h_stage_ = nullptr;  // pinned staging, slots views
    cudaStream_t s_comp_ = nullptr, s_copy_ = nullptr;
    cudaStream_t s_comp2_ = nullptr;   // second compute stream: alternate z-chunks of the band tail
    cudaStream_t s_launch_ = nullptr;  // where launch() enqueues (s_comp_ except inside the band tail)
    cudaEvent_t ev_join_ = nullptr;
    cudaStream_t s_prep_ = nullptr;  // low priority: filter + expansion of queued batches
    cudaStream_t s_aux_ = nullptr;   // highest priority: expansion under a running kernel
    bool overlap_expand_ = true;     // BP_NO_OVERLAP_EXPAND=1: resident expansions in series
    int num_sms_ = 0;
    std::vector<cudaEvent_t> ev_ready_, ev_free_, ev_prep_;
    std::vector<bool> used_;
    cudaEvent_t ev_t0_ = nullptr, ev_t1_ = nullptr, ev_h0_ = nullptr, ev_h1_ = nullptr,
                ev_d0_ = nullptr, ev_d1_ = nullptr;
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> launch_ev_;
    size_t launch_ev_used_ = 0;

    // optional FDK preprocessing of every uploaded view (cfg_.filter)
    std::unique_ptr<RampFilter> filt_;
    std::array<int, bpg::kMaxBatch> fr0_{}, fr1_{};  // current batch's filtered rows

    // tiled kernel
    bool tiled_ = false;
    bpg::TileShape ts_{};
    alignas(64) unsigned char tmap_[128];
    // fast-mode pair ring: [slots][isy + 1][pitch] float2, built per
    // batch from d_ring_ by bp_expand_kernel
    bool pair_ok_ = true;  // BP_NO_PAIR=1 keeps the raw-tile fast kernel (A/B)
    float2* d_ringx_ = nullptr;
    alignas(64) unsigned char tmapx_[128];

    // deferred tail: the last tail_batches_ batches are held back and, when the
    // volume is read back, processed z-chunk-major so each finished chunk's D2H
    // overlaps the next chunk's kernels
    std::vector<Pending> pending_;
    int tail_batches_ = 3, tail_chunks_ = 8, bounce_chunks_ = 16;
    int merge_ = 1;  // view-major batches per launch (set by the reconstruction's first batch)
    uint64_t win_rows_ = 0;  // detector rows uploaded (or withheld) so far, summed over views
    uint64_t batch_index_ = 0;
    cudaStream_t s_d2h_ = nullptr;
    std::vector<cudaEvent_t> ev_chunk_;
    std::vector<cudaEvent_t> ev_dchunk_;  // a chunk's D2H has landed (pageable readback)
    float* h_bounce_ = nullptr;           // pinned bounce for a pageable host volume
    size_t bounce_bytes_ = 0;
    // band tail: views from band_start_ on are withheld; per ring slot their host image
    // (row 0), row window and matrix
    int band_start_ = -1;  // < 0: off
    bool band_on_ = false;  // this reconstruction withholds its tail
    int band_tail_zc_ = 0, band_tail_copy_ = 0;  // tail batches for zero-copy / copy callers
    int band_chunks_ = 16;
    std::vector<const char*> band_img_;
    std::vector<int> band_r0_, band_r1_;
    std::vector<bph::Mat> band_m_;
    std::vector<cudaEvent_t> ev_band_;
    cudaEvent_t ev_band_pre_ = nullptr;  // BP_BAND_TRACE: the view-major uploads are done

    // pending H2D run on s_copy_: run_n_ views whose images start at run_img0_ + i * view
    // bytes, into ring slots run_slot0_ + i, rows [run_r0_, run_r1_) (the union of their
    // row windows); run_actual_ = the views' own window bytes
    const char* run_img0_ = nullptr;
    int run_slot0_ = 0, run_n_ = 0, run_r0_ = 0, run_r1_ = 0;
    size_t run_actual_ = 0, run_limit_ = (size_t)32 << 20;

    // per-reconstruction state
    bpg::BatchArgs cur_{};
    int nb_ = 0;
    int rg_ = 0;
    bool any_launch_ = false;
    bool t0_rec_ = false;
    bool any_h2d_ = false;
    uint64_t views_ = 0, launches_ = 0, prep_launches_ = 0, h2d_bytes_ = 0;
    double wall_t0_ = 0.0;

    // resident views
    int resident_ = 0;
    std::vector<std::array<float, 12>> resident_A_;
};

double now_ms();

}  // namespace bpr
