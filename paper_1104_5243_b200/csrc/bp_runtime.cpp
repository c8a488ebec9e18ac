// bp_runtime.cpp -- see bp_runtime.hpp.
#include "bp_runtime.hpp"

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <string>

namespace bpr {

void check(cudaError_t e, const char* what) {
    if (e != cudaSuccess) {
        cudaGetLastError();
        throw bph::device_error(std::string(what) + ": " + cudaGetErrorString(e));
    }
}

double now_ms() {
    return std::chrono::duration<double, std::milli>(
               std::chrono::steady_clock::now().time_since_epoch())
        .count();
}

namespace {
int round_up(int v, int m) { return (v + m - 1) / m * m; }
}  // namespace

RampFilter::RampFilter(int isx, int isy, double sid, double sdd, double pitch) {
    if (isx > bpg::kMaxFilterM / 2) throw bph::config_error("filter: detector wider than 8192 pixels");
    if (isx < 2) throw bph::config_error("detector must be at least 2 pixels wide");
    if (!(sid > 0) || !(sdd > 0) || !(pitch > 0)) throw bph::config_error("filter geometry must be positive");
    // FFT length: the linear convolution of isx samples with the (2 isx - 1)-tap kernel
    // needs M >= 2 isx - 1.  Mixed radix M = R0 * 2^q (R0 in {1, 3, 5}, 2^q >= 16 when
    // R0 > 1) takes the smallest such length: 2560 instead of 4096 at isx = 1248.
    const int need = 2 * isx - 1;
    int M = 0, R0 = 1;
    for (int r0 : {1, 3, 5})
        for (int n2 = (r0 == 1 ? 2 : 16); (long long)r0 * n2 <= bpg::kMaxFilterM; n2 *= 2)
            if (r0 * n2 >= need) {
                if (M == 0 || r0 * n2 < M) { M = r0 * n2; R0 = r0; }
                break;
            }
    if (const char* e = std::getenv("BP_FILTER_POW2"))  // A/B: force the radix-2 length
        if (std::atoi(e)) {
            M = 2;
            while (M < need) M *= 2;
            R0 = 1;
        }
    const int N2 = M / R0;
    int q = 0;
    while ((1 << q) < N2) ++q;
    // spectrum of the zero-padded Ram-Lak kernel (bph::ramp_spectrum's h), real since h
    // is even: H[k] = sum_n h[n] cos(2 pi k n / M), in double
    const double tau = pitch * sid / sdd;
    std::vector<double> h((size_t)isx);
    for (int n = 0; n < isx; ++n)
        h[(size_t)n] = n == 0 ? 1.0 / (4.0 * tau * tau)
                              : ((n & 1) ? -1.0 / (M_PI * M_PI * (double)n * (double)n * tau * tau) : 0.0);
    std::vector<double> ctab((size_t)M), H((size_t)M);
    for (int t = 0; t < M; ++t) ctab[(size_t)t] = std::cos(2.0 * M_PI * (double)t / (double)M);
    for (int k = 0; k < M; ++k) {
        double acc = h[0];
        for (int n = 1; n < isx; n += 2) acc += 2.0 * h[(size_t)n] * ctab[(size_t)((long long)k * n % M)];
        H[(size_t)k] = acc;
    }
    // register passes of <= 4 radix-2 stages over N2; the leading pass takes the remainder
    base_.ngroups = 0;
    int lead = q % 4 == 0 ? 4 : q % 4;
    if (q < 4) lead = q;
    base_.r[base_.ngroups++] = lead;
    for (int left = q - lead; left > 0; left -= 4) base_.r[base_.ngroups++] = 4;
    // per-pass twiddle bases alpha_{i,j,s} = exp(-2 pi i j / (2 g_i 2^s)) (bp_filter.cu twiddle())
    auto w = [](double frac) {  // exp(-2 pi i frac)
        return make_float2((float)std::cos(2.0 * M_PI * frac), (float)-std::sin(2.0 * M_PI * frac));
    };
    std::vector<float2> tw;
    int lg = q;
    for (int i = 0; i < base_.ngroups; ++i) {
        lg -= base_.r[i];
        base_.twoff[i] = (int)tw.size();
        const int g = 1 << lg;
        for (int j = 0; j < g; ++j)
            for (int s2 = 0; s2 < base_.r[i]; ++s2)
                tw.push_back(w((double)j / (double)((long long)2 * g << s2)));
    }
    // leading radix-R0 twiddles W_M^(j m'), m' in [1, R0)
    std::vector<float2> twr;
    for (int m = 1; m < R0; ++m)
        for (int j = 0; j < N2; ++j) twr.push_back(w((double)((long long)j * m % M) / (double)M));
    // H in the forward network's output order: sigma(m' N2 + j) = m' + R0 * bitrev_q(j)
    std::vector<float> hp((size_t)M);
    for (int mp = 0; mp < R0; ++mp)
        for (int j = 0; j < N2; ++j) {
            int rev = 0;
            for (int b = 0; b < q; ++b) rev |= ((j >> b) & 1) << (q - 1 - b);
            hp[(size_t)mp * N2 + j] = (float)(H[(size_t)(mp + R0 * rev)] * tau / (double)M);
        }
    check(cudaMalloc(&d_tw_, (tw.size() + twr.size() + 1) * sizeof(float2)), "cudaMalloc(filter)");
    check(cudaMalloc(&d_h_, hp.size() * sizeof(float)), "cudaMalloc(filter)");
    check(cudaMemcpy(d_tw_, tw.data(), tw.size() * sizeof(float2), cudaMemcpyHostToDevice), "filter");
    if (!twr.empty())
        check(cudaMemcpy(d_tw_ + tw.size(), twr.data(), twr.size() * sizeof(float2), cudaMemcpyHostToDevice),
              "filter");
    check(cudaMemcpy(d_h_, hp.data(), hp.size() * sizeof(float), cudaMemcpyHostToDevice), "filter");
    base_.isx = isx;
    base_.M = M;
    base_.R0 = R0;
    base_.N2 = N2;
    base_.tw = d_tw_;
    base_.twr = d_tw_ + tw.size();
    base_.hperm = d_h_;
    base_.sdd = sdd;
    base_.cu = 0.5 * (isx - 1);
    base_.cv = 0.5 * (isy - 1);
    base_.pitch_mm = pitch;
}

RampFilter::~RampFilter() {
    cudaFree(d_tw_);
    cudaFree(d_h_);
}

void RampFilter::apply_batch(float* d_ring, long long view_stride, int pitch, int n, const int* slots,
                             const int* r0s, const int* r1s, cudaStream_t s) const {
    if (n < 1 || n > bpg::kMaxBatch) throw bph::config_error("filter batch out of range");
    bpg::FilterArgs a = base_;
    a.img = d_ring;
    a.view_stride = view_stride;
    a.pitch = pitch;
    a.per_view = 1;
    int lo = 0, hi = 0;
    for (int i = 0; i < n; ++i) {
        a.slot[i] = slots[i];
        a.vrow0[i] = r0s[i];
        a.vrow1[i] = r1s[i];
        hi = std::max(hi, r1s[i] - r0s[i]);
    }
    a.row0 = lo;
    a.row1 = hi;  // grid.x covers the tallest window
    check((cudaError_t)bpg::launch_ramp_filter(a, n, s), "ramp filter launch");
}

void RampFilter::apply(float* d_img, long long view_stride, int pitch, int nviews, int r0, int r1,
                       cudaStream_t s) const {
    bpg::FilterArgs a = base_;
    a.img = d_img;
    a.view_stride = view_stride;
    a.pitch = pitch;
    a.row0 = r0;
    a.row1 = r1;
    check((cudaError_t)bpg::launch_ramp_filter(a, nviews, s), "ramp filter launch");
}

void SlabContext::prepare(Pending& p) {
    // FDK preprocessing of the batch's ring slots in place, then the pair ring, on
    // the low-priority prep stream once the batch's uploads are complete.  Neither
    // delays the copy stream nor stalls earlier, ready backprojection launches; the
    // backprojection of this batch waits on p.ready.  Done once per batch, even when
    // the deferred tail launches it once per z-chunk.
    if (p.ready) return;
    const bool filt = filt_ && !p.filtered;
    const bool expd = tiled_ && ts_.dy && !p.expanded;
    if (!filt && !expd) {
        p.ready = ev_ready_[(size_t)p.rg];
        return;
    }
    mark_t0();  // the prep work belongs to the reconstruction's device time
    check(cudaStreamWaitEvent(s_prep_, ev_t0_, 0), "wait");
    check(cudaStreamWaitEvent(s_prep_, ev_ready_[(size_t)p.rg], 0), "wait");
    if (filt) {
        filt_->apply_batch(d_ring_, (long long)isy_ * pitch_, pitch_, p.b.nviews, p.b.slot,
                           p.fr0.data(), p.fr1.data(), s_prep_);
        ++prep_launches_;
        p.filtered = true;
    }
    if (expd) {
        expand(p.b, s_prep_);
        p.expanded = true;
    }
    check(cudaEventRecord(ev_prep_[(size_t)p.rg], s_prep_), "event");
    p.ready = ev_prep_[(size_t)p.rg];
}

void SlabContext::expand(const bpg::BatchArgs& b, cudaStream_t st, bool small) {
    if (!tiled_ || !ts_.dy) return;
    bpg::ExpandArgs a{};
    a.ring = d_ring_;
    a.ringx = d_ringx_;
    a.isx = isx_;
    a.isy = isy_;
    a.pitch = pitch_;
    a.pitchx = pitch_;
    for (int i = 0; i < b.nviews; ++i) a.slot[i] = b.slot[i];
    check((cudaError_t)(small ? bpg::launch_expand_small(a, b.nviews, num_sms_, st)
                              : bpg::launch_expand(a, b.nviews, st)),
          "pair ring expansion");
    ++prep_launches_;
}

void SlabContext::mark_t0() {
    if (!t0_rec_) {
        check(cudaEventRecord(ev_t0_, s_comp_), "event");
        t0_rec_ = true;
    }
}

void SlabContext::bind() const { check(cudaSetDevice(dev_), "cudaSetDevice"); }

SlabContext::SlabContext(const bp_gpu_config& cfg) : cfg_(cfg) {
    // a failed allocation part-way through must not leak what was already allocated
    try {
        init();
    } catch (...) {
        release_all();
        throw;
    }
}

size_t SlabContext::device_bytes() const {
    size_t b = (size_t)slots_ * isy_ * pitch_ * sizeof(float) + 3 * (size_t)(L_ + 160) * sizeof(float);
    if (own_vol_) b += (size_t)nz_ * L_ * L_ * sizeof(float);
    if (d_ringx_) b += (size_t)slots_ * (isy_ + 1) * pitch_ * sizeof(float2);
    return b;
}

void SlabContext::init() {
    const bp_gpu_config& cfg = cfg_;
    if (cfg.l < 1) throw bph::config_error("grid edge must be >= 1 voxel");
    if (cfg.isx < 2 || cfg.isy < 2) throw bph::config_error("detector must be at least 2x2 pixels");
    if (cfg.recip_mode < BP_RECIP_EXACT || cfg.recip_mode > BP_RECIP_HW_APPROX)
        throw bph::config_error("recip_mode out of range");
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev < 1) {
        cudaGetLastError();
        throw bph::device_error("no CUDA device available (the GPU path has no CPU fallback)");
    }
    if (cfg.device >= 0) {
        if (cfg.device >= ndev) throw bph::config_error("device ordinal out of range");
        dev_ = cfg.device;
    } else {
        check(cudaGetDevice(&dev_), "cudaGetDevice");
    }
    bind();
    L_ = (int)cfg.l;
    grid_ = bph::Grid::cube(L_, cfg.offset_mm[0], cfg.offset_mm[1], cfg.offset_mm[2]);
    z0_ = cfg.z_begin;
    z1_ = cfg.z_end > 0 ? cfg.z_end : L_;
    if (z0_ < 0 || z1_ > L_ || z0_ >= z1_) throw bph::config_error("slab [z_begin, z_end) out of range");
    nz_ = z1_ - z0_;
    isx_ = (int)cfg.isx;
    isy_ = (int)cfg.isy;
    pitch_ = round_up(isx_, 4);  // TMA global strides must be multiples of 16 B
    // default register batch: 32 views; 62 for a whole volume of 1024^3 or more, whose compute
    // outlasts its upload, so that halving the volume read-modify-write passes pays
    // (1024^3 e2e 328 -> 314 ms, A/B profiles/round2_e2e_batch_1024.txt)
    B_ = cfg.view_batch > 0 ? cfg.view_batch : ((long long)(z1_ - z0_) * L_ * L_ >= (1ll << 30) ? 62 : 32);
    if (B_ > bpg::kMaxBatch) throw bph::config_error("view_batch exceeds 256");
    R_ = cfg.ring_batches > 0 ? cfg.ring_batches : 8;
    // measured on B200 at 512^3 (tools: scratch e2e A/B): deferring 3 batches and
    // streaming 8 z-chunks back hides most of the 10 ms volume readback.  A z-slab of a
    // multi-GPU split uploads only its row windows, so its upload ends well before its
    // compute and 5 deferred batches hide more of its readback (1024^3, outer slab of 8:
    // 60.6 -> 55.7 ms; the whole volume at 512^3 prefers 3: 53.5 vs 59.2 ms)
    // With the view count known (cfg.views), the deferred tail is the band tail: its
    // ~112-128 views' rows are uploaded band-ordered at finish, so its chunks complete and
    // read back under the remaining upload (512^3: 53.5 -> 48.5 ms; 3 / 4 / 5 batches of 32
    // measured 50.7 / 48.5 / 48.6 ms)
    // A z-slab of a multi-GPU split reads back a larger share of its work (the outer slabs
    // at 1024^3, G = 8: 0.9 GB = 16 ms of D2H for 39 ms of compute), so its band tail is
    // ~186 views (3 batches of 62: slowest slab 49.3 -> 45.4 ms; 4: 45.4, 5: 48.6).
    const int band_views = (z1_ - z0_ < L_) ? 186 : 112;
    const int tail_default = cfg.views > 0 ? std::max(1, (band_views + B_ / 2) / B_)
                             : (z1_ - z0_ < L_)          ? 5
                                                          : 3;
    tail_batches_ = std::max(0, std::min(R_ - 2, cfg.tail_batches >= 0 ? cfg.tail_batches : tail_default));
    tail_chunks_ = 8;
    // a pageable destination adds a host copy per chunk after its D2H; smaller chunks
    // leave less of it exposed after the last one (e2e_copy 61.9 -> 60.9 ms at 512^3)
    bounce_chunks_ = 16;
    if (const char* e = std::getenv("BP_TAIL_BATCHES")) tail_batches_ = std::max(0, std::atoi(e));
    if (const char* e = std::getenv("BP_TAIL_CHUNKS")) bounce_chunks_ = tail_chunks_ = std::max(1, std::atoi(e));
    if (const char* e = std::getenv("BP_H2D_RUN_MB")) run_limit_ = (size_t)std::max(0, std::atoi(e)) << 20;
    if (const char* e = std::getenv("BP_NO_PAIR")) pair_ok_ = std::atoi(e) == 0;
    out_vol_ = cfg.output_volume;
    // the final batch must be launched by finish(), which knows it is the last
    if (out_vol_) tail_batches_ = std::max(tail_batches_, 1);
    slots_ = B_ * R_;

    const size_t vol_elems = (size_t)nz_ * L_ * L_;
    if (cfg.device_volume) {
        own_vol_ = false;
        d_vol_ = cfg.device_volume;
    } else {
        check(cudaMalloc(&d_vol_, vol_elems * sizeof(float)), "cudaMalloc(volume)");
    }
    check(cudaMalloc(&d_ring_, (size_t)slots_ * isy_ * pitch_ * sizeof(float)), "cudaMalloc(ring)");
    check(cudaMemset(d_ring_, 0, (size_t)slots_ * isy_ * pitch_ * sizeof(float)), "cudaMemset(ring)");
    const int tab = L_ + 160;  // padded so nominal block extents beyond L stay in-table
    auto hwx = bph::world_table(grid_.ox, grid_.MM, tab);
    auto hwy = bph::world_table(grid_.oy, grid_.MM, tab);
    auto hwz = bph::world_table(grid_.oz, grid_.MM, tab);
    check(cudaMalloc(&d_wx_, tab * sizeof(float)), "cudaMalloc(tables)");
    check(cudaMalloc(&d_wy_, tab * sizeof(float)), "cudaMalloc(tables)");
    check(cudaMalloc(&d_wz_, tab * sizeof(float)), "cudaMalloc(tables)");
    check(cudaMemcpy(d_wx_, hwx.data(), tab * sizeof(float), cudaMemcpyHostToDevice), "tables");
    check(cudaMemcpy(d_wy_, hwy.data(), tab * sizeof(float), cudaMemcpyHostToDevice), "tables");
    check(cudaMemcpy(d_wz_, hwz.data(), tab * sizeof(float), cudaMemcpyHostToDevice), "tables");
    check(cudaMalloc(&d_cnt_, 8 * sizeof(unsigned long long)), "cudaMalloc(counters)");
    check(cudaMemset(d_cnt_, 0, 8 * sizeof(unsigned long long)), "cudaMemset(counters)");
    int prio_lo = 0, prio_hi = 0;
    check(cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi), "stream priorities");
    // s_aux_ outranks s_comp_ so its small grid is dispatched ahead of a backprojection
    // grid that becomes ready at the same time
    const int prio_comp = prio_hi < prio_lo ? prio_hi + 1 : prio_hi;
    check(cudaStreamCreateWithPriority(&s_comp_, cudaStreamNonBlocking, prio_comp), "stream");
    check(cudaStreamCreateWithPriority(&s_comp2_, cudaStreamNonBlocking, prio_comp), "stream");
    check(cudaEventCreateWithFlags(&ev_join_, cudaEventDisableTiming), "event");
    s_launch_ = s_comp_;
    check(cudaStreamCreateWithPriority(&s_aux_, cudaStreamNonBlocking, prio_hi), "stream");
    check(cudaStreamCreateWithPriority(&s_prep_, cudaStreamNonBlocking, prio_lo), "stream");
    check(cudaDeviceGetAttribute(&num_sms_, cudaDevAttrMultiProcessorCount, dev_), "SM count");
    if (const char* e = std::getenv("BP_NO_OVERLAP_EXPAND")) overlap_expand_ = std::atoi(e) == 0;
    check(cudaStreamCreateWithFlags(&s_copy_, cudaStreamNonBlocking), "stream");
    check(cudaStreamCreateWithFlags(&s_d2h_, cudaStreamNonBlocking), "stream");
    // BP_BAND_TRACE=1: timing events for the band-tail diagnostics
    const unsigned trace_flags = std::getenv("BP_BAND_TRACE") ? cudaEventDefault : cudaEventDisableTiming;
    ev_chunk_.resize((size_t)std::max({tail_chunks_, bounce_chunks_, 32}));
    for (auto& e : ev_chunk_) check(cudaEventCreateWithFlags(&e, trace_flags), "event");
    ev_dchunk_.resize((size_t)std::max({tail_chunks_, bounce_chunks_, 32}));
    for (auto& e : ev_dchunk_) check(cudaEventCreateWithFlags(&e, trace_flags), "event");
    // 12 z-chunks (512^3: 8 / 12 / 16 chunks 48.8 / 48.5 / 48.6 ms), more for slabs above 1.5 GB so
    // that the last chunk's readback, which nothing overlaps, stays near 128 MB (1024^3: 12 / 16 /
    // 24 / 32 chunks 305.6 / 304.4 / 302.7 / 302.1 ms)
    band_chunks_ = (int)std::min<size_t>(
        ev_chunk_.size(), std::max<size_t>(12, std::min<size_t>(32, (vol_elems * sizeof(float)) >> 27)));
    if (const char* e = std::getenv("BP_BAND_CHUNKS"))
        band_chunks_ = std::max(1, std::min((int)ev_chunk_.size(), std::atoi(e)));
    ev_band_.resize((size_t)band_chunks_);
    for (auto& e : ev_band_) check(cudaEventCreateWithFlags(&e, trace_flags), "event");
    check(cudaEventCreateWithFlags(&ev_band_pre_, trace_flags), "event");
    band_img_.assign((size_t)slots_, nullptr);
    band_r0_.assign((size_t)slots_, 0);
    band_r1_.assign((size_t)slots_, 0);
    band_m_.assign((size_t)slots_, bph::Mat{});
    // the last tail_batches_ batches of a cfg.views-view reconstruction form the band tail
    // (BP_NO_BAND=1: off, for A/B).  The tail is settled per reconstruction by its first
    // call: zero-copy callers get the band tail; copy-semantics callers do not.  Their views
    // arrive at host-copy pace, and e2e_copy is bound by host DRAM traffic (staging, the
    // DMA's own reads, the bounce readback and its copy): band tails of 32 / 64 / 96 / 128
    // views measured 63.5 / 63.0 / 62.5 / 63.8 ms against 62.4 ms without (A/B knob
    // BP_COPY_BAND_VIEWS, views)
    if (cfg.views > 0 && tail_batches_ > 0 && !std::getenv("BP_NO_BAND")) {
        band_tail_zc_ = tail_batches_;
        int cv = 0;
        if (const char* e = std::getenv("BP_COPY_BAND_VIEWS")) cv = std::max(0, std::atoi(e));
        band_tail_copy_ = (cfg.tail_batches >= 0 || std::getenv("BP_TAIL_BATCHES"))
                              ? tail_batches_
                              : std::max(1, std::min(tail_batches_, (cv + B_ / 2) / B_));
        if (cv == 0) band_tail_copy_ = 0;
        band_start_ = 0;  // set per reconstruction
    }
    ev_ready_.resize((size_t)R_);
    ev_free_.resize((size_t)R_);
    ev_prep_.resize((size_t)R_);
    used_.assign((size_t)R_, false);
    for (int i = 0; i < R_; ++i) {
        check(cudaEventCreateWithFlags(&ev_ready_[(size_t)i], cudaEventDisableTiming), "event");
        check(cudaEventCreateWithFlags(&ev_free_[(size_t)i], cudaEventDisableTiming), "event");
        check(cudaEventCreateWithFlags(&ev_prep_[(size_t)i], cudaEventDisableTiming), "event");
    }
    for (cudaEvent_t* e : {&ev_t0_, &ev_t1_, &ev_h0_, &ev_h1_, &ev_d0_, &ev_d1_})
        check(cudaEventCreate(e), "event");
    std::memset(tmap_, 0, sizeof tmap_);
    std::memset(tmapx_, 0, sizeof tmapx_);
    if (cfg.filter) filt_ = std::make_unique<RampFilter>(isx_, isy_, cfg.sid_mm, cfg.sdd_mm, cfg.pitch_mm);
    reset_recon();
}

SlabContext::~SlabContext() { release_all(); }

void SlabContext::release_all() noexcept {
    cudaSetDevice(dev_);
    if (s_comp_) cudaStreamSynchronize(s_comp_);
    if (s_comp2_) cudaStreamSynchronize(s_comp2_);
    if (s_prep_) cudaStreamSynchronize(s_prep_);
    if (s_aux_) cudaStreamSynchronize(s_aux_);
    if (s_copy_) cudaStreamSynchronize(s_copy_);
    if (s_d2h_) cudaStreamSynchronize(s_d2h_);
    for (auto e : ev_chunk_) if (e) cudaEventDestroy(e);
    for (auto e : ev_dchunk_) if (e) cudaEventDestroy(e);
    for (auto e : ev_band_) if (e) cudaEventDestroy(e);
    if (ev_band_pre_) cudaEventDestroy(ev_band_pre_);
    for (auto e : ev_ready_) if (e) cudaEventDestroy(e);
    for (auto e : ev_free_) if (e) cudaEventDestroy(e);
    for (auto e : ev_prep_) if (e) cudaEventDestroy(e);
    for (auto& p : launch_ev_) {
        if (p.first) cudaEventDestroy(p.first);
        if (p.second) cudaEventDestroy(p.second);
    }
    for (cudaEvent_t e : {ev_t0_, ev_t1_, ev_h0_, ev_h1_, ev_d0_, ev_d1_})
        if (e) cudaEventDestroy(e);
    if (s_comp_) cudaStreamDestroy(s_comp_);
    if (s_comp2_) cudaStreamDestroy(s_comp2_);
    if (ev_join_) cudaEventDestroy(ev_join_);
    if (s_prep_) cudaStreamDestroy(s_prep_);
    if (s_aux_) cudaStreamDestroy(s_aux_);
    if (s_copy_) cudaStreamDestroy(s_copy_);
    if (s_d2h_) cudaStreamDestroy(s_d2h_);
    if (own_vol_ && d_vol_) cudaFree(d_vol_);
    for (void* p : {(void*)d_ring_, (void*)d_ringx_, (void*)d_wx_, (void*)d_wy_, (void*)d_wz_,
                    (void*)d_cnt_})
        if (p) cudaFree(p);
    if (h_stage_) bph::pinned_free(h_stage_);
    if (h_bounce_) bph::pinned_free(h_bounce_);
    h_bounce_ = nullptr;
    s_comp_ = s_comp2_ = s_launch_ = s_prep_ = s_aux_ = s_copy_ = s_d2h_ = nullptr;
    ev_join_ = nullptr;
    d_vol_ = d_ring_ = nullptr;
    d_ringx_ = nullptr;
    d_wx_ = d_wy_ = d_wz_ = nullptr;
    d_cnt_ = nullptr;
    h_stage_ = nullptr;
    ev_chunk_.clear();
    ev_dchunk_.clear();
    ev_ready_.clear();
    ev_free_.clear();
    ev_prep_.clear();
    launch_ev_.clear();
    ev_t0_ = ev_t1_ = ev_h0_ = ev_h1_ = ev_d0_ = ev_d1_ = nullptr;
    cudaGetLastError();
}

void SlabContext::reset_recon() {
    pending_.clear();
    band_on_ = false;
    batch_index_ = 0;
    nb_ = 0;
    any_launch_ = false;
    t0_rec_ = false;
    any_h2d_ = false;
    views_ = 0;
    win_rows_ = 0;
    merge_ = 1;
    launches_ = 0;
    prep_launches_ = 0;
    h2d_bytes_ = 0;
    launch_ev_used_ = 0;
    wall_t0_ = 0.0;
}

void SlabContext::backproject(const float* image, const double* A, bool copy) {
    if (!image || !A) throw bph::config_error("null argument");
    bind();
    if (resident_ > 0) resident_ = 0;  // streaming reuses the slots
    if (views_ == 0) wall_t0_ = now_ms();
    bph::Mat m;
    std::memcpy(m.data(), A, sizeof(double) * 12);
    bph::validate_matrix_for_grid(m, grid_);

    if (nb_ == 0) {
        // a deferred batch still holding this ring group must be launched first
        while (std::any_of(pending_.begin(), pending_.end(),
                           [&](const Pending& p) { return p.rg == rg_; }))
            launch_pending_front();
        // the ring group (and its pinned staging) is reusable once the kernel
        // that last read it has finished
        if (used_[(size_t)rg_]) check(cudaEventSynchronize(ev_free_[(size_t)rg_]), "ring wait");
    }
    int r0 = 0, r1 = isy_;
    if (cfg_.row_windows)
        bph::row_window(m, grid_, 0, L_ - 1, 0, L_ - 1, z0_, z1_ - 1, isy_, &r0, &r1);
    if (filt_ && r1 > r0) {
        // the filter packs rows (2i, 2i+1) into one complex FFT; align the window
        // to that pairing so results do not depend on the window (or stale rows)
        r0 &= ~1;
        if (((r1 - r0) & 1) && r1 < isy_) ++r1;
    }
    const int slot = rg_ * B_ + nb_;
    // copy semantics (staging on the caller's thread) paces the views at host-copy speed,
    // and a withheld tail would then start uploading only after the last call: the band
    // tail is for zero-copy callers (e2e_copy 61 -> 63 ms with it)
    if (band_start_ >= 0 && views_ == 0) {  // this reconstruction's tail: by its first call
        const int t = copy ? band_tail_copy_ : band_tail_zc_;
        band_on_ = t > 0;
        tail_batches_ = band_on_ ? t : band_tail_zc_;
        if (band_on_) {
            const int nbatch = (cfg_.views + B_ - 1) / B_;
            band_start_ = std::max(0, nbatch - t) * B_;
        }
    }
    const bool withhold = band_on_ && views_ >= (uint64_t)band_start_;
    if (withhold) {
        band_img_[(size_t)slot] = nullptr;
        band_r0_[(size_t)slot] = band_r1_[(size_t)slot] = 0;
        band_m_[(size_t)slot] = m;
    }
    if (r1 > r0) {
        const float* src = image + (size_t)r0 * isx_;
        if (copy) {
            if (!h_stage_) {
                h_stage_ = static_cast<float*>(
                    bph::pinned_alloc((size_t)slots_ * isy_ * isx_ * sizeof(float)));
                // rows outside a view's window may ride along in a 2-D window run (never
                // read by any kernel); keep them finite
                std::memset(h_stage_, 0, (size_t)slots_ * isy_ * isx_ * sizeof(float));
            }
            float* stg = h_stage_ + (size_t)slot * isy_ * isx_ + (size_t)r0 * isx_;
            // the caller may reuse `image` when this returns: copy now, on several host
            // threads (a pageable source reads at a fraction of PCIe speed per thread)
            bph::parallel_memcpy(stg, src, (size_t)(r1 - r0) * isx_ * sizeof(float));
            src = stg;
        }
        float* dst = d_ring_ + (size_t)slot * isy_ * pitch_ + (size_t)r0 * pitch_;
        if (withhold) {
            // uploaded at finish in row bands (or view-major by upload_withheld)
            band_img_[(size_t)slot] = reinterpret_cast<const char*>(src) - (size_t)r0 * isx_ * sizeof(float);
            band_r0_[(size_t)slot] = r0;
            band_r1_[(size_t)slot] = r1;
        } else if (!any_h2d_) {
            check(cudaEventRecord(ev_h0_, s_copy_), "event");
            any_h2d_ = true;
        }
        if (withhold) {
        } else if (pitch_ == isx_) {
            // Views whose images are equally spaced in host memory (consecutive images of
            // one stack, or consecutive staging slots) and land in consecutive ring slots
            // form one copy: a plain copy when every window is the full detector, else ONE
            // 2-D copy of the run's union row window (height = views).  A z-slab's per-view
            // windows move with the view, so per-view ~1 MB copies reached only ~17 GB/s;
            // the union costs a few % more rows.  (tools/h2d_probe.py: >= 16 MB copies
            // run at ~55 GB/s.)
            const size_t view_bytes = (size_t)isx_ * isy_ * sizeof(float);
            const size_t win_bytes = (size_t)(r1 - r0) * isx_ * sizeof(float);
            const char* img = reinterpret_cast<const char*>(src) - (size_t)r0 * isx_ * sizeof(float);
            bool extend = run_n_ > 0 && img == run_img0_ + run_n_ * view_bytes &&
                          slot == run_slot0_ + run_n_;
            if (extend) {
                const int u0 = std::min(r0, run_r0_), u1 = std::max(r1, run_r1_);
                const size_t ubytes = (size_t)(u1 - u0) * isx_ * sizeof(float) * (run_n_ + 1);
                extend = ubytes <= run_limit_ &&
                         ubytes <= (size_t)(1.15 * (double)(run_actual_ + win_bytes)) + 4 * view_bytes / 16;
                if (extend) {
                    run_r0_ = u0;
                    run_r1_ = u1;
                    run_actual_ += win_bytes;
                    ++run_n_;
                }
            }
            if (!extend) {
                issue_run();
                run_img0_ = img;
                run_slot0_ = slot;
                run_n_ = 1;
                run_r0_ = r0;
                run_r1_ = r1;
                run_actual_ = win_bytes;
            }
        } else
            check(cudaMemcpy2DAsync(dst, (size_t)pitch_ * sizeof(float), src,
                                    (size_t)isx_ * sizeof(float), (size_t)isx_ * sizeof(float),
                                    (size_t)(r1 - r0), cudaMemcpyHostToDevice, s_copy_),
                  "H2D");
        if (!withhold) h2d_bytes_ += (uint64_t)(r1 - r0) * isx_ * sizeof(float);
    }
    win_rows_ += (uint64_t)std::max(0, r1 - r0);
    if (filt_) {
        fr0_[(size_t)nb_] = r1 > r0 ? r0 : 0;
        fr1_[(size_t)nb_] = r1 > r0 ? r1 : 0;
    }
    const auto f = bph::narrowed(m);
    std::memcpy(cur_.A[nb_], f.data(), sizeof(float) * 12);
    cur_.slot[nb_] = slot;
    ++nb_;
    ++views_;
    if (nb_ == B_) flush();
}

void SlabContext::choose_tile(const bpg::BatchArgs& b) {
    // the reference's approximate reciprocals (and the strict HW approximation) run on
    // the simple kernel; fast mode + BP_RECIP_HW_APPROX has a tiled variant
    const bool tiled_recip = cfg_.recip_mode == BP_RECIP_EXACT ||
                             (cfg_.recip_mode == BP_RECIP_HW_APPROX && !cfg_.strict_mode);
    if (cfg_.kernel == bpg::kKernelSimple || !tiled_recip) {
        tiled_ = false;
        return;
    }
    bpg::TileShape t{};
    if (!bpg::tile_shape_for(L_, &t)) {
        tiled_ = false;
        return;
    }
    // fast mode reads the pair ring where a pair variant exists
    t.dy = (!cfg_.strict_mode && pair_ok_ && bpg::has_pair_variant(t)) ? 1 : 0;
    // x-quads (one y-row of 4 x-voxels per thread) for the pair kernel: +0.85% at 512^3 in
    // round 1 (then -0.55% at 1024^3 and 2048^3); with the warp-parallel cull and the SHF
    // texel addresses of round 2 also +1.4% at 1024^3 and +1.2% at 2048^3 (A/B, BP_NO_XQ=1)
    if (t.dy && !std::getenv("BP_NO_XQ")) {
        bpg::TileShape q = t;
        q.xp = 2;
        if (bpg::has_pair_variant(q)) t.xp = 2;
    }
    // Sample the block lattice (including the outermost blocks, whose shadows
    // are the largest) for a few views of this batch; size the SMEM tile from
    // the largest footprint plus a guard.  Pairs that still do not fit are
    // served exactly by the in-kernel global-memory fallback.
    const int nbx = (L_ + t.bx - 1) / t.bx, nby = (L_ + t.by - 1) / t.by,
              nbz = (nz_ + t.bz - 1) / t.bz;
    auto samples = [](int n) {
        std::vector<int> s;
        const int k = std::min(n, 9);
        for (int i = 0; i < k; ++i) s.push_back(k == 1 ? 0 : (int)((long long)i * (n - 1) / (k - 1)));
        return s;
    };
    const auto sx = samples(nbx), sy = samples(nby), sz = samples(nbz);
    const int views[3] = {0, b.nviews / 2, b.nviews - 1};
    int need_w = 0, need_h = 0, need_w2 = 0;  // need_w2: pair ring (2-texel aligned origin)
    for (int vi = 0; vi < 3; ++vi) {
        const float* A = b.A[views[vi]];
        for (int zi : sz)
            for (int yi : sy)
                for (int xi : sx) {
                    double umin = 1e300, umax = -1e300, vmin = 1e300, vmax = -1e300, wmin = 1e300;
                    for (int c = 0; c < 8; ++c) {
                        const int x = xi * t.bx + ((c & 1) ? t.bx - 1 : 0);
                        const int y = yi * t.by + ((c & 2) ? t.by - 1 : 0);
                        const int z = z0_ + zi * t.bz + ((c & 4) ? t.bz - 1 : 0);
                        const double wx = (double)(float)grid_.wx(x), wy = (double)(float)grid_.wy(y),
                                     wz = (double)(float)grid_.wz(z);
                        const double uw = (double)A[0] * wx + (double)A[3] * wy + (double)A[6] * wz + (double)A[9];
                        const double vw = (double)A[1] * wx + (double)A[4] * wy + (double)A[7] * wz + (double)A[10];
                        const double w = (double)A[2] * wx + (double)A[5] * wy + (double)A[8] * wz + (double)A[11];
                        wmin = std::min(wmin, w);
                        umin = std::min(umin, uw / w);
                        umax = std::max(umax, uw / w);
                        vmin = std::min(vmin, vw / w);
                        vmax = std::max(vmax, vw / w);
                    }
                    if (!(wmin > 0) || std::fabs(umin) > 1e6 || std::fabs(umax) > 1e6 ||
                        std::fabs(vmin) > 1e6 || std::fabs(vmax) > 1e6)
                        continue;
                    const int iu0 = ((int)std::floor(umin) - 1) & ~3;  // 16 B aligned origin
                    const int iu1 = (int)std::floor(umax) + 2;
                    const int iv0 = (int)std::floor(vmin) - 1, iv1 = (int)std::floor(vmax) + 2;
                    if (iu1 < 0 || iu0 > isx_ - 1 || iv1 < 0 || iv0 > isy_ - 1) continue;
                    need_w = std::max(need_w, iu1 - iu0 + 1);
                    need_w2 = std::max(need_w2, iu1 - (((int)std::floor(umin) - 1) & ~1) + 1);
                    need_h = std::max(need_h, iv1 - iv0 + 1);
                }
    }
    // Row pitch of the SMEM tile == TMA box width.  Pitches == 20 (mod 32) floats
    // minimise bank conflicts of the raw tile's 8x4 lane layout (tools/bank_sim.py),
    // == 8 (mod 16) 8-byte texels those of the pair ring (tools/bank_sim64.py).
    // The kernel checks every (block, view) footprint exactly and serves the rare one
    // that does not fit through the exact global-memory fallback, so the pitch needs
    // no guard beyond the TMA alignment.  (A guard that pushed the pair ring past its
    // compile-time 152 forced a taller ring than two CTAs per SM hold: -25%, measured.)
    int tw = t.dy ? round_up(std::max(need_w2, 8), 2) : round_up(std::max(need_w, 8) + 4, 4);
    const bool twc_ok = !std::getenv("BP_NO_TWC") && t.bx >= 32;
    // compile-time pitches (== 16 mod 32: immediate row offsets, low conflicts); the
    // smallest listed one that holds the footprint
    int twcs[3] = {0, 0, 0};
    if (t.dy) {
        twcs[0] = 152;  // 8-byte texels, == 8 (mod 16): lowest simulated conflicts
    } else if (t.bx == 64) {
        twcs[0] = 240;
    } else if (t.by == 32) {
        twcs[0] = 176;  // narrower 112 at 1024^3 measured 0.9% slower (A/B)
    } else {
        twcs[0] = 144;
    }
    int twc = 0;
    for (int c : twcs)
        if (c > 0 && tw <= c) { twc = c; break; }
    if (const char* e = std::getenv("BP_TWC")) twc = std::atoi(e);
    if (twc_ok && twc > 0 && tw <= twc) {
        tw = twc;
    } else if (t.dy) {
        tw = round_up(tw, 8);
        if (tw % 16 != 8) tw += 8;
    } else if (tw % 32 != 20) {
        const int t2 = tw + ((20 - tw % 32) + 32) % 32;
        if (t2 <= 256) tw = t2;
    }
    int th = round_up(std::max(need_h, 8) + 8, 8);  // rows of the largest tile (+ guard)
    tw = std::min(tw, 256);
    if (tiled_ && tw <= ts_.tw && th <= ts_.th) return;
    if (tiled_) {
        tw = std::max(tw, ts_.tw);
        th = std::max(th, ts_.th);
    }
    // The tile rows live in a ring shared by the in-flight views; size it to the
    // SMEM of `ctas` CTAs per SM (3 for the 288-thread 512^3+ variant).
    t.tw = tw;
    int ctas = (t.bx * t.by * t.bz == 4096) ? 3 : 4;
    if (t.bx == 32 && t.by == 16 && t.bz == 4) ctas = 5;
    if ((t.bx == 32 && t.by == 32 && t.bz == 8) || t.bx == 64) ctas = 2;
    if (t.bx == 16 && t.by == 32) ctas = 4;
    if (const char* e = std::getenv("BP_CTAS")) ctas = std::max(1, std::atoi(e));
    // Prefer `ctas` CTAs per SM: the ring takes what their SMEM leaves, unless that
    // cannot hold the largest sampled footprint (taller views use the fallback).
    const int budget = bpg::ring_rows_for_shape(t, 0, ctas);
    t.th = budget >= round_up(std::max(need_h, 8), 8) ? budget : bpg::ring_rows_for_shape(t, th, ctas);
    t.smem_bytes = bpg::smem_bytes_for(t);
    if (t.smem_bytes > 227 * 1024) throw bph::device_error("tile ring exceeds shared memory");
    char err[256];
    if (bpg::encode_ring_tmap(tmap_, d_ring_, isx_, isy_, pitch_, slots_, t, err, sizeof err) != 0)
        throw bph::device_error(err);
    if (t.dy) {
        if (!d_ringx_) {
            const size_t n = (size_t)slots_ * (isy_ + 1) * pitch_;
            check(cudaMalloc(&d_ringx_, n * sizeof(float2)), "cudaMalloc(pair ring)");
        }
        if (bpg::encode_pair_tmap(tmapx_, d_ringx_, isx_, isy_, pitch_, slots_, t, err, sizeof err) != 0)
            throw bph::device_error(err);
    }
    ts_ = t;
    tiled_ = true;
}

void SlabContext::launch(const bpg::BatchArgs& b, int zc0, int zc1, bool final_pass) {
    if (zc1 < 0) zc1 = nz_;
    bpg::SlabArgs s{};
    s.vol = d_vol_ + (size_t)zc0 * L_ * L_;
    // the last batch of a reconstruction stores its results straight into the output
    // volume when one is configured (fused gather over NVLink / CUDA IPC)
    s.vol_out = (final_pass && out_vol_) ? out_vol_ + (size_t)zc0 * L_ * L_ : nullptr;
    s.proj = d_ring_;
    s.wx = d_wx_;
    s.wy = d_wy_;
    s.wz = d_wz_;
    s.counters = d_cnt_;
    s.L = L_;
    s.z0 = z0_ + zc0;
    s.nz = zc1 - zc0;
    s.isx = isx_;
    s.isy = isy_;
    s.pitch = pitch_;
    if (const char* d = std::getenv("BP_DEBUG")) s.debug = std::atoi(d);
    if (tiled_) {
        s.nbx = (L_ + ts_.bx - 1) / ts_.bx;
        s.nby = (L_ + ts_.by - 1) / ts_.by;
        s.nbz = (s.nz + ts_.bz - 1) / ts_.bz;
    }
    if (cfg_.count_visible) check((cudaError_t)bpg::launch_clip_count(s, b, s_launch_), "clip count");
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    if (cfg_.profile_launches) {
        if (launch_ev_used_ == launch_ev_.size()) {
            cudaEvent_t a, c;
            check(cudaEventCreate(&a), "event");
            check(cudaEventCreate(&c), "event");
            launch_ev_.emplace_back(a, c);
        }
        e0 = launch_ev_[launch_ev_used_].first;
        e1 = launch_ev_[launch_ev_used_].second;
        ++launch_ev_used_;
        check(cudaEventRecord(e0, s_launch_), "event");
    }
    int rc;
    if (tiled_)
        rc = bpg::launch_tiled(ts_.dy ? tmapx_ : tmap_, s, b, ts_, cfg_.strict_mode != 0,
                               cfg_.distance_weight != 0, cfg_.recip_mode == BP_RECIP_HW_APPROX, s_launch_);
    else
        rc = bpg::launch_simple(s, b, cfg_.distance_weight != 0, cfg_.recip_mode, s_launch_);
    check((cudaError_t)rc, "backprojection kernel launch");
    if (e1) check(cudaEventRecord(e1, s_launch_), "event");
    ++launches_;
}

void SlabContext::launch_pending_front(bool final_pass) {
    Pending p = pending_.front();
    pending_.erase(pending_.begin());
    if (p.band) upload_withheld(p);
    prepare(p);
    check(cudaStreamWaitEvent(s_comp_, p.ready, 0), "wait");
    mark_t0();
    p.b.load_volume = p.index > 0 ? 1 : 0;
    launch(p.b, 0, -1, final_pass);
    any_launch_ = true;
    check(cudaEventRecord(ev_free_[(size_t)p.rg], s_comp_), "event");
    used_[(size_t)p.rg] = true;
}

// The first n pending batches as ONE launch (n * B_ <= kMaxBatch): one volume read-modify-write
// and fuller waves instead of n.  Ascending view order per voxel is kept, so results are
// unchanged bit for bit.
void SlabContext::launch_pending_group(int n, bool final_pass) {
    n = std::min(n, (int)pending_.size());
    if (n <= 1) {
        launch_pending_front(final_pass);
        return;
    }
    std::vector<Pending> g(pending_.begin(), pending_.begin() + n);
    pending_.erase(pending_.begin(), pending_.begin() + n);
    bpg::BatchArgs b = g.front().b;
    b.nviews = 0;
    for (auto& p : g) {
        if (p.band) upload_withheld(p);
        prepare(p);
        check(cudaStreamWaitEvent(s_comp_, p.ready, 0), "wait");
        for (int i = 0; i < p.b.nviews; ++i) {
            b.slot[b.nviews] = p.b.slot[i];
            std::memcpy(b.A[b.nviews], p.b.A[i], sizeof(float) * 12);
            ++b.nviews;
        }
    }
    mark_t0();
    b.load_volume = g.front().index > 0 ? 1 : 0;
    launch(b, 0, -1, final_pass);
    any_launch_ = true;
    for (const auto& p : g) {
        check(cudaEventRecord(ev_free_[(size_t)p.rg], s_comp_), "event");
        used_[(size_t)p.rg] = true;
    }
}

// View-major batches are launched `merge_` at a time when the slab's compute per view outlasts
// its upload per view (z-slabs of a multi-GPU split, whole volumes of 1024^3 and more): the
// first batch alone, so the GPU starts as early as it can, then groups.  Waiting for a group's
// last batch costs nothing there, because the uploads run far ahead of the kernels.
void SlabContext::launch_ready() {
    const int avail = (int)pending_.size() - tail_batches_;
    if (avail <= 0) return;
    const int hold = std::max(0, std::min(merge_ - 1, R_ - 2 - tail_batches_));
    if (!any_launch_ || hold == 0) {
        while ((int)pending_.size() > tail_batches_) launch_pending_front();
        return;
    }
    if (avail > hold) launch_pending_group(avail);
}

void SlabContext::issue_run() {
    if (run_n_ == 0) return;
    const size_t row = (size_t)isx_ * sizeof(float);
    const size_t view_bytes = row * isy_;
    char* dst = reinterpret_cast<char*>(d_ring_ + (size_t)run_slot0_ * isy_ * pitch_) + (size_t)run_r0_ * row;
    const char* src = run_img0_ + (size_t)run_r0_ * row;
    const size_t width = (size_t)(run_r1_ - run_r0_) * row;
    if (width == view_bytes || run_n_ == 1)  // contiguous: full windows, or one view
        check(cudaMemcpyAsync(dst, src, width + (size_t)(run_n_ - 1) * view_bytes,
                              cudaMemcpyHostToDevice, s_copy_), "H2D");
    else
        check(cudaMemcpy2DAsync(dst, view_bytes, src, view_bytes, width, (size_t)run_n_,
                                cudaMemcpyHostToDevice, s_copy_), "H2D (2-D window run)");
    run_n_ = 0;
}

void SlabContext::copy_rows(const Pending& p, int r0, int r1) {
    if (r1 <= r0) return;
    const size_t row = (size_t)isx_ * sizeof(float), view_bytes = row * isy_;
    const size_t slot_bytes = (size_t)isy_ * pitch_ * sizeof(float);
    if (!any_h2d_) {
        check(cudaEventRecord(ev_h0_, s_copy_), "event");
        any_h2d_ = true;
    }
    int i = 0;
    while (i < p.b.nviews) {
        const int s0 = p.b.slot[i];
        const char* img0 = band_img_[(size_t)s0];
        if (!img0) {
            ++i;
            continue;
        }
        // a run of views equally spaced in host memory in consecutive slots: one 2-D copy
        int n = 1;
        while (pitch_ == isx_ && i + n < p.b.nviews && p.b.slot[i + n] == s0 + n &&
               band_img_[(size_t)(s0 + n)] == img0 + (size_t)n * view_bytes)
            ++n;
        char* dst = reinterpret_cast<char*>(d_ring_) + (size_t)s0 * slot_bytes + (size_t)r0 * pitch_ * sizeof(float);
        const char* src = img0 + (size_t)r0 * row;
        if (pitch_ == isx_)
            check(cudaMemcpy2DAsync(dst, slot_bytes, src, view_bytes, (size_t)(r1 - r0) * row, (size_t)n,
                                    cudaMemcpyHostToDevice, s_copy_),
                  "H2D (row band)");
        else
            check(cudaMemcpy2DAsync(dst, (size_t)pitch_ * sizeof(float), src, row, row, (size_t)(r1 - r0),
                                    cudaMemcpyHostToDevice, s_copy_),
                  "H2D (row band)");
        h2d_bytes_ += (uint64_t)(r1 - r0) * row * n;
        i += n;
    }
}

void SlabContext::upload_withheld(Pending& p) {
    if (!p.band) return;
    Pending one = p;
    for (int i = 0; i < p.b.nviews; ++i) {
        const int sl = p.b.slot[i];
        if (!band_img_[(size_t)sl]) continue;
        one.b.nviews = 1;
        one.b.slot[0] = sl;
        copy_rows(one, band_r0_[(size_t)sl], band_r1_[(size_t)sl]);
        band_img_[(size_t)sl] = nullptr;
    }
    check(cudaEventRecord(ev_ready_[(size_t)p.rg], s_copy_), "event");
    p.band = false;
    p.ready = nullptr;
}

void SlabContext::band_tail(float* host_volume, std::vector<std::pair<size_t, size_t>>& chunks) {
    // z-chunks on block layers; each one's union row window over the tail's views
    const int C = std::max(1, std::min(band_chunks_, nz_ / ts_.bz));
    std::vector<int> zb((size_t)C + 1);
    for (int c = 0; c <= C; ++c) zb[(size_t)c] = (int)((long long)nz_ * c / C / ts_.bz) * ts_.bz;
    zb[(size_t)C] = nz_;
    std::vector<int> lo((size_t)C, isy_), hi((size_t)C, 0);
    for (const auto& p : pending_)
        for (int i = 0; i < p.b.nviews; ++i) {
            const int sl = p.b.slot[i];
            if (!band_img_[(size_t)sl]) continue;
            for (int c = 0; c < C; ++c) {
                int r0 = 0, r1 = 0;
                bph::row_window(band_m_[(size_t)sl], grid_, 0, L_ - 1, 0, L_ - 1, z0_ + zb[(size_t)c],
                                z0_ + zb[(size_t)c + 1] - 1, isy_, &r0, &r1);
                // never beyond the view's own (slab) window, which is all that is staged
                r0 = std::max(r0, band_r0_[(size_t)sl]);
                r1 = std::min(r1, band_r1_[(size_t)sl]);
                if (r1 > r0) {
                    lo[(size_t)c] = std::min(lo[(size_t)c], r0);
                    hi[(size_t)c] = std::max(hi[(size_t)c], r1);
                }
            }
        }
    // FDK filtering (cfg_.filter) transforms rows (2i, 2i+1) as one complex FFT: band runs
    // then consist of whole row pairs, so filtering band by band equals filtering whole views
    if (filt_)
        for (int c = 0; c < C; ++c)
            if (hi[(size_t)c] > lo[(size_t)c]) {
                lo[(size_t)c] &= ~1;
                hi[(size_t)c] = std::min(isy_, (hi[(size_t)c] + 1) & ~1);
            }
    // outside in: chunks whose rows lie farthest from the detector centre complete first,
    // so their compute and D2H run while the inner bands are still uploading
    std::vector<int> order((size_t)C);
    for (int c = 0; c < C; ++c) order[(size_t)c] = c;
    auto dist = [&](int c) {
        if (hi[(size_t)c] <= lo[(size_t)c]) return 1e30;  // reads no rows: first
        return std::fabs(0.5 * (lo[(size_t)c] + hi[(size_t)c]) - 0.5 * isy_);
    };
    std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return dist(a) > dist(b); });
    // the tail's batches as ONE launch per chunk (ascending view order is kept): one volume
    // read-modify-write per chunk instead of one per batch, and fewer, fuller waves
    int total = 0;
    for (const auto& p : pending_) total += p.b.nviews;
    std::vector<Pending> tail;
    if (total <= bpg::kMaxBatch) {
        Pending m = pending_.front();
        m.b.nviews = 0;
        for (const auto& p : pending_)
            for (int i = 0; i < p.b.nviews; ++i) {
                m.b.slot[m.b.nviews] = p.b.slot[i];
                std::memcpy(m.b.A[m.b.nviews], p.b.A[i], sizeof(float) * 12);
                ++m.b.nviews;
            }
        tail.push_back(m);
    } else {
        tail = pending_;
    }
    // Pair rows (fast mode) are built on the prep stream as soon as their raw rows are in,
    // each exactly once: pair row e = (p[e-1], p[e] - p[e-1]) (p[-1] = p[isy] = 0) is
    // built when both raw rows are uploaded.  A voxel at texel row iv reads pair row iv+1,
    // and a chunk's window holds every in-detector row its voxels read, so every pair row
    // a chunk reads is built by its own band or an earlier one -- and none is ever
    // rewritten while a kernel reads it.
    const bool expd = tiled_ && ts_.dy;
    const bool trace = std::getenv("BP_BAND_TRACE") != nullptr;
    if (trace) check(cudaEventRecord(ev_band_pre_, s_copy_), "event");
    std::vector<char> up((size_t)isy_, 0), built((size_t)isy_ + 1, 0);
    auto raw_in = [&](int r) { return r < 0 || r >= isy_ || up[(size_t)r]; };
    std::vector<std::pair<int, int>> runs;  // this band's newly uploaded rows
    for (int k = 0; k < C; ++k) {
        const int c = order[(size_t)k];
        int r = lo[(size_t)c];
        while (r < hi[(size_t)c]) {  // the window's rows not uploaded yet, as runs
            if (up[(size_t)r]) {
                ++r;
                continue;
            }
            int e = r;
            while (e < hi[(size_t)c] && !up[(size_t)e]) up[(size_t)e++] = 1;
            for (const auto& p : pending_) copy_rows(p, r, e);
            runs.emplace_back(r, e);
            r = e;
        }
        check(cudaEventRecord(ev_band_[(size_t)k], s_copy_), "event");
        if (filt_ && !runs.empty()) {  // the band's new rows, filtered in place
            mark_t0();
            check(cudaStreamWaitEvent(s_aux_, ev_t0_, 0), "wait");
            check(cudaStreamWaitEvent(s_aux_, ev_band_[(size_t)k], 0), "wait");
            for (const auto& run : runs)
                for (const auto& p : tail) {
                    std::array<int, bpg::kMaxBatch> r0s{}, r1s{};
                    for (int i = 0; i < p.b.nviews; ++i) {
                        r0s[(size_t)i] = run.first;
                        r1s[(size_t)i] = run.second;
                    }
                    filt_->apply_batch(d_ring_, (long long)isy_ * pitch_, pitch_, p.b.nviews, p.b.slot,
                                       r0s.data(), r1s.data(), s_aux_);
                    ++prep_launches_;
                }
            runs.clear();
            check(cudaEventRecord(ev_band_[(size_t)k], s_aux_), "event");
        }
        runs.clear();
        if (expd) {
            // on the highest-priority stream: the prep stream may still hold the expansions
            // of the last view-major batches (measured: 3.8 ms of lag behind the copies)
            mark_t0();
            check(cudaStreamWaitEvent(s_aux_, ev_t0_, 0), "wait");
            check(cudaStreamWaitEvent(s_aux_, ev_band_[(size_t)k], 0), "wait");
            int e = 0;
            while (e <= isy_) {  // runs of pair rows that just became buildable
                if (built[(size_t)e] || !raw_in(e - 1) || !raw_in(e)) {
                    ++e;
                    continue;
                }
                int f = e;
                while (f <= isy_ && !built[(size_t)f] && raw_in(f - 1) && raw_in(f)) built[(size_t)f++] = 1;
                for (const auto& p : tail) {
                    bpg::ExpandArgs a{};
                    a.ring = d_ring_;
                    a.ringx = d_ringx_;
                    a.isx = isx_;
                    a.isy = isy_;
                    a.pitch = pitch_;
                    a.pitchx = pitch_;
                    a.e0 = e;
                    a.e1 = f;
                    for (int i = 0; i < p.b.nviews; ++i) a.slot[i] = p.b.slot[i];
                    check((cudaError_t)bpg::launch_expand(a, p.b.nviews, s_aux_), "pair ring expansion (band)");
                    ++prep_launches_;
                }
                e = f;
            }
            // the chunk's kernels wait on this (its band, and the pair rows built so far)
            check(cudaEventRecord(ev_band_[(size_t)k], s_aux_), "event");
        }
    }
    mark_t0();
    // The z-chunks are independent of one another, so they alternate between two compute
    // streams: the next chunk's blocks fill the SMs that the current chunk's last wave leaves
    // idle (on one stream every chunk ended in a partly filled wave).
    // Only where the tail is compute-bound (merge_ > 1, see flush): with the uploads still
    // running (512^3 on one GPU) a chunk must finish as early as it can for its readback to
    // fit under them, and sharing the SMs with its successor delayed it (48.9 -> 55.6 ms).
    const bool two = !std::getenv("BP_NO_CHUNK_OVERLAP") && C > 1 && merge_ > 1;
    if (two) {  // the second stream starts after the view-major launches
        check(cudaEventRecord(ev_join_, s_comp_), "event");
        check(cudaStreamWaitEvent(s_comp2_, ev_join_, 0), "wait");
    }
    for (int k = 0; k < C; ++k) {
        const int c = order[(size_t)k];
        s_launch_ = (two && (k & 1)) ? s_comp2_ : s_comp_;
        check(cudaStreamWaitEvent(s_launch_, ev_band_[(size_t)k], 0), "wait");
        for (size_t i = 0; i < tail.size(); ++i) {
            auto p = tail[i];
            p.b.load_volume = p.index > 0 ? 1 : 0;
            launch(p.b, zb[(size_t)c], zb[(size_t)c + 1], i + 1 == tail.size());
        }
        check(cudaEventRecord(ev_chunk_[(size_t)k], s_launch_), "event");
        check(cudaStreamWaitEvent(s_d2h_, ev_chunk_[(size_t)k], 0), "wait");
        if (k == 0) check(cudaEventRecord(ev_d0_, s_d2h_), "event");
        const size_t off = (size_t)zb[(size_t)c] * L_ * L_;
        const size_t n = (size_t)(zb[(size_t)c + 1] - zb[(size_t)c]) * L_ * L_;
        check(cudaMemcpyAsync(host_volume + off, result() + off, n * sizeof(float), cudaMemcpyDefault, s_d2h_),
              "D2H");
        check(cudaEventRecord(ev_dchunk_[(size_t)k], s_d2h_), "event");
        chunks.emplace_back(off, n);
    }
    s_launch_ = s_comp_;
    if (two) {  // whatever follows on the compute stream follows both
        check(cudaEventRecord(ev_join_, s_comp2_), "event");
        check(cudaStreamWaitEvent(s_comp_, ev_join_, 0), "wait");
    }
    for (const auto& p : pending_)
        for (int i = 0; i < p.b.nviews; ++i) band_img_[(size_t)p.b.slot[i]] = nullptr;
    if (trace) {  // diagnostics: per chunk, ms after the first H2D
        check(cudaDeviceSynchronize(), "sync");
        auto ms = [&](cudaEvent_t e) {
            float t = 0;
            return cudaEventElapsedTime(&t, ev_h0_, e) == cudaSuccess ? t : -1.0f;
        };
        std::fprintf(stderr, "band tail: %d views of %d batches; view-major uploads done %7.2f\n", total,
                     (int)pending_.size(), ms(ev_band_pre_));
        for (int k = 0; k < C; ++k) {
            const int c = order[(size_t)k];
            std::fprintf(stderr, "band chunk %2d z[%4d,%4d) rows[%4d,%4d): uploaded %7.2f computed %7.2f read back %7.2f\n",
                         k, zb[(size_t)c], zb[(size_t)c + 1], lo[(size_t)c], hi[(size_t)c], ms(ev_band_[(size_t)k]),
                         ms(ev_chunk_[(size_t)k]), ms(ev_dchunk_[(size_t)k]));
        }
    }
}

void SlabContext::flush() {
    if (nb_ == 0) return;
    issue_run();  // every copy of the batch precedes its ready event
    cur_.nviews = nb_;
    choose_tile(cur_);
    check(cudaEventRecord(ev_ready_[(size_t)rg_], s_copy_), "event");
    pending_.push_back(Pending{cur_, rg_, batch_index_++, fr0_, fr1_});
    // band_start_ is batch-aligned: a batch is withheld whole or not at all
    pending_.back().band = band_on_ && views_ - (uint64_t)nb_ >= (uint64_t)band_start_;
    if (!pending_.back().band) prepare(pending_.back());
    if (pending_.back().index == 0) {
        // compute-bound or upload-bound?  per view: the slab's voxels at ~1.5e12 updates/s
        // against the batch's row window at ~55 GB/s
        const double t_comp = (double)nz_ * L_ * L_ / 1.5e12;
        const double t_up = (double)std::max<uint64_t>(1, win_rows_ / std::max<uint64_t>(1, views_)) * isx_ *
                            sizeof(float) / 55e9;
        merge_ = (tiled_ && t_comp > 3.0 * t_up) ? std::max(1, std::min(3, bpg::kMaxBatch / B_)) : 1;
        if (const char* e = std::getenv("BP_MERGE"))
            merge_ = std::max(1, std::min(std::atoi(e), bpg::kMaxBatch / B_));
    }
    rg_ = (rg_ + 1) % R_;
    nb_ = 0;
    launch_ready();
}

void SlabContext::finish(float* host_volume, bp_gpu_stats* st) {
    bind();
    if (views_ == 0) wall_t0_ = now_ms();
    flush();
    // view-major batches still held for a merged launch
    while ((int)pending_.size() > tail_batches_)
        launch_pending_group(std::min(merge_, (int)pending_.size() - tail_batches_));
    const size_t vbytes = (size_t)nz_ * L_ * L_ * sizeof(float);
    bool d2h_done = false;
    // a pageable destination is read back through a pinned bounce buffer, each z-chunk
    // copied out by the host thread pool as soon as its D2H lands
    float* const dest = host_volume;
    const bool bounce = host_volume && bph::is_pageable(host_volume);
    if (bounce) {
        if (!h_bounce_ || bounce_bytes_ < vbytes) {
            if (h_bounce_) bph::pinned_free(h_bounce_);
            h_bounce_ = static_cast<float*>(bph::pinned_alloc(vbytes));
            bounce_bytes_ = vbytes;
        }
        host_volume = h_bounce_;
    }
    std::vector<std::pair<size_t, size_t>> chunks;  // (offset, count) of the D2H copies
    const int tail_chunks = bounce ? bounce_chunks_ : tail_chunks_;
    const bool band = host_volume && tiled_ && !pending_.empty() && nz_ >= 2 * ts_.bz &&
                      std::all_of(pending_.begin(), pending_.end(), [](const Pending& p) { return p.band; });
    if (!band)
        for (auto& p : pending_) upload_withheld(p);
    if (band) {
        band_tail(host_volume, chunks);
        any_launch_ = true;
        for (const auto& p : pending_) {
            check(cudaEventRecord(ev_free_[(size_t)p.rg], s_comp_), "event");
            used_[(size_t)p.rg] = true;
        }
        pending_.clear();
        check(cudaEventRecord(ev_t1_, s_comp_), "event");
        check(cudaEventRecord(ev_d1_, s_d2h_), "event");
        d2h_done = true;
    } else if (host_volume && !pending_.empty() && tiled_ && tail_chunks > 1 && nz_ >= 2 * ts_.bz) {
        // chunk-major tail: for each z-chunk run all deferred batches (ascending
        // view order per voxel is preserved), then stream that chunk back while the
        // next chunk computes
        const int C = std::min(tail_chunks, nz_ / ts_.bz);
        std::vector<int> zb((size_t)C + 1);
        for (int c = 0; c <= C; ++c) zb[(size_t)c] = (int)((long long)nz_ * c / C / ts_.bz) * ts_.bz;
        zb[(size_t)C] = nz_;
        for (auto& p : pending_) {
            prepare(p);
            check(cudaStreamWaitEvent(s_comp_, p.ready, 0), "wait");
        }
        mark_t0();
        for (int c = 0; c < C; ++c) {
            for (size_t i = 0; i < pending_.size(); ++i) {
                auto p = pending_[i];
                p.b.load_volume = p.index > 0 ? 1 : 0;
                launch(p.b, zb[(size_t)c], zb[(size_t)c + 1], i + 1 == pending_.size());
            }
            check(cudaEventRecord(ev_chunk_[(size_t)c], s_comp_), "event");
            check(cudaStreamWaitEvent(s_d2h_, ev_chunk_[(size_t)c], 0), "wait");
            if (c == 0) check(cudaEventRecord(ev_d0_, s_d2h_), "event");
            const size_t off = (size_t)zb[(size_t)c] * L_ * L_;
            const size_t n = (size_t)(zb[(size_t)c + 1] - zb[(size_t)c]) * L_ * L_;
            check(cudaMemcpyAsync(host_volume + off, result() + off, n * sizeof(float),
                                  cudaMemcpyDefault, s_d2h_),
                  "D2H");
            check(cudaEventRecord(ev_dchunk_[(size_t)c], s_d2h_), "event");
            chunks.emplace_back(off, n);
        }
        any_launch_ = true;
        for (const auto& p : pending_) {
            check(cudaEventRecord(ev_free_[(size_t)p.rg], s_comp_), "event");
            used_[(size_t)p.rg] = true;
        }
        pending_.clear();
        check(cudaEventRecord(ev_t1_, s_comp_), "event");
        check(cudaEventRecord(ev_d1_, s_d2h_), "event");
        d2h_done = true;
    } else {
        while (!pending_.empty()) launch_pending_front(pending_.size() == 1);
        if (!any_launch_) {
            mark_t0();
            check(cudaMemsetAsync(result(), 0, vbytes, s_comp_), "memset");
        }
        check(cudaEventRecord(ev_t1_, s_comp_), "event");
    }
    if (any_h2d_) check(cudaEventRecord(ev_h1_, s_copy_), "event");
    if (host_volume && !d2h_done) {
        check(cudaEventRecord(ev_d0_, s_comp_), "event");
        check(cudaMemcpyAsync(host_volume, result(), vbytes, cudaMemcpyDefault, s_comp_), "D2H");
        check(cudaEventRecord(ev_d1_, s_comp_), "event");
        check(cudaEventRecord(ev_dchunk_[0], s_comp_), "event");
        chunks.emplace_back(0, vbytes / sizeof(float));
    }
    if (bounce)
        for (size_t c = 0; c < chunks.size(); ++c) {
            check(cudaEventSynchronize(ev_dchunk_[c]), "D2H chunk");
            bph::parallel_memcpy(dest + chunks[c].first, h_bounce_ + chunks[c].first,
                                 chunks[c].second * sizeof(float));
        }
    unsigned long long cnt[8] = {0};
    check(cudaMemcpyAsync(cnt, d_cnt_, sizeof cnt, cudaMemcpyDeviceToHost, s_comp_), "counters");
    check(cudaMemsetAsync(d_cnt_, 0, sizeof cnt, s_comp_), "counters");
    check(cudaStreamSynchronize(s_copy_), "sync");
    check(cudaStreamSynchronize(s_comp_), "sync");
    check(cudaStreamSynchronize(s_d2h_), "sync");
    if (st) {
        std::memset(st, 0, sizeof *st);
        st->wall_ms = now_ms() - wall_t0_;
        float ms = 0;
        check(cudaEventElapsedTime(&ms, ev_t0_, ev_t1_), "elapsed");
        st->device_ms = ms;
        if (any_h2d_) {
            check(cudaEventElapsedTime(&ms, ev_h0_, ev_h1_), "elapsed");
            st->h2d_ms = ms;
        }
        if (host_volume) {
            check(cudaEventElapsedTime(&ms, ev_d0_, ev_d1_), "elapsed");
            st->d2h_ms = ms;
            st->d2h_bytes = vbytes;
        }
        double kms = 0;
        for (size_t i = 0; i < launch_ev_used_; ++i) {
            check(cudaEventElapsedTime(&ms, launch_ev_[i].first, launch_ev_[i].second), "elapsed");
            kms += ms;
        }
        st->kernel_ms = kms;
        st->views = views_;
        st->launches = launches_;
        st->prep_launches = prep_launches_;
        st->nominal_updates = views_ * (uint64_t)nz_ * L_ * L_;
        st->visible_updates = cnt[3];
        st->tile_pairs = cnt[0];
        st->skipped_pairs = cnt[1];
        st->fallback_pairs = cnt[2];
        st->h2d_bytes = h2d_bytes_;
        st->tile_w = tiled_ ? ts_.tw : 0;
        st->tile_h = tiled_ ? ts_.th : 0;
        st->block_x = tiled_ ? ts_.bx : 1;
        st->block_y = tiled_ ? ts_.by : 1;
        st->block_z = tiled_ ? ts_.bz : 1;
    }
    reset_recon();
}

void SlabContext::read_lines(const int* ys, const int* zs, int n, float* out) {
    if (!ys || !zs || !out || n < 0) throw bph::config_error("null argument");
    bind();
    check(cudaStreamSynchronize(s_comp_), "sync");
    for (int i = 0; i < n; ++i) {
        if (ys[i] < 0 || ys[i] >= L_ || zs[i] < z0_ || zs[i] >= z1_)
            throw bph::config_error("line outside the slab");
        const float* src = result() + ((size_t)(zs[i] - z0_) * L_ + ys[i]) * L_;
        check(cudaMemcpyAsync(out + (size_t)i * L_, src, (size_t)L_ * sizeof(float),
                              cudaMemcpyDeviceToHost, s_comp_),
              "D2H line");
    }
    check(cudaStreamSynchronize(s_comp_), "sync");
}

void SlabContext::clip_table(const double* mats, int count, uint16_t* host_ranges,
                             uint64_t* total) {
    if (!mats || count < 1) throw bph::config_error("null argument");
    if (z0_ != 0 || z1_ != L_) throw bph::config_error("clip tables cover the whole grid");
    if (L_ > 65535) throw bph::config_error("clip table supports at most 65535 voxels per edge");
    bind();
    const size_t n = (size_t)2 * count * L_ * L_;
    uint16_t* d = nullptr;
    check(cudaMalloc(&d, n * sizeof(uint16_t)), "cudaMalloc(clip table)");
    bpg::SlabArgs s{};
    s.wx = d_wx_;
    s.wy = d_wy_;
    s.wz = d_wz_;
    s.counters = d_cnt_;
    s.L = L_;
    s.z0 = 0;
    s.nz = L_;
    s.isx = isx_;
    s.isy = isy_;
    check(cudaMemsetAsync(d_cnt_, 0, 8 * sizeof(unsigned long long), s_comp_), "memset");
    for (int k0 = 0; k0 < count; k0 += bpg::kMaxBatch) {
        bpg::BatchArgs b{};
        b.nviews = std::min(bpg::kMaxBatch, count - k0);
        for (int i = 0; i < b.nviews; ++i) {
            bph::Mat m;
            std::memcpy(m.data(), mats + 12 * (size_t)(k0 + i), sizeof(double) * 12);
            bph::validate_matrix_for_grid(m, grid_);
            const auto f = bph::narrowed(m);
            std::memcpy(b.A[i], f.data(), sizeof(float) * 12);
        }
        check((cudaError_t)bpg::launch_clip_ranges(s, b, d, k0, s_comp_), "clip ranges");
        check((cudaError_t)bpg::launch_clip_count(s, b, s_comp_), "clip count");
    }
    unsigned long long cnt[8] = {0};
    check(cudaMemcpyAsync(cnt, d_cnt_, sizeof cnt, cudaMemcpyDeviceToHost, s_comp_), "counters");
    if (host_ranges)
        check(cudaMemcpyAsync(host_ranges, d, n * sizeof(uint16_t), cudaMemcpyDeviceToHost, s_comp_),
              "D2H clip table");
    check(cudaMemsetAsync(d_cnt_, 0, sizeof cnt, s_comp_), "memset");
    check(cudaStreamSynchronize(s_comp_), "sync");
    cudaFree(d);
    if (total) *total = cnt[3];
}

void SlabContext::upload_views(const float* pixels, const double* mats, int count) {
    if (!pixels || !mats) throw bph::config_error("null argument");
    if (count < 1 || count > slots_)
        throw bph::config_error("resident views exceed the ring capacity (ring_batches * view_batch)");
    bind();
    issue_run();
    check(cudaStreamSynchronize(s_comp_), "sync");
    resident_A_.resize((size_t)count);
    for (int k = 0; k < count; ++k) {
        bph::Mat m;
        std::memcpy(m.data(), mats + 12 * k, sizeof(double) * 12);
        bph::validate_matrix_for_grid(m, grid_);
        resident_A_[(size_t)k] = bph::narrowed(m);
        float* dst = d_ring_ + (size_t)k * isy_ * pitch_;
        const float* src = pixels + (size_t)k * isy_ * isx_;
        check(cudaMemcpy2DAsync(dst, (size_t)pitch_ * sizeof(float), src, (size_t)isx_ * sizeof(float),
                                (size_t)isx_ * sizeof(float), (size_t)isy_, cudaMemcpyHostToDevice,
                                s_copy_),
              "H2D");
    }
    if (filt_) filt_->apply(d_ring_, (long long)isy_ * pitch_, pitch_, count, 0, isy_, s_copy_);
    check(cudaStreamSynchronize(s_copy_), "sync");
    std::fill(used_.begin(), used_.end(), false);
    resident_ = count;
}

double SlabContext::time_resident(int iters, bp_gpu_stats* st) {
    if (resident_ < 1) throw bph::config_error("no resident views (bp_gpu_upload_views first)");
    if (iters < 1) throw bph::config_error("iters must be >= 1");
    bind();
    reset_recon();
    check(cudaEventRecord(ev_t0_, s_comp_), "event");
    for (int it = 0; it < iters; ++it) {
        // this pass's pair-ring expansions overwrite slots the previous pass read
        check(cudaEventRecord(ev_free_[0], s_comp_), "event");
        check(cudaStreamWaitEvent(s_prep_, ev_free_[0], 0), "wait");
        // Batch schedule: view_batch-sized batches behind a quarter-size first one when
        // the pair ring's expansions overlap the kernels.  Only the first batch's
        // expansion runs in series, and a quarter batch's kernel still lasts long enough
        // for the next batch's expansion underneath it: +0.65% at 512^3 (62 + 248 + 186
        // views), an eighth is too short (-0.6%).  BP_FIRST_BATCH overrides (A/B).
        std::vector<int> k0s;
        {
            if (!tiled_) {
                bpg::BatchArgs b0{};
                b0.nviews = std::min(B_, resident_);
                for (int i = 0; i < b0.nviews; ++i) {
                    std::memcpy(b0.A[i], resident_A_[(size_t)i].data(), sizeof(float) * 12);
                    b0.slot[i] = i;
                }
                choose_tile(b0);
            }
            int first = (tiled_ && ts_.dy && overlap_expand_ && resident_ > B_) ? std::max(1, B_ / 4) : B_;
            if (const char* e = std::getenv("BP_FIRST_BATCH")) first = std::max(1, std::min(B_, std::atoi(e)));
            for (int k0 = 0; k0 < resident_; k0 += (k0 == 0 ? first : B_)) k0s.push_back(k0);
            k0s.push_back(resident_);
        }
        const int nbt = (int)k0s.size() - 1;
        auto make_batch = [&](int bi) {
            bpg::BatchArgs b{};
            b.nviews = k0s[(size_t)bi + 1] - k0s[(size_t)bi];
            b.load_volume = bi > 0 ? 1 : 0;
            for (int i = 0; i < b.nviews; ++i) {
                std::memcpy(b.A[i], resident_A_[(size_t)(k0s[(size_t)bi] + i)].data(), sizeof(float) * 12);
                b.slot[i] = k0s[(size_t)bi] + i;
            }
            return b;
        };
        for (int bi = 0; bi < nbt; ++bi) {
            bpg::BatchArgs b = make_batch(bi);
            choose_tile(b);
            if (tiled_ && ts_.dy) {
                // Inside the timed region (part of every reconstruction).  The first
                // batch's pair rows come from the full-grid expansion; each later
                // batch's from the small grid launched just before the previous
                // batch's kernel, which it runs under (co-resident, higher priority)
                const size_t gi = (size_t)bi % ev_prep_.size();
                if (bi == 0 || !overlap_expand_) {
                    expand(b, s_prep_);
                    check(cudaEventRecord(ev_prep_[gi], s_prep_), "event");
                }
                check(cudaStreamWaitEvent(s_comp_, ev_prep_[gi], 0), "wait");
                if (overlap_expand_ && bi + 1 < nbt) {
                    const bpg::BatchArgs nb = make_batch(bi + 1);
                    const size_t gn = (size_t)(bi + 1) % ev_prep_.size();
                    check(cudaStreamWaitEvent(s_aux_, ev_prep_[gi], 0), "wait");
                    expand(nb, s_aux_, true);
                    check(cudaEventRecord(ev_prep_[gn], s_aux_), "event");
                }
            }
            launch(b, 0, -1, bi + 1 == nbt);
        }
    }
    check(cudaEventRecord(ev_t1_, s_comp_), "event");
    unsigned long long cnt[8] = {0};
    check(cudaMemcpyAsync(cnt, d_cnt_, sizeof cnt, cudaMemcpyDeviceToHost, s_comp_), "counters");
    check(cudaMemsetAsync(d_cnt_, 0, sizeof cnt, s_comp_), "counters");
    check(cudaStreamSynchronize(s_comp_), "sync");
    float ms = 0;
    check(cudaEventElapsedTime(&ms, ev_t0_, ev_t1_), "elapsed");
    if (st) {
        std::memset(st, 0, sizeof *st);
        st->device_ms = ms;
        double kms = 0;
        float m2 = 0;
        for (size_t i = 0; i < launch_ev_used_; ++i) {
            check(cudaEventElapsedTime(&m2, launch_ev_[i].first, launch_ev_[i].second), "elapsed");
            kms += m2;
        }
        st->kernel_ms = kms;
        st->views = (uint64_t)resident_ * iters;
        st->launches = launches_;
        st->prep_launches = prep_launches_;
        st->nominal_updates = st->views * (uint64_t)nz_ * L_ * L_;
        st->visible_updates = cnt[3];
        st->tile_pairs = cnt[0];
        st->skipped_pairs = cnt[1];
        st->fallback_pairs = cnt[2];
        st->tile_w = tiled_ ? ts_.tw : 0;
        st->tile_h = tiled_ ? ts_.th : 0;
        st->block_x = tiled_ ? ts_.bx : 1;
        st->block_y = tiled_ ? ts_.by : 1;
        st->block_z = tiled_ ? ts_.bz : 1;
    }
    reset_recon();
    return ms;
}

}  // namespace bpr
