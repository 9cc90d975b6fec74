// engine.cu -- host orchestrator and C-ABI of liblsort_cuda.so.
//
// Drives the AIPS2o recursion on the
// GPU: per level, one batched launch sequence over all segments being
// partitioned --
//   build models -> classify+histogram -> scan/children -> scatter ->
//   base cases + equality fills of the finished children
// -- with the next level's segment list read back once per level. Workspace
// (scratch keys, model arena, bucket counters, work lists) lives in the
// context and is reused across calls. Out-of-place ping-pong between the
// caller's buffer and one scratch buffer replaces IPS4o's in-place block
// permutation; the result always lands in the caller's
// buffer because base cases and fills write there directly.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <string>
#include <atomic>
#include <chrono>
#include <mutex>
#include <thread>
#include <vector>

#include <cuda_runtime.h>

#include "../../include/lsort_cuda.h"
#include "kernels.cuh"

using namespace lsort_dev;

namespace {

struct DevBuf {
    void* p = nullptr;
    size_t cap = 0;
    ~DevBuf() { if (p) cudaFree(p); }
    bool ensure(size_t bytes) {
        if (bytes <= cap) return true;
        if (p) cudaFree(p);
        p = nullptr;
        cap = 0;
        size_t want = std::max<size_t>(bytes, 256);
        want = want + want / 8;  // headroom against regrowth
        if (cudaMalloc(&p, want) != cudaSuccess) {
            cudaGetLastError();
            if (cudaMalloc(&p, bytes) != cudaSuccess) { cudaGetLastError(); p = nullptr; return false; }
            want = bytes;
        }
        cap = want;
        return true;
    }
    template <class T> T* as() const { return (T*)p; }
    void swap(DevBuf& o) {
        std::swap(p, o.p);
        std::swap(cap, o.cap);
    }
};

struct PinBuf {
    void* p = nullptr;
    size_t cap = 0;
    ~PinBuf() { if (p) cudaFreeHost(p); }
    bool ensure(size_t bytes) {
        if (bytes <= cap) return true;
        if (p) cudaFreeHost(p);
        p = nullptr;
        cap = 0;
        size_t want = std::max<size_t>(bytes * 2, 4096);
        if (cudaMallocHost(&p, want) != cudaSuccess) { cudaGetLastError(); p = nullptr; return false; }
        cap = want;
        return true;
    }
    template <class T> T* as() const { return (T*)p; }
};

struct LsortError {
    int code;
    std::string msg;
};

#define CU(call)                                                                               \
    do {                                                                                       \
        cudaError_t e__ = (call);                                                              \
        if (e__ != cudaSuccess)                                                                \
            throw LsortError{LSORT_ECUDA, std::string(#call) + ": " + cudaGetErrorString(e__)}; \
    } while (0)

// leftover keys in 16 Ki..kClCap segments below which a level >= 1 goes to the
// fused cluster kernel (measured: C1's 15 leaves of ~365 Ki keys 0.618 -> 0.562 ms
// per sort; C2's full level 1 of 1e8 keys is 2x slower there)
constexpr uint64_t kAutoClusterKeys = 4ull << 20;

uint32_t fanout(uint64_t n, uint32_t cfg_count, uint32_t target) {
    if (target == 0) return cfg_count;
    uint64_t want = (n + target - 1) / target;
    uint32_t b = 2;
    while (b < want && b < cfg_count) b <<= 1;
    return std::min(b, cfg_count);
}

bool trace_enabled() {
    static int v = -1;
    if (v < 0) {
        const char* e = getenv("LSORT_TRACE");
        v = (e && *e && *e != '0') ? 1 : 0;
    }
    return v == 1;
}

uint64_t seg_seed_host(uint64_t cfg_seed, uint64_t begin, uint32_t depth) {
    return splitmix64(cfg_seed ^ splitmix64(begin + ((uint64_t)depth << 48)));
}
uint64_t sample_size_host(double frac, uint32_t cap, uint64_t n) {
    double v = frac * (double)n;
    double c = (double)cap;
    uint64_t s = (uint64_t)std::ceil(v < c ? v : c);
    return s < 2 ? 2 : s;
}

}  // namespace

struct lsort_ctx {
    int device = 0;
    cudaStream_t stream = nullptr;
    cudaStream_t own_stream = nullptr;
    std::string err;
    int depth = 0;  // nesting level (sample sorts run in a nested context)
    DevBuf scratch, data, segs, idx, tile_prefix, models, buckets, rec, base[3], fill, ctrl, sample, aux, train_ws,
        kseg, ktp, kplan, qws, ids, clus, bat[3], psample, slices, dist_hist, fwd_model, fwd_slices, piv, fsample;
    cudaStream_t h2d_stream = nullptr, d2h_stream = nullptr;
    cudaEvent_t bev[11] = {};  // batch pipeline: h2d[3], sorted[3], d2h[3], start, end
    PinBuf hctrl, hrec, hsegs, hidx, hprefix, hmodel;
    std::unique_ptr<lsort_ctx> nested;
    // lanes: workspaces + streams on which the models of the big segments of
    // one level are built concurrently (fork/join with events on `stream`)
    std::vector<std::unique_ptr<lsort_ctx>> lanes;
    std::vector<std::unique_ptr<lsort_ctx>> subs;  // sort_many: one context per concurrent sort
    bool zero_copy = false;  // control transfers as kernels (copy engines busy with a batch)
    // dist: bucket ids of (keys, n, kind) under the model with this fingerprint,
    // left in `ids` by lsort_cuda_dist_histogram for lsort_cuda_dist_partition
    const void* dist_keys = nullptr;
    uint64_t dist_n = 0, dist_fp = 0;
    int dist_kind = -1;
    PinBuf hstage;           // staging for small host->device transfers from pageable memory
    size_t hstage_off = 0;
    cudaEvent_t fork_ev = nullptr, join_ev = nullptr;
    cudaEvent_t ev[6] = {};
    cudaEvent_t pev[8] = {};  // phase timing
    uint64_t launches = 0;
    ~lsort_ctx() {
        if (stream) cudaStreamSynchronize(stream);
        lanes.clear();
        subs.clear();
        nested.reset();
        for (auto& e : ev) if (e) cudaEventDestroy(e);
        for (auto& e : pev) if (e) cudaEventDestroy(e);
        if (fork_ev) cudaEventDestroy(fork_ev);
        if (h2d_stream) { cudaStreamSynchronize(h2d_stream); cudaStreamDestroy(h2d_stream); }
        if (d2h_stream) { cudaStreamSynchronize(d2h_stream); cudaStreamDestroy(d2h_stream); }
        for (auto& e : bev) if (e) cudaEventDestroy(e);
        if (join_ev) cudaEventDestroy(join_ev);
        if (own_stream) cudaStreamDestroy(own_stream);
    }
};

namespace {

struct SegPlan {
    uint64_t begin, n;
    uint32_t depth, flags;
    uint64_t pslice = 0;  // slice of the parent's sorted sample (SegDesc::pslice)
};

void validate_cfg(const lsort_cfg& c) {
    auto pow2 = [](uint32_t v) { return v >= 2 && (v & (v - 1)) == 0; };
    if (!pow2(c.rmi_bucket_count) || c.rmi_bucket_count > LSORT_MAX_RMI)
        throw LsortError{LSORT_EINVAL, "rmi_bucket_count must be a power of two in [2, 2048]"};
    if (!pow2(c.tree_bucket_count) || c.tree_bucket_count > LSORT_MAX_TREE)
        throw LsortError{LSORT_EINVAL, "tree_bucket_count must be a power of two in [2, 1024]"};
    if (c.first_sample_cap < 2 || c.first_sample_cap > kSmallSampleCap)
        throw LsortError{LSORT_EINVAL, "first_sample_cap must be in [2, 8192]"};
    if (c.rmi_sample_cap < 2) throw LsortError{LSORT_EINVAL, "rmi_sample_cap must be >= 2"};
    if (!(c.sample_fraction > 0.0) || c.sample_fraction > 1.0)
        throw LsortError{LSORT_EINVAL, "sample_fraction must be in (0, 1]"};
    if (c.base_case_capacity < 1024 || c.base_case_capacity > 16384)
        throw LsortError{LSORT_EINVAL, "base_case_capacity must be in [1024, 16384]"};
    if (c.insertion_base_case > c.radix_base_case)
        throw LsortError{LSORT_EINVAL, "insertion_base_case must be <= radix_base_case"};
}

// GPU policy (unless LSORT_FLAG_STRICT_POLICY): segments from kGpuMinRmi keys
// up may take the learned branch of Alg. 5 -- on the GPU a learned model
// classifies at ~2/3 of the cost of a splitter-tree descent, and poor learned
// models are caught by the quality check. Sorted output is the same.
constexpr uint64_t kGpuMinRmi = 32768;
uint64_t effective_min_rmi(const lsort_cfg& c) {
    return (c.flags & LSORT_FLAG_STRICT_POLICY) ? c.min_rmi_input : std::min<uint64_t>(c.min_rmi_input, kGpuMinRmi);
}

DevCfg dev_cfg(const lsort_cfg& c) {
    DevCfg d;
    d.min_rmi_input = effective_min_rmi(c);
    d.max_dup = c.max_duplicate_fraction;
    d.sample_fraction = c.sample_fraction;
    d.first_sample_cap = c.first_sample_cap;
    d.rmi_sample_cap = c.rmi_sample_cap;
    d.seed = c.seed;
    d.quality = (c.flags & LSORT_FLAG_STRICT_POLICY) ? 0u : 1u;
    d.psample = nullptr;
    return d;
}

// Model forwarding (LearnedSort 2.0 classic path, cdf_lo/cdf_hi
// models.hpp:128-138): the root level reuses a given learned model restricted
// to a CDF range instead of sampling and training; its children train on
// slices of the given sorted sample.
struct Forward {
    const uint8_t* model = nullptr;  // device ModelHdr + learned payload (cdf range, nb local buckets)
    size_t model_bytes = 0;
    uint32_t nb = 0, B = 0;          // local buckets, submodels
    const uint32_t* slices = nullptr;  // device [nb+1] offsets into psample, or nullptr
    const uint64_t* psample = nullptr;
};

struct Engine {
    lsort_ctx* C;
    const lsort_cfg& cfg;
    cudaStream_t st;
    Engine(lsort_ctx* c, const lsort_cfg& g) : C(c), cfg(g), st(c->stream) {}

    uint32_t rmi_b(uint64_t n) const { return fanout(n, cfg.rmi_bucket_count, cfg.bucket_target); }
    uint32_t tree_k(uint64_t n) const { return fanout(n, cfg.tree_bucket_count, cfg.bucket_target); }
    // largest sample the segment's model may need (the RMI sample only if the
    // policy can pick the learned branch)
    uint64_t sample_need(const SegPlan& s) const {
        uint64_t s1 = sample_size_host(cfg.sample_fraction, cfg.first_sample_cap, s.n);
        uint64_t s2 = s.n >= effective_min_rmi(cfg) ? sample_size_host(cfg.sample_fraction, cfg.rmi_sample_cap, s.n) : 0;
        return std::max(s1, s2);
    }
    // 0 small model CTA, 1 mid model CTA, 2 big pipeline
    int model_class(const SegPlan& s) const {
        if (s.flags & kSegForceRadix) return 0;
        uint64_t need = s.pslice ? std::min<uint64_t>(s.pslice & 0xffffffu, kSmallSampleCap) : sample_need(s);
        if (need <= kModelSmallCap) return 0;
        if (need <= kSmallSampleCap) return 1;
        return 2;
    }

    void launched(int k = 1) { C->launches += k; }

    // host -> device of a small control block. `h` may be pageable: with zero
    // copy it is staged in mapped pinned memory that stays untouched until
    // the level's closing stream synchronisation (stage_reset).
    void up(void* d, const void* h, size_t bytes, bool h_pinned = false, cudaStream_t s = nullptr) {
        if (!bytes) return;
        if (!s) s = st;
        if (!C->zero_copy) {
            CU(cudaMemcpyAsync(d, h, bytes, cudaMemcpyHostToDevice, s));
            return;
        }
        const void* src = h;
        if (!h_pinned) {
            const size_t off = (C->hstage_off + 15) & ~(size_t)15;
            if (off + bytes > C->hstage.cap) {  // does not fit the staging area: plain DMA
                CU(cudaMemcpyAsync(d, h, bytes, cudaMemcpyHostToDevice, s));
                return;
            }
            std::memcpy(C->hstage.as<uint8_t>() + off, h, bytes);
            src = C->hstage.as<uint8_t>() + off;
            C->hstage_off = off + bytes;
        }
        launch_copy_bytes(d, src, bytes, s);
        launched();
    }
    // device -> pinned host
    void down(void* hpinned, const void* d, size_t bytes) {
        if (!bytes) return;
        if (!C->zero_copy) {
            CU(cudaMemcpyAsync(hpinned, d, bytes, cudaMemcpyDeviceToHost, st));
            return;
        }
        launch_copy_bytes(hpinned, d, bytes, st);
        launched();
    }
    void stage_reset() { C->hstage_off = 0; }

    // Sort the device buffer `sample` (u64) with a nested context.
    void nested_sort(uint64_t* sample, uint64_t s) {
        if (C->depth >= 2) throw LsortError{LSORT_EINTERNAL, "sample sort nesting too deep"};
        nested_ctx();
        lsort_cfg nc = cfg;
        nc.seed = splitmix64(cfg.seed ^ 0x5a3c9e1f0b7d2468ull);
        Engine ne(C->nested.get(), nc);
        lsort_stats nst{};
        if (trace_enabled()) nc.flags |= LSORT_FLAG_PHASE_TIMING;
        ne.sort(sample, s, false, trace_enabled() ? &nst : nullptr);
        C->launches += C->nested->launches;
        C->nested->launches = 0;
    }

    lsort_ctx* nested_ctx() {
        if (!C->nested) {
            C->nested.reset(new lsort_ctx());
            C->nested->device = C->device;
            C->nested->depth = C->depth + 1;
            for (auto& e : C->nested->ev) CU(cudaEventCreate(&e));
            for (auto& e : C->nested->pev) CU(cudaEventCreate(&e));
        }
        C->nested->stream = C->stream;
        return C->nested.get();
    }

    lsort_ctx* lane(uint32_t i) {
        while (C->lanes.size() <= i) {
            std::unique_ptr<lsort_ctx> L(new lsort_ctx());
            L->device = C->device;
            L->depth = C->depth + 1;
            // lanes carry the dependent chains (big-segment pipelines, mid
            // models): highest priority so their CTAs are scheduled ahead of
            // the wide small-model grid on the context stream
            int lo = 0, hi = 0;
            CU(cudaDeviceGetStreamPriorityRange(&lo, &hi));
            CU(cudaStreamCreateWithPriority(&L->own_stream, cudaStreamNonBlocking, hi));
            L->stream = L->own_stream;
            CU(cudaEventCreateWithFlags(&L->join_ev, cudaEventDisableTiming));
            C->lanes.push_back(std::move(L));
        }
        return C->lanes[i].get();
    }
    static constexpr uint32_t kLanes = 8;

    // All models of a level: the big segments' pipelines on up to kLanes
    // lane streams, the mid-size CTAs (8192-sample, the long pole among the
    // one-CTA models) on one more lane, the small models on the context
    // stream -- forked from and joined back into the context stream.
    void level_models(const std::vector<uint32_t>& bigs, const SegDesc* dsegs, const std::vector<SegPlan>& segs,
                      const SegDesc* hs, const void* src, bool f64, const uint32_t* didx, uint32_t nsmall,
                      uint32_t nmid, const DevCfg& dc, uint32_t* root_slices = nullptr) {
        const uint32_t nl = (uint32_t)std::min<size_t>(bigs.size(), kLanes);
        const bool mid_lane = nmid && (nsmall || !bigs.empty());
        const uint32_t used = nl + (mid_lane ? 1 : 0);
        if (used) {
            if (!C->fork_ev) CU(cudaEventCreateWithFlags(&C->fork_ev, cudaEventDisableTiming));
            CU(cudaEventRecord(C->fork_ev, st));
            for (uint32_t l = 0; l < used; ++l) CU(cudaStreamWaitEvent(lane(l)->stream, C->fork_ev, 0));
        }
        for (uint32_t bi = 0; bi < bigs.size(); ++bi)
            big_model(dsegs + bigs[bi], segs[bigs[bi]], hs[bigs[bi]], src, f64, lane(bi % nl),
                      bi == 0 ? root_slices : nullptr);
        if (root_slices && !bigs.empty()) C->psample.swap(lane(0)->sample);  // keep the root's sorted sample
        launch_build_models(dsegs, didx + nsmall, nmid, src, f64, C->models.as<uint8_t>(), dc, 1,
                            mid_lane ? lane(nl)->stream : st);
        launch_build_models(dsegs, didx, nsmall, src, f64, C->models.as<uint8_t>(), dc, 0, st);
        launched((nsmall ? 1 : 0) + (nmid ? 1 : 0));
        for (uint32_t l = 0; l < used; ++l) {
            CU(cudaEventRecord(lane(l)->join_ev, lane(l)->stream));
            CU(cudaStreamWaitEvent(st, lane(l)->join_ev, 0));
        }
    }
    void big_models(const std::vector<uint32_t>& bigs, const SegDesc* dsegs, const std::vector<SegPlan>& segs,
                    const SegDesc* hs, const void* src, bool f64) {
        level_models(bigs, dsegs, segs, hs, src, f64, nullptr, 0, 0, dev_cfg(cfg));
    }

    // Base cases of a level: the 16 Ki and 1 Ki classes on two lane streams
    // (high priority: the long 1024-thread CTAs start first) beside the 4 Ki
    // class on the context stream, joined back before the next level.
    void base_cases(const LevelParams& p, const uint64_t* src, void* out, bool f64) {
        static const bool serial = getenv("LSORT_BASE_SERIAL") != nullptr;
        if (serial) {
            launch_base_cases(p, src, out, f64, st);
            return;
        }
        if (!C->fork_ev) CU(cudaEventCreateWithFlags(&C->fork_ev, cudaEventDisableTiming));
        CU(cudaEventRecord(C->fork_ev, st));
        for (uint32_t l = 0; l < 2; ++l) CU(cudaStreamWaitEvent(lane(l)->stream, C->fork_ev, 0));
        launch_base_class(p, 2, src, out, f64, lane(0)->stream);
        launch_base_class(p, 0, src, out, f64, lane(1)->stream);
        launch_base_class(p, 1, src, out, f64, st);
        for (uint32_t l = 0; l < 2; ++l) {
            CU(cudaEventRecord(lane(l)->join_ev, lane(l)->stream));
            CU(cudaStreamWaitEvent(st, lane(l)->join_ev, 0));
        }
    }

    // Model for one big segment (RMI sample > one CTA), with no host round
    // trip: (1) one CTA draws + sorts the first sample, decides the policy
    // (writes *gate) and builds a splitter tree over the first sample;
    // (2) device-wide gather of the RMI sample; (3) the sample is sorted by one
    // distribution level with that tree + shared-memory base cases; (4)
    // multi-CTA training. Every step after (1) is gated on the device.
    void big_model(const SegDesc* dseg, const SegPlan& sp, const SegDesc& hseg, const void* src, bool f64,
                   lsort_ctx* N, uint32_t* slices = nullptr) {
        const cudaStream_t st = N->stream;  // this lane's stream
        DevCfg dc = dev_cfg(cfg);
        const uint64_t n = sp.n;
        const uint64_t s1 = sample_size_host(cfg.sample_fraction, cfg.first_sample_cap, n);
        const uint64_t s2 = sample_size_host(cfg.sample_fraction, cfg.rmi_sample_cap, n);
        // sample-sort splitter budget: ~2 Ki samples per bucket (base-case class <= 4 Ki)
        uint32_t k = cfg.tree_bucket_count;
        while (k < LSORT_MAX_TREE_DEV && (uint64_t)k * 2048 < s2) k <<= 1;
        const uint32_t nb = 2 * k - 1;
        const size_t aux_bytes = sizeof(ModelHdr) + ((tree_payload_bytes(k, k - 1) + 15) & ~15ull);
        const uint64_t ntiles = (s2 + kTileKeys - 1) / kTileKeys;
        if (!N->sample.ensure(s2 * 8) || !N->scratch.ensure(s2 * 8) || !N->models.ensure(aux_bytes) ||
            !N->segs.ensure(sizeof(SegDesc)) || !N->tile_prefix.ensure(16) || !N->buckets.ensure(8 * (size_t)nb) ||
            !N->rec.ensure(nb * sizeof(SegOut)) || !N->fill.ensure(nb * sizeof(FillItem)) ||
            !N->base[0].ensure(nb * sizeof(BaseItem)) || !N->base[1].ensure(nb * sizeof(BaseItem)) ||
            !N->base[2].ensure(nb * sizeof(BaseItem)) || !N->kseg.ensure(64) || !N->ktp.ensure(64) ||
            !N->kplan.ensure(3 * sizeof(KindPlan)) || !N->ctrl.ensure(sizeof(Ctrl)) || !N->ids.ensure(2 * s2) ||
            !N->aux.ensure(4) || !N->train_ws.ensure(train_workspace_bytes(s2, hseg.rmi_b)))
            throw LsortError{LSORT_ENOMEM, "big model workspace"};
        uint32_t* gate = N->aux.as<uint32_t>();
        Ctrl* nctrl = N->ctrl.as<Ctrl>();
        // the RMI-sample gather does not depend on the first sample: it runs on
        // the lane's helper stream while k_first_sample decides the policy
        // (ungated: wasted work only if the policy picks the tree branch)
        if (!N->h2d_stream) {
            int lo = 0, hi = 0;
            CU(cudaDeviceGetStreamPriorityRange(&lo, &hi));
            CU(cudaStreamCreateWithPriority(&N->h2d_stream, cudaStreamNonBlocking, hi));
        }
        for (int e = 0; e < 2; ++e)
            if (!N->bev[e]) CU(cudaEventCreateWithFlags(&N->bev[e], cudaEventDisableTiming));
        CU(cudaEventRecord(N->bev[0], st));
        CU(cudaStreamWaitEvent(N->h2d_stream, N->bev[0], 0));
        const uint64_t seed = seg_seed_host(cfg.seed, sp.begin, sp.depth);
        launch_gather(dseg, src, f64, seed, s1, s2, N->sample.as<uint64_t>(), nullptr, N->h2d_stream);
        CU(cudaEventRecord(N->bev[1], N->h2d_stream));
        // the first sample's random gather over many CTAs (one CTA cannot keep
        // 8 Ki random loads in flight: ~30 us), then the policy CTA
        if (!N->fsample.ensure(s1 * 8)) throw LsortError{LSORT_ENOMEM, "first sample"};
        launch_gather(dseg, src, f64, seed, 0, s1, N->fsample.as<uint64_t>(), nullptr, st);
        launch_first_sample(dseg, src, f64, C->models.as<uint8_t>(), dc, N->models.as<uint8_t>(), k, gate, st,
                            N->fsample.as<uint64_t>());
        launched();
        CU(cudaStreamWaitEvent(st, N->bev[1], 0));
        // one distribution level over the sample with the first-sample tree
        SegDesc d{};
        d.begin = 0;
        d.n = s2;
        d.model_off = 0;
        d.bucket_off = 0;
        d.nb_max = nb;
        d.tree_k = k;
        uint64_t pref[2] = {0, ntiles};
        up(N->segs.p, &d, sizeof(d), false, st);
        up(N->tile_prefix.p, pref, 16, false, st);
        CU(cudaMemsetAsync(N->buckets.p, 0, 8 * (size_t)nb, st));
        CU(cudaMemsetAsync(nctrl, 0, sizeof(Ctrl), st));
        CU(cudaMemsetAsync(&nctrl->nan_index, 0xff, 8, st));
        LevelParams q{};
        q.segs = N->segs.as<SegDesc>();
        q.nsegs = 1;
        q.tile_prefix = N->tile_prefix.as<uint64_t>();
        q.ntiles = ntiles;
        q.models = N->models.as<uint8_t>();
        q.buckets = N->buckets.as<unsigned long long>();
        q.src = N->sample.p;
        q.dst = N->scratch.as<uint64_t>();
        q.ids = N->ids.as<uint16_t>();
        q.ctrl = nctrl;
        q.rec = N->rec.as<SegOut>();
        for (int c = 0; c < 3; ++c) q.base[c] = N->base[c].as<BaseItem>();
        q.fill = N->fill.as<FillItem>();
        q.base_cap[0] = kWarpBaseCap;
        q.base_cap[1] = 4096;
        q.base_cap[2] = 16384;
        q.depth_cap = 64;
        q.list_cap = nb;
        q.gate = gate;
        q.kseg = N->kseg.as<uint32_t>();
        q.ktp = N->ktp.as<uint64_t>();
        q.kplan = N->kplan.as<KindPlan>();
        q.kstride = 1;
        const int nsm = num_sms();
        const int g = (int)std::min<uint64_t>(ntiles, (uint64_t)nsm * kPartPerSM);
        launch_kind_plan(q, st);
        launch_hist(q, 0, 2u, 0, g, st);
        launch_scan_children(q, nb, st);
        launch_scatter(q, 0, nb, g, st);
        launch_base_cases(q, N->scratch.as<uint64_t>(), N->sample.p, 0, st);
        launch_fill(q, N->sample.p, 0, nsm, st);
        launch_train_rmi(N->sample.as<uint64_t>(), s2, hseg.rmi_b, C->models.as<uint8_t>() + hseg.model_off,
                         hseg.rmi_b, N->train_ws.p, gate, st);
        launched(2 + 9 + 8);
        if (dc.quality) {  // (and the children's sample slices for the root)
            if (!N->qws.ensure(quality_workspace_bytes())) throw LsortError{LSORT_ENOMEM, "quality workspace"};
            launch_quality_check(N->sample.as<uint64_t>(), s2, C->models.as<uint8_t>() + hseg.model_off, hseg.tree_k,
                                 N->qws.p, slices, gate, st);
            launched(slices ? 3 : 2);
        } else if (slices) {
            launch_sample_slices(N->sample.as<uint64_t>(), s2, C->models.as<uint8_t>() + hseg.model_off, slices,
                                 hseg.nb_max, gate, st);
            launched();
        }
    }

    // Sort n keys at `keys` (device) in place. Returns LSORT_ENAN via throw.
    // in_encoded: the keys are already encoded u64 (keys.hpp:36-42); with f64
    // the sorted result is decoded to float64 in place (the decode fused into
    // the final stores -- used for the keys a multi-GPU exchange delivers)
    // start (nullable): the keys are already partitioned into these segments
    // (contiguous, each > the base-case capacity); the recursion starts at
    // level 1 with them instead of sampling a root model over all n keys.
    void sort(void* keys, uint64_t n, bool f64, lsort_stats* stats, bool in_encoded = false,
              const Forward* fw = nullptr, const std::vector<SegPlan>* start = nullptr) {
        // the bucket ids a dist_histogram left in C->ids are overwritten below
        C->dist_keys = nullptr;
        if (n < 2) {
            if (n == 1 && f64 && in_encoded) {
                launch_decode((uint64_t*)keys, n, st);
                launched();
            }
            return;
        }
        if (!C->ctrl.ensure(sizeof(Ctrl)) || !C->hctrl.ensure(sizeof(Ctrl)) || !C->hmodel.ensure(sizeof(ModelHdr)))
            throw LsortError{LSORT_ENOMEM, "control block"};
        Ctrl* dctrl = C->ctrl.as<Ctrl>();
        CU(cudaMemsetAsync(dctrl, 0, sizeof(Ctrl), st));
        CU(cudaMemsetAsync(&dctrl->nan_index, 0xff, 8, st));
        Ctrl* hc = C->hctrl.as<Ctrl>();
        const uint32_t cap = cfg.base_case_capacity;
        if (n <= cap && !start) {
            launch_small_sort(keys, n, f64 && !in_encoded, dctrl, st);
            launched();
            if (f64 && in_encoded) {
                launch_decode((uint64_t*)keys, n, st);
                launched();
            }
            down(hc, dctrl, sizeof(Ctrl));
            CU(cudaStreamSynchronize(st));
            if (hc->nan_index != ~0ull) throw LsortError{LSORT_ENAN, std::to_string(hc->nan_index)};
            if (stats) { stats->level0_kind = 2; stats->base_case_keys += n; }
            return;
        }
        if (!C->scratch.ensure(n * 8) || !C->ids.ensure(n * 2)) throw LsortError{LSORT_ENOMEM, "scratch keys"};
        const uint32_t depth_cap =
            (uint32_t)std::ceil(std::log2((double)n) / std::log2((double)cfg.tree_bucket_count)) + 4;
        std::vector<SegPlan> segs{{0, n, 0, 0}};
        if (start) segs = *start;
        void* src = keys;
        bool src_f64 = f64 && !in_encoded && !start;
        uint64_t* dst = C->scratch.as<uint64_t>();
        uint32_t level = start ? 1 : 0;
        DevCfg dc = dev_cfg(cfg);
        while (!segs.empty()) {
            const uint32_t ns = (uint32_t)segs.size();
            // ---- plan the level on the host
            if (!C->hsegs.ensure(ns * sizeof(SegDesc)) || !C->hprefix.ensure((ns + 1) * 8) ||
                !C->hidx.ensure(ns * 4))
                throw LsortError{LSORT_ENOMEM, "host plan"};
            SegDesc* hs = C->hsegs.as<SegDesc>();
            uint64_t* hp = C->hprefix.as<uint64_t>();
            uint32_t* hi = C->hidx.as<uint32_t>();
            uint64_t model_bytes = 0, nbuckets = 0, ntiles = 0;
            uint32_t max_payload = 0, max_nb = 0, nsmall = 0, kinds = 0, max_rmi_b = 0;
            std::vector<uint32_t> mids;
            std::vector<uint32_t> bigs;
            // segments of the last distribution level that fit a cluster go to the
            // fused DSMEM kernel (cluster.cu); the rest are partitioned here
            // GPU policy: a FEW leftover segments just above the base-case capacity
            // (C1's handful of 16-35 Ki leaves) are cheaper in the fused cluster
            // kernel than through a whole latency-bound partition level; many of
            // them (a full level 1) are not -- the cluster kernel runs one CTA per SM
            uint64_t elig_keys = 0;
            if (level >= 1)
                for (const SegPlan& q : segs)
                    if (q.n > cap && q.n <= kClCap) elig_keys += q.n;
            static const bool no_auto_cluster = getenv("LSORT_NO_AUTO_CLUSTER") != nullptr;
            const bool auto_cluster = !no_auto_cluster && !(cfg.flags & LSORT_FLAG_STRICT_POLICY) &&
                                      elig_keys > 0 && elig_keys <= kAutoClusterKeys;
            const bool use_cluster = level >= 1 && !src_f64 && cluster_available() &&
                                     ((cfg.flags & LSORT_FLAG_CLUSTER) || auto_cluster) && cap >= 16384;
            std::vector<BaseItem> clus;
            std::vector<SegPlan> psegs;
            psegs.reserve(ns);
            for (uint32_t i = 0; i < ns; ++i) {
                const SegPlan& s = segs[i];
                if (use_cluster && s.n > cap && s.n <= kClCap) {
                    clus.push_back(BaseItem{s.begin, s.n});
                    continue;
                }
                const uint32_t j = (uint32_t)psegs.size();
                psegs.push_back(s);
                SegDesc& d = hs[j];
                d.begin = s.begin;
                d.n = s.n;
                d.depth = s.depth;
                d.flags = s.flags;
                d.pslice = s.pslice;
                d.rmi_b = (fw && level == 0) ? fw->nb : rmi_b(s.n);
                max_rmi_b = std::max(max_rmi_b, d.rmi_b);
                d.tree_k = tree_k(s.n);
                uint32_t payload, nb;
                if (s.flags & kSegForceRadix) {
                    payload = 0;
                    nb = 1u << kRadixBits;
                } else {
                    uint32_t tp = (uint32_t)((tree_payload_bytes(d.tree_k, d.tree_k - 1) + 15) & ~15ull);
                    payload = std::max<uint32_t>(kLearnedEntryBytes * d.rmi_b, tp);
                    nb = std::max<uint32_t>(d.rmi_b, 2 * d.tree_k - 1);
                }
                d.nb_max = nb;
                d.model_off = model_bytes;
                model_bytes += sizeof(ModelHdr) + payload;
                d.bucket_off = nbuckets;
                nbuckets += nb;
                max_payload = std::max(max_payload, payload);
                max_nb = std::max(max_nb, nb);
                hp[j] = ntiles;
                ntiles += (s.n + kTileKeys - 1) / kTileKeys;
                if (fw && level == 0) {  // forwarded root model: nothing to build
                    payload = std::max<uint32_t>(payload, (uint32_t)fw->model_bytes);
                    kinds |= 1u;
                    max_rmi_b = std::max(max_rmi_b, fw->B);
                    model_bytes = d.model_off + sizeof(ModelHdr) + payload;
                    continue;
                }
                const int mc = model_class(s);
                if (mc == 2) bigs.push_back(j);
                else if (mc == 1) mids.push_back(j);
                else hi[nsmall++] = j;
                if (s.flags & kSegForceRadix) kinds |= 4u;
                else kinds |= (s.n >= effective_min_rmi(cfg) ? 1u : 0u) | 2u;
            }
            const uint32_t np = (uint32_t)psegs.size();
            const uint32_t ncl = (uint32_t)clus.size();
            hp[np] = ntiles;
            const uint64_t list_cap = nbuckets + (uint64_t)ncl * kClSub;
            if (!C->segs.ensure(np * sizeof(SegDesc) + 16) || !C->tile_prefix.ensure((np + 1) * 8) ||
                !C->idx.ensure(np * 4 + 4) || !C->models.ensure(model_bytes + 16) ||
                !C->buckets.ensure(nbuckets * 8 + 8) || !C->rec.ensure(list_cap * sizeof(SegOut)) ||
                !C->fill.ensure(list_cap * sizeof(FillItem)) || !C->base[0].ensure(list_cap * sizeof(BaseItem)) ||
                !C->base[1].ensure(list_cap * sizeof(BaseItem)) || !C->base[2].ensure(list_cap * sizeof(BaseItem)) ||
                !C->kseg.ensure(3 * (size_t)np * 4 + 16) || !C->ktp.ensure(3 * ((size_t)np + 1) * 8) ||
                !C->kplan.ensure(3 * sizeof(KindPlan)) || !C->clus.ensure(ncl * sizeof(BaseItem) + 16))
                throw LsortError{LSORT_ENOMEM, "level workspace"};
            if (np) {
                up(C->segs.p, hs, np * sizeof(SegDesc), true);
                up(C->tile_prefix.p, hp, (np + 1) * 8, true);
            }
            if (ncl) up(C->clus.p, clus.data(), ncl * sizeof(BaseItem));
            for (uint32_t i = 0; i < mids.size(); ++i) hi[nsmall + i] = mids[i];
            const uint32_t nmid = (uint32_t)mids.size();
            if (nsmall + nmid) up(C->idx.p, hi, (nsmall + nmid) * 4, true);
            if (nbuckets) CU(cudaMemsetAsync(C->buckets.p, 0, nbuckets * 8, st));
            CU(cudaMemsetAsync(&dctrl->n_rec, 0, offsetof(Ctrl, keys_fill) - offsetof(Ctrl, n_rec), st));

            LevelParams p{};
            p.segs = C->segs.as<SegDesc>();
            p.nsegs = np;
            p.tile_prefix = C->tile_prefix.as<uint64_t>();
            p.ntiles = ntiles;
            p.models = C->models.as<uint8_t>();
            p.buckets = C->buckets.as<unsigned long long>();
            p.src = src;
            p.dst = dst;
            p.ids = C->ids.as<uint16_t>();
            p.ctrl = dctrl;
            p.rec = C->rec.as<SegOut>();
            for (int c = 0; c < 3; ++c) p.base[c] = C->base[c].as<BaseItem>();
            p.fill = C->fill.as<FillItem>();
            p.base_cap[0] = std::min<uint32_t>(kWarpBaseCap, cap);
            p.base_cap[1] = std::min<uint32_t>(4096, cap);
            p.base_cap[2] = cap;
            p.depth_cap = depth_cap;
            p.list_cap = (uint32_t)std::min<uint64_t>(list_cap, 0xffffffffu);
            p.kseg = C->kseg.as<uint32_t>();
            p.ktp = C->ktp.as<uint64_t>();
            p.kplan = C->kplan.as<KindPlan>();
            p.kstride = np;

            const bool timing = (cfg.flags & LSORT_FLAG_PHASE_TIMING) && stats;
            auto mark = [&](int i) {
                if (timing) CU(cudaEventRecord(C->pev[i], st));
            };
            mark(0);
            // ---- models
            const int nsm = num_sms();
            // GPU policy: the root's sorted model sample seeds its children's models
            uint32_t* root_slices = nullptr;
            dc.psample = (level == 1 && C->psample.p) ? C->psample.as<uint64_t>() : nullptr;
            if (fw) dc.psample = level == 1 ? fw->psample : nullptr;
            if (fw && level == 0) {
                CU(cudaMemcpyAsync(C->models.p, fw->model, fw->model_bytes, cudaMemcpyDeviceToDevice, st));
                p.slices = fw->slices;
            }
            if (!fw && level == 0 && np == 1 && bigs.size() == 1 && !(cfg.flags & LSORT_FLAG_STRICT_POLICY)) {
                if (!C->slices.ensure(4 * ((size_t)hs[0].nb_max + 2))) throw LsortError{LSORT_ENOMEM, "slices"};
                CU(cudaMemsetAsync(C->slices.p, 0, 4 * ((size_t)hs[0].nb_max + 2), st));
                root_slices = C->slices.as<uint32_t>();
                p.slices = root_slices;
            }
            if (np) {
                const auto th0 = std::chrono::steady_clock::now();
                level_models(bigs, p.segs, psegs, hs, src, src_f64, C->idx.as<uint32_t>(), nsmall, nmid, dc,
                             root_slices);
                if (trace_enabled())
                    fprintf(stderr, "    level_models host %.3f ms\n",
                            std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - th0).count());
            }
            // ---- partition
            const int grid_h = (int)std::min<uint64_t>(ntiles, (uint64_t)nsm * kPartPerSM);
            const int grid_s = (int)std::min<uint64_t>(ntiles, (uint64_t)nsm * kPartPerSM);
            const int nk = __builtin_popcount(kinds);
            mark(1);
            if (np) {
                launch_kind_plan(p, st);
                launch_hist(p, src_f64, kinds, max_rmi_b, grid_h, st);
                launch_scan_children(p, max_nb, st);
            }
            mark(2);
            // The next level is planned from the child list, which is final once
            // k_scan_children has run: it is read back here and the host plans
            // level L+1 while the GPU still scatters / sorts level L (unless the
            // cluster level appends children, or per-level timing wants a sync).
            constexpr uint32_t kRecSpec = 4096;  // children read back speculatively
            const uint32_t spec = (uint32_t)std::min<uint64_t>(kRecSpec, list_cap);
            if (!C->hrec.ensure((size_t)spec * sizeof(SegOut) + 64)) throw LsortError{LSORT_ENOMEM, "host rec list"};
            const bool early = ncl == 0 && !timing;
            auto read_back = [&]() {
                down(hc, dctrl, sizeof(Ctrl));
                if (level == 0 && stats) down(C->hmodel.p, C->models.p, sizeof(ModelHdr));
                down(C->hrec.p, C->rec.p, (size_t)spec * sizeof(SegOut));
            };
            if (early) {
                read_back();
                CU(cudaEventRecord(C->ev[5], st));
            }
            if (np) {
                launch_scatter(p, src_f64, max_nb, grid_s, st);
                launched(3 + nk);
            }
            mark(3);
            if (ncl) {
                launch_cluster_sort(C->clus.as<BaseItem>(), ncl, (const uint64_t*)src, dst, keys, f64, p, level + 1,
                                    st);
                launched();
            }
            base_cases(p, dst, keys, f64);
            mark(4);
            launch_fill(p, keys, f64, nsm * 4, st);
            mark(5);
            launched(3 + 1);
            if (early) {
                CU(cudaEventSynchronize(C->ev[5]));
            } else {
                read_back();
                CU(cudaStreamSynchronize(st));
            }
            stage_reset();
            CU(cudaGetLastError());
            if (hc->nan_index != ~0ull) throw LsortError{LSORT_ENAN, std::to_string(hc->nan_index)};
            if (hc->err) throw LsortError{LSORT_EINTERNAL, "work list overflow (" + std::to_string(hc->err) + ")"};
            if (timing) {
                float t[5];
                for (int i = 0; i < 5; ++i) CU(cudaEventElapsedTime(&t[i], C->pev[i], C->pev[i + 1]));
                if (trace_enabled()) {
                    uint64_t keys = 0, mx = 0;
                    for (auto& q : segs) { keys += q.n; mx = std::max(mx, q.n); }
                    fprintf(stderr,
                            "[lsort d%d L%u] segs=%u clus=%u big=%zu keys=%llu max=%llu tiles=%llu | models %.3f "
                            "classify %.3f scatter %.3f base %.3f fill %.3f ms | rec=%u base=%u/%u/%u fill=%u\n",
                            C->depth, level, ns, ncl, bigs.size(), (unsigned long long)keys, (unsigned long long)mx,
                            (unsigned long long)ntiles, t[0], t[1], t[2], t[3], t[4], hc->n_rec, hc->n_base[0],
                            hc->n_base[1], hc->n_base[2], hc->n_fill);
                }
                if (trace_enabled() && np) {
                    KindPlan kp[3];
                    CU(cudaMemcpy(kp, C->kplan.p, sizeof(kp), cudaMemcpyDeviceToHost));
                    fprintf(stderr, "    kinds: learned %u segs / %llu tiles, tree %u / %llu, radix %u / %llu\n",
                            kp[0].nsegs, (unsigned long long)kp[0].ntiles, kp[1].nsegs, (unsigned long long)kp[1].ntiles,
                            kp[2].nsegs, (unsigned long long)kp[2].ntiles);
                    if (getenv("LSORT_TRACE_KINDS")) {
                        std::string ks;
                        for (uint32_t j = 0; j < np; ++j) {
                            ModelHdr mh;
                            CU(cudaMemcpy(&mh, C->models.as<uint8_t>() + hs[j].model_off, sizeof(mh), cudaMemcpyDeviceToHost));
                            ks += mh.kind == kLearned ? (mh.s2 ? 'L' : 'l') : (mh.kind == kTree ? 'T' : 'R');
                            if (j % 37 == 1)
                                fprintf(stderr, "      seg %u n=%llu slice=%llu kind=%u nb=%u dup=%.4f s1=%llu s2=%llu rmi_b=%u\n", j,
                                        (unsigned long long)hs[j].n, (unsigned long long)(hs[j].pslice & 0xffffff), mh.kind,
                                        mh.nbuckets, mh.dup, (unsigned long long)mh.s1, (unsigned long long)mh.s2, hs[j].rmi_b);
                        }
                        fprintf(stderr, "    seg kinds: %s\n", ks.c_str());
                    }
                }
                if (trace_enabled()) {
                    for (uint32_t bi = 0; bi < bigs.size(); ++bi) {
                        ModelHdr mh;
                        CU(cudaMemcpy(&mh, C->models.as<uint8_t>() + hs[bigs[bi]].model_off, sizeof(mh),
                                      cudaMemcpyDeviceToHost));
                        fprintf(stderr,
                                "    big seg begin=%llu n=%llu depth=%u: kind=%u nb=%u B=%u dup=%.4f s1=%llu s2=%llu "
                                "root=(%.6g, %.6g) base=%.6g scale=%.6g cdf_lo=%.6g inv_span=%.6g\n",
                                (unsigned long long)psegs[bigs[bi]].begin, (unsigned long long)psegs[bigs[bi]].n,
                                psegs[bigs[bi]].depth, mh.kind, mh.nbuckets, mh.B, mh.dup, (unsigned long long)mh.s1,
                                (unsigned long long)mh.s2, mh.root_slope, mh.root_icpt, mh.key_base, mh.key_scale,
                                mh.cdf_lo, mh.inv_span);
                    }
                }
                stats->ms_models += t[0];
                stats->ms_classify += t[1];
                stats->ms_scatter += t[2];
                stats->ms_base += t[3];
                stats->ms_fill += t[4];
                if (level == 0) {
                    stats->ms_level0_classify = t[1];
                    stats->ms_level0_scatter = t[2];
                    stats->level0_keys = n;
                }
            }
            if (level == 0 && stats) {
                const ModelHdr& h0 = *C->hmodel.as<ModelHdr>();
                stats->level0_kind = h0.kind == kLearned ? 0 : 1;
            }
            if (stats) {
                stats->levels = level + 1;
                stats->segments += ns;
                uint64_t moved = 0;
                for (uint32_t i = 0; i < ns; ++i) moved += segs[i].n;
                stats->partitioned_keys += moved;
                stats->base_case_keys += hc->keys_base;
                stats->fill_keys += hc->keys_fill;
                stats->base_segments += (uint64_t)hc->n_base[0] + hc->n_base[1] + hc->n_base[2];
            }
            // ---- next level
            uint32_t nrec = hc->n_rec;
            segs.clear();
            if (nrec) {
                if (nrec > spec) {
                    if (!C->hrec.ensure(nrec * sizeof(SegOut))) throw LsortError{LSORT_ENOMEM, "host rec list"};
                    down(C->hrec.p, C->rec.p, nrec * sizeof(SegOut));
                    CU(cudaStreamSynchronize(st));
                }
                const SegOut* r = C->hrec.as<SegOut>();
                segs.reserve(nrec);
                for (uint32_t i = 0; i < nrec; ++i)
                    segs.push_back({r[i].begin, r[i].n, r[i].depth, r[i].flags,
                                    (C->psample.p || (fw && fw->psample)) ? r[i].pslice : 0});
                std::sort(segs.begin(), segs.end(),
                          [](const SegPlan& a, const SegPlan& b) { return a.begin < b.begin; });
            }
            // ping-pong: this level's output becomes the next level's input
            src = dst;
            src_f64 = false;
            dst = (dst == C->scratch.as<uint64_t>()) ? (uint64_t*)keys : C->scratch.as<uint64_t>();
            ++level;
            if (level > 64) throw LsortError{LSORT_EINTERNAL, "recursion did not terminate"};
        }
    }
};

constexpr uint32_t kManyWays = 3;  // concurrent sorts in lsort_cuda_sort_many

int fail(lsort_ctx* ctx, const LsortError& e) {
    if (ctx) ctx->err = e.msg;
    return e.code;
}

lsort_cfg cfg_or_default(const lsort_cfg* cfg) {
    lsort_cfg c;
    if (cfg) c = *cfg;
    else lsort_cfg_default(&c);
    return c;
}

}  // namespace

// ======================================================================= C-ABI
extern "C" {

void lsort_cfg_default(lsort_cfg* c) {
    std::memset(c, 0, sizeof(*c));
    c->rmi_bucket_count = 1024;
    c->tree_bucket_count = 256;
    c->min_rmi_input = 100000;
    c->max_duplicate_fraction = 0.10;
    c->radix_base_case = 4096;
    c->insertion_base_case = 16;
    c->first_sample_cap = 2 * 256 * 16;
    c->rmi_sample_cap = 1u << 20;
    c->sample_fraction = 0.01;
    c->seed = 0x5EEDull;
    c->workers = 0;
    c->base_case_capacity = 16384;
    c->bucket_target = 4096;
    c->flags = 0;
}

int lsort_cuda_ctx_create(lsort_ctx** out, int device, void* stream, size_t workspace_hint) {
    if (!out) return LSORT_EINVAL;
    *out = nullptr;
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) { cudaGetLastError(); return LSORT_ECUDA; }
    if (device < 0 || device >= ndev) return LSORT_EINVAL;
    if (cudaSetDevice(device) != cudaSuccess) return LSORT_ECUDA;
    lsort_ctx* c = new lsort_ctx();
    c->device = device;
    try {
        kernels_init();
        if (stream) c->stream = (cudaStream_t)stream;
        else {
            CU(cudaStreamCreateWithFlags(&c->own_stream, cudaStreamNonBlocking));
            c->stream = c->own_stream;
        }
        for (auto& e : c->ev) CU(cudaEventCreate(&e));
        for (auto& e : c->pev) CU(cudaEventCreate(&e));
        if (workspace_hint && !c->scratch.ensure(workspace_hint * 8)) throw LsortError{LSORT_ENOMEM, "workspace"};
    } catch (const LsortError& e) {
        delete c;
        return e.code;
    }
    *out = c;
    return LSORT_OK;
}

int lsort_cuda_ctx_destroy(lsort_ctx* c) {
    if (!c) return LSORT_OK;
    cudaSetDevice(c->device);
    delete c;  // ~lsort_ctx: drains the stream, frees lanes / nested contexts, events, own stream
    return LSORT_OK;
}

const char* lsort_cuda_last_error(const lsort_ctx* c) { return c ? c->err.c_str() : "null context"; }

int lsort_cuda_set_stream(lsort_ctx* c, void* stream) {
    if (!c) return LSORT_EINVAL;
    c->stream = stream ? (cudaStream_t)stream : c->own_stream;
    return LSORT_OK;
}

int lsort_cuda_sort(lsort_ctx* C, void* keys, uint64_t n, int key_kind, int mem_kind, const lsort_cfg* cfgp,
                    lsort_stats* stats, uint64_t* nan_index_out) {
    if (!C) return LSORT_EINVAL;
    C->err.clear();
    if (nan_index_out) *nan_index_out = ~0ull;
    if (key_kind != LSORT_KEY_U64 && key_kind != LSORT_KEY_F64 && key_kind != LSORT_KEY_ENC_F64)
        return fail(C, {LSORT_EINVAL, "key_kind"});
    if (mem_kind != LSORT_MEM_DEVICE && mem_kind != LSORT_MEM_HOST) return fail(C, {LSORT_EINVAL, "mem_kind"});
    if (n > 0 && !keys) return fail(C, {LSORT_EINVAL, "null keys"});
    lsort_cfg cfg = cfg_or_default(cfgp);
    if (stats) std::memset(stats, 0, sizeof(*stats));
    try {
        validate_cfg(cfg);
        CU(cudaSetDevice(C->device));
        const bool f64 = key_kind == LSORT_KEY_F64 || key_kind == LSORT_KEY_ENC_F64;
        const bool enc = key_kind == LSORT_KEY_ENC_F64;
        C->launches = 0;
        void* dkeys = keys;
        cudaStream_t st = C->stream;
        if (mem_kind == LSORT_MEM_HOST) {
            if (!C->data.ensure(std::max<uint64_t>(n, 1) * 8)) throw LsortError{LSORT_ENOMEM, "device keys"};
            dkeys = C->data.p;
            CU(cudaEventRecord(C->ev[2], st));
            CU(cudaMemcpyAsync(dkeys, keys, n * 8, cudaMemcpyHostToDevice, st));
            CU(cudaEventRecord(C->ev[3], st));
        }
        CU(cudaEventRecord(C->ev[0], st));
        Engine E(C, cfg);
        E.sort(dkeys, n, f64, stats, enc);
        CU(cudaEventRecord(C->ev[1], st));
        if (mem_kind == LSORT_MEM_HOST) {
            CU(cudaMemcpyAsync(keys, dkeys, n * 8, cudaMemcpyDeviceToHost, st));
            CU(cudaEventRecord(C->ev[4], st));
        }
        CU(cudaStreamSynchronize(st));
        if (stats) {
            float ms = 0;
            cudaEventElapsedTime(&ms, C->ev[0], C->ev[1]);
            stats->ms_total = ms;
            if (mem_kind == LSORT_MEM_HOST) {
                cudaEventElapsedTime(&ms, C->ev[2], C->ev[3]);
                stats->ms_h2d = ms;
                cudaEventElapsedTime(&ms, C->ev[1], C->ev[4]);
                stats->ms_d2h = ms;
                stats->h2d_bytes = n * 8;
                stats->d2h_bytes = n * 8;
            }
            stats->kernel_launches = C->launches;
        }
    } catch (const LsortError& e) {
        if (e.code == LSORT_ENAN) {
            if (nan_index_out) *nan_index_out = std::stoull(e.msg);
            C->err = "NaN at index " + e.msg;
            cudaStreamSynchronize(C->stream);
            return LSORT_ENAN;
        }
        cudaStreamSynchronize(C->stream);
        cudaGetLastError();
        return fail(C, e);
    }
    return LSORT_OK;
}

int lsort_cuda_sort_many(lsort_ctx* C, void* const* keys, const uint64_t* n, uint32_t count, int key_kind,
                         const lsort_cfg* cfgp, lsort_stats* stats, uint64_t* nan_index_out) {
    if (!C) return LSORT_EINVAL;
    C->err.clear();
    if (count && (!keys || !n)) return fail(C, {LSORT_EINVAL, "null batch"});
    if (key_kind != LSORT_KEY_U64 && key_kind != LSORT_KEY_F64) return fail(C, {LSORT_EINVAL, "key_kind"});
    for (uint32_t i = 0; i < count; ++i) {
        if (nan_index_out) nan_index_out[i] = ~0ull;
        if (n[i] > 0 && !keys[i]) return fail(C, {LSORT_EINVAL, "null keys"});
    }
    lsort_cfg cfg = cfg_or_default(cfgp);
    if (stats) std::memset(stats, 0, sizeof(*stats));
    try {
        validate_cfg(cfg);
        CU(cudaSetDevice(C->device));
    } catch (const LsortError& e) {
        return fail(C, e);
    }
    const bool f64 = key_kind == LSORT_KEY_F64;
    const uint32_t nt = std::min<uint32_t>(count, kManyWays);
    try {
        CU(cudaStreamSynchronize(C->stream));  // work the caller queued on the context stream comes first
        while (C->subs.size() < nt) {
            std::unique_ptr<lsort_ctx> s(new lsort_ctx());
            s->device = C->device;
            CU(cudaStreamCreateWithFlags(&s->own_stream, cudaStreamNonBlocking));
            s->stream = s->own_stream;
            for (auto& e : s->ev) CU(cudaEventCreate(&e));
            for (auto& e : s->pev) CU(cudaEventCreate(&e));
            C->subs.push_back(std::move(s));
        }
    } catch (const LsortError& e) {
        return fail(C, e);
    }
    std::atomic<uint32_t> next{0};
    std::mutex mu;
    LsortError first_err{LSORT_OK, ""};
    bool any_nan = false;
    auto worker = [&](uint32_t t) {
        lsort_ctx* S = C->subs[t].get();
        cudaSetDevice(S->device);
        for (uint32_t i = next++; i < count; i = next++) {
            lsort_stats sti;
            std::memset(&sti, 0, sizeof(sti));
            try {
                S->launches = 0;
                Engine E(S, cfg);
                E.sort(keys[i], n[i], f64, stats ? &sti : nullptr);
                CU(cudaStreamSynchronize(S->stream));
            } catch (const LsortError& e) {
                cudaStreamSynchronize(S->stream);
                std::lock_guard<std::mutex> g(mu);
                if (e.code == LSORT_ENAN) {
                    any_nan = true;
                    if (nan_index_out) nan_index_out[i] = std::stoull(e.msg);
                } else if (first_err.code == LSORT_OK) {
                    first_err = e;
                }
                continue;
            }
            if (stats) {
                std::lock_guard<std::mutex> g(mu);
                stats->levels += sti.levels;  // summed over the arrays (per-array levels = levels / count)
                stats->partitioned_keys += sti.partitioned_keys;
                stats->base_case_keys += sti.base_case_keys;
                stats->fill_keys += sti.fill_keys;
                stats->segments += sti.segments;
                stats->base_segments += sti.base_segments;
                stats->kernel_launches += S->launches;
                stats->ms_models += sti.ms_models;
                stats->ms_classify += sti.ms_classify;
                stats->ms_scatter += sti.ms_scatter;
                stats->ms_base += sti.ms_base;
                stats->ms_fill += sti.ms_fill;
            }
        }
    };
    std::vector<std::thread> th;
    for (uint32_t t = 1; t < nt; ++t) th.emplace_back(worker, t);
    if (nt) worker(0);
    for (auto& x : th) x.join();
    if (first_err.code != LSORT_OK) return fail(C, first_err);
    if (any_nan) {
        C->err = "NaN in batch";
        return LSORT_ENAN;
    }
    return LSORT_OK;
}

int lsort_cuda_sort_batch(lsort_ctx* C, void* const* keys, const uint64_t* n, uint32_t count, int key_kind,
                          const lsort_cfg* cfgp, lsort_stats* stats, uint64_t* nan_index_out) {
    if (!C) return LSORT_EINVAL;
    C->err.clear();
    if (count && (!keys || !n)) return fail(C, {LSORT_EINVAL, "null batch"});
    if (key_kind != LSORT_KEY_U64 && key_kind != LSORT_KEY_F64) return fail(C, {LSORT_EINVAL, "key_kind"});
    for (uint32_t i = 0; i < count; ++i) {
        if (nan_index_out) nan_index_out[i] = ~0ull;
        if (n[i] > 0 && !keys[i]) return fail(C, {LSORT_EINVAL, "null keys"});
    }
    lsort_cfg cfg = cfg_or_default(cfgp);
    if (stats) std::memset(stats, 0, sizeof(*stats));
    bool any_nan = false;
    try {
        validate_cfg(cfg);
        CU(cudaSetDevice(C->device));
        const bool f64 = key_kind == LSORT_KEY_F64;
        uint64_t nmax = 1;
        for (uint32_t i = 0; i < count; ++i) nmax = std::max(nmax, n[i]);
        const uint32_t slots = std::min<uint32_t>(3, std::max<uint32_t>(count, 1));
        for (uint32_t s = 0; s < slots; ++s)
            if (!C->bat[s].ensure(nmax * 8)) throw LsortError{LSORT_ENOMEM, "batch buffers"};
        if (!C->h2d_stream) CU(cudaStreamCreateWithFlags(&C->h2d_stream, cudaStreamNonBlocking));
        if (!C->d2h_stream) CU(cudaStreamCreateWithFlags(&C->d2h_stream, cudaStreamNonBlocking));
        for (auto& e : C->bev)
            if (!e) CU(cudaEventCreate(&e));
        cudaEvent_t* ev_h2d = C->bev;
        cudaEvent_t* ev_sorted = C->bev + 3;
        cudaEvent_t* ev_d2h = C->bev + 6;
        if (!C->hstage.ensure(1u << 20)) throw LsortError{LSORT_ENOMEM, "staging"};
        C->zero_copy = true;  // the copy engines stream the arrays: control traffic goes by kernels
        CU(cudaEventRecord(C->bev[9], C->h2d_stream));
        std::vector<bool> used(slots, false);
        auto issue_h2d = [&](uint32_t i) {
            const uint32_t s = i % slots;
            if (used[s]) CU(cudaStreamWaitEvent(C->h2d_stream, ev_d2h[s], 0));  // slot's previous copy-out
            CU(cudaMemcpyAsync(C->bat[s].p, keys[i], n[i] * 8, cudaMemcpyHostToDevice, C->h2d_stream));
            CU(cudaEventRecord(ev_h2d[s], C->h2d_stream));
            used[s] = true;
        };
        for (uint32_t i = 0; i < std::min(count, slots - 1); ++i) issue_h2d(i);
        lsort_stats sti;
        for (uint32_t i = 0; i < count; ++i) {
            if (i + slots - 1 < count) issue_h2d(i + slots - 1);
            const uint32_t s = i % slots;
            CU(cudaStreamWaitEvent(C->stream, ev_h2d[s], 0));
            bool nan = false;
            try {
                std::memset(&sti, 0, sizeof(sti));
                C->launches = 0;
                Engine E(C, cfg);
                E.sort(C->bat[s].p, n[i], f64, stats ? &sti : nullptr);
            } catch (const LsortError& e) {
                if (e.code != LSORT_ENAN) throw;
                nan = any_nan = true;
                if (nan_index_out) nan_index_out[i] = std::stoull(e.msg);
            }
            CU(cudaEventRecord(ev_sorted[s], C->stream));
            CU(cudaStreamWaitEvent(C->d2h_stream, ev_sorted[s], 0));
            if (!nan) CU(cudaMemcpyAsync(keys[i], C->bat[s].p, n[i] * 8, cudaMemcpyDeviceToHost, C->d2h_stream));
            CU(cudaEventRecord(ev_d2h[s], C->d2h_stream));
            if (stats) {
                stats->levels += sti.levels;  // summed over the arrays (per-array levels = levels / count)
                stats->partitioned_keys += sti.partitioned_keys;
                stats->base_case_keys += sti.base_case_keys;
                stats->fill_keys += sti.fill_keys;
                stats->segments += sti.segments;
                stats->base_segments += sti.base_segments;
                stats->kernel_launches += C->launches;
                stats->h2d_bytes += n[i] * 8;
                stats->d2h_bytes += nan ? 0 : n[i] * 8;
                stats->ms_models += sti.ms_models;
                stats->ms_classify += sti.ms_classify;
                stats->ms_scatter += sti.ms_scatter;
                stats->ms_base += sti.ms_base;
                stats->ms_fill += sti.ms_fill;
            }
        }
        CU(cudaStreamWaitEvent(C->d2h_stream, C->bev[9], 0));
        CU(cudaEventRecord(C->bev[10], C->d2h_stream));
        CU(cudaStreamSynchronize(C->d2h_stream));
        CU(cudaStreamSynchronize(C->h2d_stream));
        CU(cudaStreamSynchronize(C->stream));
        CU(cudaGetLastError());
        if (stats) {
            float ms = 0;
            cudaEventElapsedTime(&ms, C->bev[9], C->bev[10]);
            stats->ms_total = ms;
        }
        C->zero_copy = false;
    } catch (const LsortError& e) {
        C->zero_copy = false;
        if (C->h2d_stream) cudaStreamSynchronize(C->h2d_stream);
        if (C->d2h_stream) cudaStreamSynchronize(C->d2h_stream);
        cudaStreamSynchronize(C->stream);
        cudaGetLastError();
        return fail(C, e);
    }
    if (any_nan) {
        C->err = "NaN in batch";
        return LSORT_ENAN;
    }
    return LSORT_OK;
}

// ---------------------------------------------------------------- unit entries
static void upload_learned(lsort_ctx* C, const lsort_rmi_header* h, const lsort_rmi_entry* e, uint32_t bucket_count,
                           double cdf_lo, double cdf_hi) {
    uint32_t B = h->submodels;
    size_t bytes = sizeof(ModelHdr) + kLearnedEntryBytes * (size_t)B;
    if (!C->models.ensure(bytes) || !C->hmodel.ensure(bytes)) throw LsortError{LSORT_ENOMEM, "model"};
    ModelHdr* m = C->hmodel.as<ModelHdr>();
    std::memset(m, 0, sizeof(ModelHdr));
    m->kind = kLearned;
    m->nbuckets = bucket_count;
    m->B = B;
    m->root_slope = h->root_slope;
    m->root_icpt = h->root_intercept;
    m->key_base = h->key_base;
    m->key_scale = h->key_scale;
    double span = cdf_hi - cdf_lo;  // Learned::inv_span (models.hpp:134-137)
    m->cdf_lo = cdf_lo;
    m->inv_span = span > 0.0 ? 1.0 / span : 0.0;
    std::memcpy((uint8_t*)m + sizeof(ModelHdr), e, 32 * (size_t)B);
    // compiled table (lsort_device.cuh RmiBucketEntry), same arithmetic as compile_learned
    auto gb = [&](double v) -> uint32_t {
        if (v < 0.0) v = 0.0;
        if (v > 1.0) v = 1.0;
        double t = ((v - m->cdf_lo) * m->inv_span) * (double)bucket_count;
        if (!(t > 0.0)) return 0;
        if (t >= (double)bucket_count) return bucket_count - 1;
        return (uint32_t)t;
    };
    RmiBucketEntry* cb = (RmiBucketEntry*)((uint8_t*)m + sizeof(ModelHdr) + 32 * (size_t)B);
    for (uint32_t i = 0; i < B; ++i) {
        cb[i].slope = e[i].slope;
        cb[i].intercept = e[i].intercept;
        cb[i].glo = gb(e[i].lo);
        cb[i].ghi = gb(e[i].hi);
        cb[i].pad = 0;
    }
    m->flags = (m->cdf_lo == 0.0 && m->inv_span == 1.0) ? kModelIdentityCdf : 0u;
    CU(cudaMemcpyAsync(C->models.p, m, bytes, cudaMemcpyHostToDevice, C->stream));
}

static size_t upload_tree(lsort_ctx* C, const lsort_tree* t) {
    size_t payload = (tree_payload_bytes(t->leaf_origin, t->nsplitters) + 15) & ~15ull;
    size_t bytes = sizeof(ModelHdr) + payload;
    if (!C->models.ensure(bytes) || !C->hmodel.ensure(bytes)) throw LsortError{LSORT_ENOMEM, "model"};
    ModelHdr* m = C->hmodel.as<ModelHdr>();
    std::memset(m, 0, bytes);
    m->kind = kTree;
    m->nbuckets = t->bucket_count;
    m->levels = t->levels;
    m->leaf_origin = t->leaf_origin;
    m->nsplit = t->nsplitters;
    uint64_t* tree = (uint64_t*)((uint8_t*)m + sizeof(ModelHdr));
    std::memcpy(tree, t->tree, 8 * (size_t)t->leaf_origin);
    std::memcpy(tree + t->leaf_origin, t->splitters, 8 * (size_t)t->nsplitters);
    std::memcpy(tree + t->leaf_origin + t->nsplitters, t->eq_offset, 4 * ((size_t)t->nsplitters + 1));
    CU(cudaMemcpyAsync(C->models.p, m, bytes, cudaMemcpyHostToDevice, C->stream));
    return payload;
}

static void download_tree(lsort_ctx* C, const uint8_t* dmodel, lsort_tree* out) {
    if (!C->hmodel.ensure(sizeof(ModelHdr) + 24 * LSORT_MAX_TREE)) throw LsortError{LSORT_ENOMEM, "host model"};
    CU(cudaMemcpyAsync(C->hmodel.p, dmodel, sizeof(ModelHdr) + 20 * LSORT_MAX_TREE + 16, cudaMemcpyDeviceToHost,
                       C->stream));
    CU(cudaStreamSynchronize(C->stream));
    const ModelHdr* m = C->hmodel.as<ModelHdr>();
    std::memset(out, 0, sizeof(*out));
    out->levels = m->levels;
    out->leaf_origin = m->leaf_origin;
    out->nsplitters = m->nsplit;
    out->bucket_count = m->nbuckets;
    const uint64_t* tree = (const uint64_t*)((const uint8_t*)m + sizeof(ModelHdr));
    std::memcpy(out->tree, tree, 8 * (size_t)m->leaf_origin);
    std::memcpy(out->splitters, tree + m->leaf_origin, 8 * (size_t)m->nsplit);
    std::memcpy(out->eq_offset, tree + m->leaf_origin + m->nsplit, 4 * ((size_t)m->nsplit + 1));
}

static void download_learned(lsort_ctx* C, const uint8_t* dmodel, uint32_t B, lsort_rmi_header* h,
                             lsort_rmi_entry* e) {
    size_t bytes = sizeof(ModelHdr) + 32 * (size_t)B;
    if (!C->hmodel.ensure(bytes)) throw LsortError{LSORT_ENOMEM, "host model"};
    CU(cudaMemcpyAsync(C->hmodel.p, dmodel, bytes, cudaMemcpyDeviceToHost, C->stream));
    CU(cudaStreamSynchronize(C->stream));
    const ModelHdr* m = C->hmodel.as<ModelHdr>();
    if (h) {
        h->root_slope = m->root_slope;
        h->root_intercept = m->root_icpt;
        h->key_base = m->key_base;
        h->key_scale = m->key_scale;
        h->submodels = m->B;
        h->reserved = 0;
    }
    if (e) std::memcpy(e, (const uint8_t*)m + sizeof(ModelHdr), 32 * (size_t)B);
}

int lsort_cuda_rmi_train(lsort_ctx* C, const uint64_t* d_sample, uint64_t s, uint32_t B, lsort_rmi_header* h_out,
                         lsort_rmi_entry* e_out) {
    if (!C) return LSORT_EINVAL;
    if (s < 2 || B == 0) return fail(C, {LSORT_EINVAL, "Rmi::train: sample must hold at least 2 keys / B > 0"});
    if (B > LSORT_MAX_RMI || s > 0xffffffffull) return fail(C, {LSORT_EINVAL, "Rmi::train: size limits"});
    try {
        CU(cudaSetDevice(C->device));
        if (!C->models.ensure(sizeof(ModelHdr) + kLearnedEntryBytes * (size_t)B) ||
            !C->train_ws.ensure(train_workspace_bytes(s, B)))
            throw LsortError{LSORT_ENOMEM, "model"};
        CU(cudaMemsetAsync(C->models.p, 0, sizeof(ModelHdr), C->stream));
        launch_train_rmi(d_sample, s, B, C->models.as<uint8_t>(), B, C->train_ws.p, nullptr, C->stream);
        CU(cudaGetLastError());
        download_learned(C, C->models.as<uint8_t>(), B, h_out, e_out);
    } catch (const LsortError& e) {
        return fail(C, e);
    }
    return LSORT_OK;
}

int lsort_cuda_classify_rmi(lsort_ctx* C, const lsort_rmi_header* h, const lsort_rmi_entry* e, uint32_t bucket_count,
                            double cdf_lo, double cdf_hi, const void* d_keys, uint64_t n, int key_kind,
                            uint32_t* d_ids, uint64_t* d_hist) {
    if (!C || !h || !e || bucket_count == 0 || h->submodels == 0 || h->submodels > LSORT_MAX_RMI)
        return fail(C, {LSORT_EINVAL, "classify_rmi: bad model"});
    try {
        CU(cudaSetDevice(C->device));
        upload_learned(C, h, e, bucket_count, cdf_lo, cdf_hi);
        if (d_hist) CU(cudaMemsetAsync(d_hist, 0, 8 * (size_t)bucket_count, C->stream));
        if (n) launch_classify_ids(C->models.as<uint8_t>(), d_keys, n, key_kind == LSORT_KEY_F64, d_ids, nullptr,
                                   (unsigned long long*)d_hist, (int)kLearnedEntryBytes * (int)h->submodels, C->stream);
        CU(cudaStreamSynchronize(C->stream));
        CU(cudaGetLastError());
    } catch (const LsortError& er) {
        return fail(C, er);
    }
    return LSORT_OK;
}

int lsort_cuda_tree_build(lsort_ctx* C, const uint64_t* d_sample, uint64_t s, uint32_t budget, int eq_mode,
                          lsort_tree* out) {
    if (!C || !out) return LSORT_EINVAL;
    if (s == 0) return fail(C, {LSORT_EINVAL, "SplitterTree::build: sample must not be empty"});
    if (budget < 2 || (budget & (budget - 1)) || budget > LSORT_MAX_TREE)
        return fail(C, {LSORT_EINVAL, "SplitterTree::build: bucket budget must be a power of two >= 2"});
    if (s > 16384) return fail(C, {LSORT_EINVAL, "SplitterTree::build: GPU sample limit 16384"});
    try {
        CU(cudaSetDevice(C->device));
        if (!C->models.ensure(sizeof(ModelHdr) + 24 * LSORT_MAX_TREE + 16)) throw LsortError{LSORT_ENOMEM, "model"};
        launch_tree_build(d_sample, s, budget, eq_mode, C->models.as<uint8_t>(), C->stream);
        CU(cudaGetLastError());
        download_tree(C, C->models.as<uint8_t>(), out);
    } catch (const LsortError& e) {
        return fail(C, e);
    }
    return LSORT_OK;
}

int lsort_cuda_classify_tree(lsort_ctx* C, const lsort_tree* t, const void* d_keys, uint64_t n, int key_kind,
                             uint32_t* d_ids, uint64_t* d_hist) {
    if (!C || !t || t->leaf_origin == 0 || t->leaf_origin > LSORT_MAX_TREE) return LSORT_EINVAL;
    try {
        CU(cudaSetDevice(C->device));
        size_t payload = upload_tree(C, t);
        if (d_hist) CU(cudaMemsetAsync(d_hist, 0, 8 * (size_t)t->bucket_count, C->stream));
        if (n) launch_classify_ids(C->models.as<uint8_t>(), d_keys, n, key_kind == LSORT_KEY_F64, d_ids, nullptr,
                                   (unsigned long long*)d_hist, (int)payload, C->stream);
        CU(cudaStreamSynchronize(C->stream));
        CU(cudaGetLastError());
    } catch (const LsortError& er) {
        return fail(C, er);
    }
    return LSORT_OK;
}

int lsort_cuda_build_model(lsort_ctx* C, const void* d_keys, uint64_t n, int key_kind, const lsort_cfg* cfgp,
                           lsort_model_info* info, lsort_rmi_header* h_out, lsort_rmi_entry* e_out,
                           lsort_tree* tree_out) {
    if (!C) return LSORT_EINVAL;
    if (n < 2) return fail(C, {LSORT_EINVAL, "build_model: n < 2"});
    lsort_cfg cfg = cfg_or_default(cfgp);
    cfg.flags |= LSORT_FLAG_STRICT_POLICY;  // the reference's Alg. 5 model, unit-for-unit
    try {
        validate_cfg(cfg);
        CU(cudaSetDevice(C->device));
        Engine E(C, cfg);
        SegPlan sp{0, n, 0, 0};
        SegDesc d{};
        d.begin = 0;
        d.n = n;
        d.rmi_b = E.rmi_b(n);
        d.tree_k = E.tree_k(n);
        d.model_off = 0;
        size_t bytes = sizeof(ModelHdr) + std::max<size_t>(kLearnedEntryBytes * (size_t)d.rmi_b, 24 * LSORT_MAX_TREE + 16);
        if (!C->models.ensure(bytes) || !C->segs.ensure(sizeof(SegDesc)) || !C->idx.ensure(4))
            throw LsortError{LSORT_ENOMEM, "model"};
        CU(cudaMemsetAsync(C->models.p, 0, bytes, C->stream));
        CU(cudaMemcpyAsync(C->segs.p, &d, sizeof(d), cudaMemcpyHostToDevice, C->stream));
        uint32_t zero = 0;
        CU(cudaMemcpyAsync(C->idx.p, &zero, 4, cudaMemcpyHostToDevice, C->stream));
        const bool f64 = key_kind == LSORT_KEY_F64;
        const int mc = E.model_class(sp);
        if (mc == 2) E.big_models({0u}, C->segs.as<SegDesc>(), {sp}, &d, d_keys, f64);
        else launch_build_models(C->segs.as<SegDesc>(), C->idx.as<uint32_t>(), 1, d_keys, f64,
                                 C->models.as<uint8_t>(), dev_cfg(cfg), mc, C->stream);
        CU(cudaStreamSynchronize(C->stream));
        CU(cudaGetLastError());
        ModelHdr h;
        CU(cudaMemcpy(&h, C->models.p, sizeof(h), cudaMemcpyDeviceToHost));
        if (info) {
            info->kind = h.kind;
            info->nbuckets = h.nbuckets;
            info->first_sample = h.s1;
            info->rmi_sample = h.kind == kLearned ? h.s2 : 0;
            info->duplicate_fraction = h.dup;
        }
        if (h.kind == kLearned) download_learned(C, C->models.as<uint8_t>(), h.B, h_out, e_out);
        else if (tree_out) download_tree(C, C->models.as<uint8_t>(), tree_out);
    } catch (const LsortError& e) {
        return fail(C, e);
    }
    return LSORT_OK;
}

int lsort_cuda_block_sort(lsort_ctx* C, uint64_t* d_keys, uint64_t n) {
    if (!C) return LSORT_EINVAL;
    if (n > kSmallSampleCap) return fail(C, {LSORT_EINVAL, "block sort holds at most 8192 keys"});
    try {
        CU(cudaSetDevice(C->device));
        if (n > 1) launch_block_sort(d_keys, n, C->stream);
        CU(cudaStreamSynchronize(C->stream));
        CU(cudaGetLastError());
    } catch (const LsortError& e) {
        return fail(C, e);
    }
    return LSORT_OK;
}

// ------------------------------------------------------------ pivot analysis
// keys.hpp:24-32 on the host, on bit patterns: f64 bits -> encoded key and back
static inline uint64_t encode_host(uint64_t bits) {
    return (bits >> 63) ? ~bits : (bits ^ 0x8000000000000000ull);
}
static inline uint64_t decode_bits_host(uint64_t k) {
    return (k >> 63) ? (k ^ 0x8000000000000000ull) : ~k;
}
int lsort_cuda_learned_pivots(lsort_ctx* C, const lsort_rmi_header* h, const lsort_rmi_entry* e, uint32_t b,
                              const void* d_keys, uint64_t n, int key_kind, uint64_t* pivots_out,
                              uint32_t* cells_out, uint32_t* count_out) {
    if (!C || !h || !e || !pivots_out || !count_out || b < 2 || b > kMaxNB || h->submodels == 0 ||
        h->submodels > LSORT_MAX_RMI || (key_kind != LSORT_KEY_U64 && key_kind != LSORT_KEY_F64))
        return fail(C, {LSORT_EINVAL, "learned_pivots: bad arguments"});
    try {
        CU(cudaSetDevice(C->device));
        const size_t bytes = 12 * (size_t)b;
        // host staging sized first: upload_learned copies from it asynchronously
        const size_t mb = sizeof(ModelHdr) + kLearnedEntryBytes * (size_t)h->submodels;
        if (!C->piv.ensure(bytes) || !C->hmodel.ensure(std::max(bytes, mb))) throw LsortError{LSORT_ENOMEM, "pivots"};
        upload_learned(C, h, e, b, 0.0, 1.0);
        unsigned long long* gmax = C->piv.as<unsigned long long>();
        unsigned int* ghit = (unsigned int*)(gmax + b);
        CU(cudaMemsetAsync(C->piv.p, 0, bytes, C->stream));
        if (n) launch_learned_pivots(C->models.as<uint8_t>(), d_keys, n, key_kind == LSORT_KEY_F64, gmax, ghit,
                                     (int)kLearnedEntryBytes * (int)h->submodels, C->stream);
        CU(cudaStreamSynchronize(C->stream));  // the model upload's staging buffer is reused below
        CU(cudaMemcpy(C->hmodel.p, C->piv.p, bytes, cudaMemcpyDeviceToHost));
        CU(cudaGetLastError());
        const uint64_t* hm = C->hmodel.as<uint64_t>();
        const uint32_t* hh = (const uint32_t*)(hm + b);
        uint32_t np = 0;
        uint64_t last = 0;
        for (uint32_t i = 0; i + 1 < b; ++i) {  // cells 0..b-2: boundaries (i+1)/b
            if (!hh[i] || (np && hm[i] <= last)) continue;
            last = hm[i];
            if (cells_out) cells_out[np] = i;
            pivots_out[np++] = key_kind == LSORT_KEY_F64 ? decode_bits_host(hm[i]) : hm[i];
        }
        *count_out = np;
    } catch (const LsortError& er) {
        return fail(C, er);
    }
    return LSORT_OK;
}

static void pivot_ranks(lsort_ctx* C, const void* d_sorted, uint64_t n, int key_kind, const uint64_t* pivots,
                        uint32_t np, uint64_t* ranks) {
    if (!C->piv.ensure(16 * (size_t)np + 16) || !C->hmodel.ensure(16 * (size_t)np + 16))
        throw LsortError{LSORT_ENOMEM, "pivots"};
    uint64_t* hp = C->hmodel.as<uint64_t>();
    for (uint32_t i = 0; i < np; ++i) hp[i] = key_kind == LSORT_KEY_F64 ? encode_host(pivots[i]) : pivots[i];
    uint64_t* dp = C->piv.as<uint64_t>();
    CU(cudaMemcpyAsync(dp, hp, 8 * (size_t)np, cudaMemcpyHostToDevice, C->stream));
    launch_rank_le(d_sorted, n, key_kind == LSORT_KEY_F64, dp, np, dp + np, C->stream);
    CU(cudaMemcpyAsync(ranks, dp + np, 8 * (size_t)np, cudaMemcpyDeviceToHost, C->stream));
    CU(cudaStreamSynchronize(C->stream));
    CU(cudaGetLastError());
}

int lsort_cuda_pivot_quality(lsort_ctx* C, const void* d_sorted, uint64_t n, int key_kind, const uint64_t* pivots,
                             uint32_t np, uint32_t b, double* distance_out, uint64_t* ranks_out) {
    if (!C || !distance_out || (np && !pivots) || n == 0 ||
        (key_kind != LSORT_KEY_U64 && key_kind != LSORT_KEY_F64))
        return fail(C, {LSORT_EINVAL, "pivot_quality: bad arguments"});
    if ((uint64_t)np + 1 != b) return fail(C, {LSORT_EINVAL, "pivot_quality: pivot count + 1 != b"});
    try {
        CU(cudaSetDevice(C->device));
        std::vector<uint64_t> r(np ? np : 1);
        if (np) pivot_ranks(C, d_sorted, n, key_kind, pivots, np, r.data());
        double d = 0.0;  // summed in pivot order, as the oracle does
        for (uint32_t i = 0; i < np; ++i) {
            const double c = (double)r[i] / (double)n, t = (double)(i + 1) / (double)b;
            d += c > t ? c - t : t - c;
        }
        *distance_out = d;
        if (ranks_out) std::memcpy(ranks_out, r.data(), 8 * (size_t)np);
    } catch (const LsortError& er) {
        return fail(C, er);
    }
    return LSORT_OK;
}

int lsort_cuda_eta(lsort_ctx* C, const void* d_sorted, uint64_t n, int key_kind, uint64_t pivot, double* eta_out) {
    if (!C || !eta_out || n == 0 || (key_kind != LSORT_KEY_U64 && key_kind != LSORT_KEY_F64))
        return fail(C, {LSORT_EINVAL, "eta: bad arguments"});
    try {
        CU(cudaSetDevice(C->device));
        uint64_t r = 0;
        pivot_ranks(C, d_sorted, n, key_kind, &pivot, 1, &r);
        const double c = (double)r / (double)n, o = 1.0 - c;
        *eta_out = (c > o ? c : o) - 0.5;
    } catch (const LsortError& er) {
        return fail(C, er);
    }
    return LSORT_OK;
}

int lsort_cuda_verify(lsort_ctx* C, const void* d_keys, uint64_t n, int key_kind, uint64_t* first_violation,
                      uint64_t* hash) {
    if (!C) return LSORT_EINVAL;
    try {
        CU(cudaSetDevice(C->device));
        if (!C->ctrl.ensure(sizeof(Ctrl)) || !C->hctrl.ensure(sizeof(Ctrl))) throw LsortError{LSORT_ENOMEM, "ctrl"};
        Ctrl* d = C->ctrl.as<Ctrl>();
        CU(cudaMemsetAsync(d, 0, sizeof(Ctrl), C->stream));
        CU(cudaMemsetAsync(&d->verify_first, 0xff, 8, C->stream));
        if (n) launch_verify(d_keys, n, key_kind == LSORT_KEY_F64, d, C->stream);
        CU(cudaMemcpyAsync(C->hctrl.p, d, sizeof(Ctrl), cudaMemcpyDeviceToHost, C->stream));
        CU(cudaStreamSynchronize(C->stream));
        CU(cudaGetLastError());
        const Ctrl* h = C->hctrl.as<Ctrl>();
        if (first_violation) *first_violation = h->verify_first == ~0ull ? 0 : h->verify_first;
        if (hash) *hash = h->verify_hash;
    } catch (const LsortError& e) {
        return fail(C, e);
    }
    return LSORT_OK;
}

int lsort_cuda_decode_inplace(lsort_ctx* C, uint64_t* d_keys, uint64_t n) {
    if (!C) return LSORT_EINVAL;
    try {
        CU(cudaSetDevice(C->device));
        if (n) launch_decode(d_keys, n, C->stream);
        CU(cudaStreamSynchronize(C->stream));
        CU(cudaGetLastError());
    } catch (const LsortError& e) {
        return fail(C, e);
    }
    return LSORT_OK;
}

// ------------------------------------------------------------ multi-GPU phases
int lsort_cuda_dist_sample(lsort_ctx* C, const void* d_keys, uint64_t n, int key_kind, uint64_t seed, uint64_t s,
                           uint64_t* d_out) {
    if (!C || n == 0) return LSORT_EINVAL;
    try {
        CU(cudaSetDevice(C->device));
        SegDesc d{};
        d.begin = 0;
        d.n = n;
        if (!C->segs.ensure(sizeof(SegDesc))) throw LsortError{LSORT_ENOMEM, "seg"};
        CU(cudaMemcpyAsync(C->segs.p, &d, sizeof(d), cudaMemcpyHostToDevice, C->stream));
        if (s) launch_gather(C->segs.as<SegDesc>(), d_keys, key_kind == LSORT_KEY_F64, seed, 0, s, d_out, nullptr,
                             C->stream);
        CU(cudaStreamSynchronize(C->stream));
        CU(cudaGetLastError());
    } catch (const LsortError& e) {
        return fail(C, e);
    }
    return LSORT_OK;
}

int lsort_cuda_dist_train(lsort_ctx* C, uint64_t* d_sample, uint64_t s, uint32_t buckets, lsort_rmi_header* h_out,
                          lsort_rmi_entry* e_out) {
    if (!C || s < 2 || buckets < 2 || buckets > LSORT_MAX_RMI) return LSORT_EINVAL;
    try {
        CU(cudaSetDevice(C->device));
        lsort_cfg cfg;
        lsort_cfg_default(&cfg);
        Engine E(C, cfg);
        E.nested_sort(d_sample, s);
        if (!C->models.ensure(sizeof(ModelHdr) + kLearnedEntryBytes * (size_t)buckets) ||
            !C->train_ws.ensure(train_workspace_bytes(s, buckets)))
            throw LsortError{LSORT_ENOMEM, "model"};
        launch_train_rmi(d_sample, s, buckets, C->models.as<uint8_t>(), buckets, C->train_ws.p, nullptr, C->stream);
        CU(cudaGetLastError());
        download_learned(C, C->models.as<uint8_t>(), buckets, h_out, e_out);
    } catch (const LsortError& e) {
        return fail(C, e);
    }
    return LSORT_OK;
}

}  // extern "C"

namespace {
uint64_t model_fingerprint(const lsort_rmi_header* h, const lsort_rmi_entry* e) {
    uint64_t f = splitmix64(h->submodels);
    auto mix = [&](const void* p, size_t bytes) {
        const uint64_t* w = (const uint64_t*)p;
        for (size_t i = 0; i < bytes / 8; ++i) f = splitmix64(f ^ w[i]);
    };
    mix(&h->root_slope, 8);
    mix(&h->root_intercept, 8);
    mix(&h->key_base, 8);
    mix(&h->key_scale, 8);
    mix(e, 32 * (size_t)h->submodels);
    return f;
}

// One learned segment over all n keys: LevelParams with a one-entry kind plan
// (the level-0 classify / scatter kernels of the single-GPU sort).
LevelParams dist_level(lsort_ctx* C, const void* d_keys, uint64_t n, uint32_t B, unsigned long long* counters,
                       uint64_t* d_out) {
    if (!C->segs.ensure(sizeof(SegDesc)) || !C->tile_prefix.ensure(16) || !C->ctrl.ensure(sizeof(Ctrl)) ||
        !C->kseg.ensure(16) || !C->ktp.ensure(64) || !C->kplan.ensure(3 * sizeof(KindPlan)) ||
        !C->ids.ensure(2 * std::max<uint64_t>(n, 1)))
        throw LsortError{LSORT_ENOMEM, "dist"};
    SegDesc d{};
    d.begin = 0;
    d.n = n;
    d.model_off = 0;
    d.bucket_off = 0;
    d.rmi_b = B;
    d.nb_max = B;
    const uint64_t ntiles = (n + kTileKeys - 1) / kTileKeys;
    uint64_t pref[2] = {0, ntiles};
    KindPlan kp[3] = {{1, 0, ntiles}, {0, 0, 0}, {0, 0, 0}};
    uint32_t k0 = 0;
    CU(cudaMemcpyAsync(C->segs.p, &d, sizeof(d), cudaMemcpyHostToDevice, C->stream));
    CU(cudaMemcpyAsync(C->tile_prefix.p, pref, 16, cudaMemcpyHostToDevice, C->stream));
    CU(cudaMemcpyAsync(C->kseg.p, &k0, 4, cudaMemcpyHostToDevice, C->stream));
    CU(cudaMemcpyAsync(C->ktp.p, pref, 16, cudaMemcpyHostToDevice, C->stream));
    CU(cudaMemcpyAsync(C->kplan.p, kp, sizeof(kp), cudaMemcpyHostToDevice, C->stream));
    CU(cudaMemsetAsync(C->ctrl.p, 0, sizeof(Ctrl), C->stream));
    CU(cudaMemsetAsync(&C->ctrl.as<Ctrl>()->nan_index, 0xff, 8, C->stream));
    LevelParams p{};
    p.segs = C->segs.as<SegDesc>();
    p.nsegs = 1;
    p.tile_prefix = C->tile_prefix.as<uint64_t>();
    p.ntiles = ntiles;
    p.models = C->models.as<uint8_t>();
    p.buckets = counters;
    p.src = d_keys;
    p.dst = d_out;
    p.ids = C->ids.as<uint16_t>();
    p.ctrl = C->ctrl.as<Ctrl>();
    p.kseg = C->kseg.as<uint32_t>();
    p.ktp = C->ktp.as<uint64_t>();
    p.kplan = C->kplan.as<KindPlan>();
    p.kstride = 1;
    return p;
}

// classify + histogram (d_hist, zeroed here) + bucket ids in C->ids
void dist_hist_ids(lsort_ctx* C, const void* d_keys, uint64_t n, int key_kind, const lsort_rmi_header* h,
                   const lsort_rmi_entry* e, unsigned long long* d_hist) {
    const uint32_t B = h->submodels;
    upload_learned(C, h, e, B, 0.0, 1.0);
    CU(cudaMemsetAsync(d_hist, 0, 8 * (size_t)B, C->stream));
    LevelParams p = dist_level(C, d_keys, n, B, d_hist, nullptr);
    const int grid = (int)std::max<uint64_t>(1, std::min<uint64_t>(p.ntiles, (uint64_t)num_sms() * kPartPerSM));
    if (n) launch_hist(p, key_kind == LSORT_KEY_F64, 1u, B, grid, C->stream);
    C->dist_keys = d_keys;
    C->dist_n = n;
    C->dist_kind = key_kind;
    C->dist_fp = model_fingerprint(h, e);
}
}  // namespace

extern "C" {

int lsort_cuda_sort_forward(lsort_ctx* C, void* d_keys, uint64_t n, int key_kind, const lsort_cfg* cfgp,
                            const lsort_rmi_header* h, const lsort_rmi_entry* e, uint32_t b_lo, uint32_t b_hi,
                            const uint64_t* d_sorted_sample, uint64_t sample_n, lsort_stats* stats,
                            uint64_t* nan_index_out) {
    if (!C || !h || !e) return LSORT_EINVAL;
    C->err.clear();
    if (nan_index_out) *nan_index_out = ~0ull;
    const uint32_t B = h->submodels;
    if (B < 2 || B > LSORT_MAX_RMI || b_lo >= b_hi || b_hi > B || (n && !d_keys))
        return fail(C, {LSORT_EINVAL, "sort_forward: bad model / bucket range"});
    if (key_kind != LSORT_KEY_U64 && key_kind != LSORT_KEY_F64 && key_kind != LSORT_KEY_ENC_F64)
        return fail(C, {LSORT_EINVAL, "key_kind"});
    lsort_cfg cfg = cfg_or_default(cfgp);
    if (stats) std::memset(stats, 0, sizeof(*stats));
    try {
        validate_cfg(cfg);
        CU(cudaSetDevice(C->device));
        Forward fw;
        fw.B = B;
        fw.nb = b_hi - b_lo;
        if (d_sorted_sample && sample_n >= 2 && !(cfg.flags & LSORT_FLAG_STRICT_POLICY)) {
            // bucket offsets of the sorted sample under the full model (nb = B); the
            // slice of local bucket b starts at offsets[b_lo + b]
            upload_learned(C, h, e, B, 0.0, 1.0);
            if (!C->fwd_slices.ensure(4 * ((size_t)B + 2))) throw LsortError{LSORT_ENOMEM, "forward"};
            launch_sample_slices(d_sorted_sample, sample_n, C->models.as<uint8_t>(), C->fwd_slices.as<uint32_t>(), B,
                                 nullptr, C->stream);
            fw.slices = C->fwd_slices.as<uint32_t>() + b_lo;
            fw.psample = d_sorted_sample;
        }
        // the forwarded root: the same RMI restricted to CDF [b_lo/B, b_hi/B) with
        // b_hi - b_lo buckets (Learned::bucket_index, models.hpp:128-138,162-171)
        upload_learned(C, h, e, fw.nb, (double)b_lo / B, (double)b_hi / B);
        fw.model_bytes = sizeof(ModelHdr) + kLearnedEntryBytes * (size_t)B;
        if (!C->fwd_model.ensure(fw.model_bytes)) throw LsortError{LSORT_ENOMEM, "forward"};
        CU(cudaMemcpyAsync(C->fwd_model.p, C->models.p, fw.model_bytes, cudaMemcpyDeviceToDevice, C->stream));
        fw.model = C->fwd_model.as<uint8_t>();
        C->launches = 0;
        Engine E(C, cfg);
        E.sort(d_keys, n, key_kind != LSORT_KEY_U64, stats, key_kind == LSORT_KEY_ENC_F64, &fw);
        CU(cudaStreamSynchronize(C->stream));
        if (stats) stats->kernel_launches = C->launches;
    } catch (const LsortError& e2) {
        cudaStreamSynchronize(C->stream);
        cudaGetLastError();
        if (e2.code == LSORT_ENAN) {
            if (nan_index_out) *nan_index_out = std::stoull(e2.msg);
            C->err = "NaN at index " + e2.msg;
            return LSORT_ENAN;
        }
        return fail(C, e2);
    }
    return LSORT_OK;
}

int lsort_cuda_copy_runs(lsort_ctx* C, const uint64_t* d_src, uint64_t* d_dst, const uint64_t* runs,
                         uint64_t nruns) {
    if (!C || (nruns && (!runs || !d_src || !d_dst))) return fail(C, {LSORT_EINVAL, "copy_runs: bad arguments"});
    try {
        CU(cudaSetDevice(C->device));
        if (!nruns) return LSORT_OK;
        if (!C->piv.ensure(24 * nruns) || !C->hmodel.ensure(24 * nruns)) throw LsortError{LSORT_ENOMEM, "runs"};
        std::memcpy(C->hmodel.p, runs, 24 * nruns);
        CU(cudaMemcpyAsync(C->piv.p, C->hmodel.p, 24 * nruns, cudaMemcpyHostToDevice, C->stream));
        launch_copy_runs(d_src, d_dst, C->piv.as<uint64_t>(), nruns, C->stream);
        CU(cudaStreamSynchronize(C->stream));
        CU(cudaGetLastError());
    } catch (const LsortError& e) {
        return fail(C, e);
    }
    return LSORT_OK;
}

int lsort_cuda_sort_buckets(lsort_ctx* C, void* d_keys, uint64_t n, int key_kind, const lsort_cfg* cfgp,
                            const lsort_rmi_header* h, const lsort_rmi_entry* e, uint32_t b_lo, uint32_t b_hi,
                            const uint64_t* bucket_sizes, const uint64_t* d_sorted_sample, uint64_t sample_n,
                            lsort_stats* stats) {
    if (!C || !h || !e) return LSORT_EINVAL;
    C->err.clear();
    const uint32_t B = h->submodels;
    if (B < 2 || B > LSORT_MAX_RMI || b_lo > b_hi || b_hi > B || (n && (!d_keys || !bucket_sizes)))
        return fail(C, {LSORT_EINVAL, "sort_buckets: bad model / bucket range"});
    if (key_kind != LSORT_KEY_U64 && key_kind != LSORT_KEY_ENC_F64)
        return fail(C, {LSORT_EINVAL, "sort_buckets: keys must be u64 or encoded f64"});
    uint64_t tot = 0;
    for (uint32_t j = 0; j < b_hi - b_lo; ++j) tot += bucket_sizes[j];
    if (tot != n) return fail(C, {LSORT_EINVAL, "sort_buckets: bucket sizes do not add up to n"});
    lsort_cfg cfg = cfg_or_default(cfgp);
    if (stats) std::memset(stats, 0, sizeof(*stats));
    try {
        validate_cfg(cfg);
        CU(cudaSetDevice(C->device));
        if (n == 0) return LSORT_OK;
        const bool f64 = key_kind == LSORT_KEY_ENC_F64;
        const uint32_t nb = b_hi - b_lo, cap = cfg.base_case_capacity;
        // children train on their slice of the sorted global sample (GPU policy)
        std::vector<uint32_t> offs;
        Forward fw;
        const bool slices = d_sorted_sample && sample_n >= 2 && !(cfg.flags & LSORT_FLAG_STRICT_POLICY);
        if (slices) {
            upload_learned(C, h, e, B, 0.0, 1.0);
            if (!C->fwd_slices.ensure(4 * ((size_t)B + 2))) throw LsortError{LSORT_ENOMEM, "slices"};
            launch_sample_slices(d_sorted_sample, sample_n, C->models.as<uint8_t>(), C->fwd_slices.as<uint32_t>(), B,
                                 nullptr, C->stream);
            offs.resize(B + 1);
            CU(cudaMemcpyAsync(offs.data(), C->fwd_slices.p, 4 * ((size_t)B + 1), cudaMemcpyDeviceToHost, C->stream));
            CU(cudaStreamSynchronize(C->stream));
            fw.psample = d_sorted_sample;
        }
        // buckets within the base-case capacity are sorted in place right away;
        // the others start the recursion at level 1
        std::vector<SegPlan> big;
        std::vector<BaseItem> small[3];
        uint64_t at = 0, small_keys = 0;
        const uint32_t cls_cap[3] = {std::min<uint32_t>(kWarpBaseCap, cap), std::min<uint32_t>(4096, cap), cap};
        for (uint32_t j = 0; j < nb; ++j) {
            const uint64_t len = bucket_sizes[j];
            if (len > cap) {
                uint64_t ps = 0;
                if (slices) {
                    const uint32_t o = offs[b_lo + j], l = offs[b_lo + j + 1] - o;
                    if (l >= kMinSlice) ps = (uint64_t)o << 24 | std::min<uint32_t>(l, 0xffffffu);
                }
                big.push_back({at, len, 1, 0, ps});
            } else if (len > 1 || (len == 1 && f64)) {
                const int c = len <= cls_cap[0] ? 0 : (len <= cls_cap[1] ? 1 : 2);
                small[c].push_back(BaseItem{at, len});
                small_keys += len;
            }
            at += len;
        }
        C->launches = 0;
        if (small_keys) {
            size_t maxl = 1;
            for (auto& v : small) maxl = std::max(maxl, v.size());
            if (!C->ctrl.ensure(sizeof(Ctrl)) || !C->hctrl.ensure(sizeof(Ctrl)) ||
                !C->base[0].ensure(maxl * sizeof(BaseItem)) || !C->base[1].ensure(maxl * sizeof(BaseItem)) ||
                !C->base[2].ensure(maxl * sizeof(BaseItem)))
                throw LsortError{LSORT_ENOMEM, "bucket base cases"};
            Ctrl* hc = C->hctrl.as<Ctrl>();
            std::memset(hc, 0, sizeof(Ctrl));
            hc->nan_index = ~0ull;
            LevelParams p{};
            p.ctrl = C->ctrl.as<Ctrl>();
            for (int c = 0; c < 3; ++c) {
                hc->n_base[c] = (unsigned)small[c].size();
                if (!small[c].empty())
                    CU(cudaMemcpyAsync(C->base[c].p, small[c].data(), small[c].size() * sizeof(BaseItem),
                                       cudaMemcpyHostToDevice, C->stream));
                p.base[c] = C->base[c].as<BaseItem>();
            }
            p.list_cap = (uint32_t)maxl;
            CU(cudaMemcpyAsync(p.ctrl, hc, sizeof(Ctrl), cudaMemcpyHostToDevice, C->stream));
            // in place: every base-case CTA holds its whole segment before it stores
            launch_base_cases(p, (const uint64_t*)d_keys, d_keys, f64, C->stream);
            C->launches += 3;
            CU(cudaStreamSynchronize(C->stream));  // the host control block is reused by the engine
            if (stats) { stats->base_case_keys += small_keys; stats->base_segments += small[0].size() + small[1].size() + small[2].size(); }
        }
        if (!big.empty()) {
            Engine E(C, cfg);
            E.sort(d_keys, n, f64, stats, f64, slices ? &fw : nullptr, &big);
        }
        CU(cudaStreamSynchronize(C->stream));
        CU(cudaGetLastError());
        if (stats) stats->kernel_launches = C->launches;
    } catch (const LsortError& e2) {
        cudaStreamSynchronize(C->stream);
        cudaGetLastError();
        return fail(C, e2);
    }
    return LSORT_OK;
}

int lsort_cuda_dist_histogram(lsort_ctx* C, const void* d_keys, uint64_t n, int key_kind, const lsort_rmi_header* h,
                              const lsort_rmi_entry* e, uint64_t* d_hist) {
    if (!C || !h || !e || !d_hist || h->submodels < 2 || h->submodels > LSORT_MAX_RMI) return LSORT_EINVAL;
    try {
        CU(cudaSetDevice(C->device));
        dist_hist_ids(C, d_keys, n, key_kind, h, e, (unsigned long long*)d_hist);
        // the local histogram stays with the ids (the caller all-reduces d_hist)
        if (!C->dist_hist.ensure(8 * (size_t)h->submodels)) throw LsortError{LSORT_ENOMEM, "dist"};
        CU(cudaMemcpyAsync(C->dist_hist.p, d_hist, 8 * (size_t)h->submodels, cudaMemcpyDeviceToDevice, C->stream));
        Ctrl hc;
        CU(cudaMemcpyAsync(&hc, C->ctrl.p, sizeof(Ctrl), cudaMemcpyDeviceToHost, C->stream));
        CU(cudaStreamSynchronize(C->stream));
        CU(cudaGetLastError());
        if (hc.nan_index != ~0ull) {
            C->dist_keys = nullptr;
            C->err = "NaN at index " + std::to_string(hc.nan_index);
            return LSORT_ENAN;
        }
    } catch (const LsortError& er) {
        C->dist_keys = nullptr;
        return fail(C, er);
    }
    return LSORT_OK;
}

int lsort_cuda_dist_partition(lsort_ctx* C, const void* d_keys, uint64_t n, int key_kind, const lsort_rmi_header* h,
                              const lsort_rmi_entry* e, const uint32_t* bucket_bounds, uint32_t nranks,
                              uint64_t* d_out, uint64_t* send_counts) {
    if (!C || !h || !e || !bucket_bounds || nranks == 0 || nranks > kMaxNB || h->submodels < 2 ||
        h->submodels > LSORT_MAX_RMI)
        return LSORT_EINVAL;
    try {
        CU(cudaSetDevice(C->device));
        const uint32_t B = h->submodels;
        // bucket -> destination rank map and per-rank histogram
        std::vector<uint32_t> map(B);
        for (uint32_t r = 0; r < nranks; ++r)
            for (uint32_t b = bucket_bounds[r]; b < bucket_bounds[r + 1] && b < B; ++b) map[b] = r;
        if (!C->aux.ensure(B * 4 + 8 * (size_t)B + 8 * (size_t)nranks + 16)) throw LsortError{LSORT_ENOMEM, "dist"};
        uint32_t* dmap = C->aux.as<uint32_t>();
        unsigned long long* dhist = (unsigned long long*)(C->aux.as<uint8_t>() + B * 4 + 4 * (B & 1));
        unsigned long long* dcur = dhist + B;
        CU(cudaMemcpyAsync(dmap, map.data(), B * 4, cudaMemcpyHostToDevice, C->stream));
        // the ids from lsort_cuda_dist_histogram of the same keys under the same model are reused
        const bool have_ids = C->dist_keys == d_keys && C->dist_n == n && C->dist_kind == key_kind &&
                              C->dist_fp == model_fingerprint(h, e);
        if (have_ids) {
            upload_learned(C, h, e, B, 0.0, 1.0);  // (the model arena may have been reused since)
            CU(cudaMemcpyAsync(dhist, C->dist_hist.p, 8 * (size_t)B, cudaMemcpyDeviceToDevice, C->stream));
        } else {
            dist_hist_ids(C, d_keys, n, key_kind, h, e, dhist);
        }
        bool identity = nranks == B;  // one "rank" per bucket: the bucket-major partition
        for (uint32_t b = 0; identity && b < B; ++b) identity = map[b] == b;
        if (identity && !send_counts) {
            // cursors = exclusive scan of the histogram, on the device: no host round trip
            launch_excl_scan_u64(dhist, dcur, B, C->stream);
        } else {
            std::vector<uint64_t> hist(B);
            CU(cudaMemcpyAsync(hist.data(), dhist, 8 * (size_t)B, cudaMemcpyDeviceToHost, C->stream));
            CU(cudaStreamSynchronize(C->stream));
            std::vector<uint64_t> cur(nranks, 0);
            for (uint32_t b = 0; b < B; ++b) cur[map[b]] += hist[b];
            uint64_t acc = 0;
            for (uint32_t r = 0; r < nranks; ++r) {
                if (send_counts) send_counts[r] = cur[r];
                uint64_t c = cur[r];
                cur[r] = acc;
                acc += c;
            }
            CU(cudaMemcpyAsync(dcur, cur.data(), 8 * (size_t)nranks, cudaMemcpyHostToDevice, C->stream));
        }
        LevelParams p = dist_level(C, d_keys, n, B, dcur, d_out);
        const int grid = (int)std::max<uint64_t>(1, std::min<uint64_t>(p.ntiles, (uint64_t)num_sms() * kPartPerSM));
        if (n && identity) launch_scatter(p, key_kind == LSORT_KEY_F64, B, grid, C->stream);  // no map lookups
        else if (n) launch_scatter_mapped(p, key_kind == LSORT_KEY_F64, dmap, nranks, grid, C->stream);
        CU(cudaStreamSynchronize(C->stream));
        CU(cudaGetLastError());
    } catch (const LsortError& er) {
        return fail(C, er);
    }
    return LSORT_OK;
}

}  // extern "C"
