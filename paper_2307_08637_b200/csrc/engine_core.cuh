// engine_core.cuh -- host orchestrator core shared by engine.cu (single-GPU
// C-ABI) and dist.cu (multi-GPU driver): workspace buffers, the context,
// and the Engine that drives the AIPS2o recursion on one device.
#pragma once
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

namespace lsort_host {

// why the last failed allocation of this thread failed (appended to ENOMEM messages by
// fail(): a sticky fault of an earlier kernel makes every later cudaMalloc fail too, and
// must not read as "out of memory")
inline std::string& last_alloc_error() {
    static thread_local std::string s;
    return s;
}
inline void note_alloc_error(cudaError_t e, size_t bytes, const char* what) {
    last_alloc_error() = std::string(what) + " of " + std::to_string(bytes) + " bytes: " + cudaGetErrorString(e);
}

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
            const cudaError_t e = cudaMalloc(&p, bytes);
            if (e != cudaSuccess) { note_alloc_error(e, bytes, "cudaMalloc"); cudaGetLastError(); p = nullptr; return false; }
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
        const cudaError_t e = cudaMallocHost(&p, want);
        if (e != cudaSuccess) { note_alloc_error(e, want, "cudaMallocHost"); cudaGetLastError(); p = nullptr; return false; }
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
constexpr uint32_t kBigRootBuckets = 512;
constexpr uint64_t kBigRootMinKeys = 32ull << 20;
constexpr uint64_t kRootSampleMin = 256ull << 10;
inline bool root_lut_enabled() {
    static const bool off = getenv("LSORT_NO_ROOT_LUT") != nullptr;
    return !off;
}

inline uint32_t fanout(uint64_t n, uint32_t cfg_count, uint32_t target) {
    if (target == 0) return cfg_count;
    uint64_t want = (n + target - 1) / target;
    uint32_t b = 2;
    while (b < want && b < cfg_count) b <<= 1;
    return std::min(b, cfg_count);
}

inline bool trace_enabled() {
    static int v = -1;
    if (v < 0) {
        const char* e = getenv("LSORT_TRACE");
        v = (e && *e && *e != '0') ? 1 : 0;
    }
    return v == 1;
}

inline uint64_t seg_seed_host(uint64_t cfg_seed, uint64_t begin, uint32_t depth) {
    return splitmix64(cfg_seed ^ splitmix64(begin + ((uint64_t)depth << 48)));
}
inline uint64_t sample_size_host(double frac, uint32_t cap, uint64_t n) {
    double v = frac * (double)n;
    double c = (double)cap;
    uint64_t s = (uint64_t)std::ceil(v < c ? v : c);
    return s < 2 ? 2 : s;
}

}  // namespace lsort_host
using namespace lsort_host;  // (internal header: the library's own translation units)

struct lsort_ctx {
    int device = 0;
    cudaStream_t stream = nullptr;
    cudaStream_t own_stream = nullptr;
    std::string err;
    int depth = 0;  // nesting level (sample sorts run in a nested context)
    DevBuf scratch, data, segs, idx, tile_prefix, models, buckets, rec, base[3], fill, ctrl, sample, aux, train_ws,
        kseg, ktp, kplan, qws, ids, clus, cidx, scratch2, dws, bat[3], psample, slices, fwd_model, fwd_slices, piv, fsample,
        lutws, scratch3, segd;
    cudaStream_t h2d_stream = nullptr, d2h_stream = nullptr;
    cudaEvent_t bev[11] = {};  // batch pipeline: h2d[3], sorted[3], d2h[3], start, end
    PinBuf hctrl, hrec, hsegs, hidx, hprefix, hmodel;
    std::unique_ptr<lsort_ctx> nested;
    // lanes: workspaces + streams on which the models of the big segments of
    // one level are built concurrently (fork/join with events on `stream`)
    std::vector<std::unique_ptr<lsort_ctx>> lanes;
    std::vector<std::unique_ptr<lsort_ctx>> subs;  // sort_many: one context per concurrent sort
    bool zero_copy = false;  // control transfers as kernels (copy engines busy with a batch)
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

namespace lsort_host {

struct SegPlan {
    uint64_t begin, n;
    uint32_t depth, flags;
    uint64_t pslice = 0;       // slice of the parent's sorted sample (SegDesc::pslice)
    uint64_t in_begin = ~0ull;  // read position (SegDesc::in_begin); ~0 = begin
    uint64_t rd() const { return in_begin == ~0ull ? begin : in_begin; }
};

inline void validate_cfg(const lsort_cfg& c) {
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
inline uint64_t effective_min_rmi(const lsort_cfg& c) {
    return (c.flags & LSORT_FLAG_STRICT_POLICY) ? c.min_rmi_input : std::min<uint64_t>(c.min_rmi_input, kGpuMinRmi);
}

inline DevCfg dev_cfg(const lsort_cfg& c) {
    DevCfg d;
    d.min_rmi_input = effective_min_rmi(c);
    d.max_dup = c.max_duplicate_fraction;
    d.sample_fraction = c.sample_fraction;
    d.first_sample_cap = c.first_sample_cap;
    d.rmi_sample_cap = c.rmi_sample_cap;
    d.seed = c.seed;
    d.quality = (c.flags & LSORT_FLAG_STRICT_POLICY) ? 0u : 1u;
    d.psample = nullptr;
    static const bool no_lut = getenv("LSORT_NO_LUT") != nullptr;
    d.lut = d.quality && !no_lut;
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

    // Multi-GPU global model (dist.cu): big_model trains on this already
    // gathered (unsorted, device) sample instead of drawing one from the
    // segment, and a learned model is also replaced by the splitter tree when
    // its largest bucket holds more than 1/share_den of the sample (the rank
    // cuts need fine buckets; 0 = the single-GPU quality test only).
    const uint64_t* given_sample = nullptr;
    uint64_t given_n = 0;
    uint32_t share_den = 0;
    // GPU policy for a big learned root: RMI submodels (0 = the segment's
    // rmi_b) when the root's output buckets are capped below them
    uint32_t root_sub = 0;
    // LearnedSort 2.0 classic path (classic.cu): the root RMI (device model
    // record, CDF [0,1), classic_B buckets) is forwarded to level 0 (Forward)
    // and, restricted to each round-1 bucket's CDF range, to level 1; the
    // buckets finished at levels 0 and 1 are sorted by model-based counting
    // sort + fix-up instead of the radix base case.
    const uint8_t* classic = nullptr;
    uint32_t classic_B = 0;

    uint32_t rmi_b(uint64_t n) const { return fanout(n, cfg.rmi_bucket_count, cfg.bucket_target); }
    // RMI sample of a root segment. GPU policy: min(SPEC size, max(256 Ki, n / 512))
    // -- ~2 Ki samples per level-1 segment of a 512-way root still train the
    // children's models (they take slices of this sample); a 1e8-key root sorted
    // its 1 Mi sample for nothing (Normal 1e8: models 0.45 -> 0.29 ms, base
    // unchanged; C5 keeps ~1 Mi). Sorted output is the same.
    uint64_t root_rmi_sample(uint64_t n) const {
        const uint64_t s = sample_size_host(cfg.sample_fraction, cfg.rmi_sample_cap, n);
        if (cfg.flags & LSORT_FLAG_STRICT_POLICY) return s;
        static const int sh = getenv("LSORT_ROOT_SAMPLE_SHIFT") ? atoi(getenv("LSORT_ROOT_SAMPLE_SHIFT")) : 9;
        return std::min<uint64_t>(s, std::max<uint64_t>(kRootSampleMin, n >> sh));
    }
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

    // Base cases of a level: the > 8 Ki, <= 8 Ki and 1 Ki classes on three
    // lane streams (high priority: the long CTAs start first) beside the 4 Ki
    // class on the context stream, joined back before the next level.
    void base_cases(const LevelParams& p, const uint64_t* src, void* out, bool f64) {
        static const bool serial = getenv("LSORT_BASE_SERIAL") != nullptr;
        if (serial) {
            launch_base_cases(p, src, out, f64, st);
            return;
        }
        if (!C->fork_ev) CU(cudaEventCreateWithFlags(&C->fork_ev, cudaEventDisableTiming));
        CU(cudaEventRecord(C->fork_ev, st));
        for (uint32_t l = 0; l < 3; ++l) CU(cudaStreamWaitEvent(lane(l)->stream, C->fork_ev, 0));
        launch_base_class(p, 2, src, out, f64, lane(0)->stream);
        launch_base_class(p, 3, src, out, f64, lane(2)->stream);
        launch_base_class(p, 0, src, out, f64, lane(1)->stream);
        launch_base_class(p, 1, src, out, f64, st);
        for (uint32_t l = 0; l < 3; ++l) {
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
        const uint32_t sub = (sp.depth == 0 && root_sub) ? root_sub : hseg.rmi_b;  // RMI submodels
        const uint64_t s1 = sample_size_host(cfg.sample_fraction, cfg.first_sample_cap, n);
        const uint64_t s2 = given_sample ? given_n
                            : sp.depth == 0 ? root_rmi_sample(n)
                                            : sample_size_host(cfg.sample_fraction, cfg.rmi_sample_cap, n);
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
            !N->aux.ensure(4) || !N->train_ws.ensure(train_workspace_bytes(s2, sub)))
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
        // (the sample-partition segment descriptor: also the first sample's
        // source segment when the sample is given)
        SegDesc d{};
        d.begin = 0;
        d.n = s2;
        d.model_off = 0;
        d.bucket_off = 0;
        d.nb_max = nb;
        d.tree_k = k;
        up(N->segs.p, &d, sizeof(d), false, st);
        if (given_sample)
            CU(cudaMemcpyAsync(N->sample.p, given_sample, s2 * 8, cudaMemcpyDeviceToDevice, N->h2d_stream));
        else
            launch_gather(dseg, src, f64, seed, s1, s2, N->sample.as<uint64_t>(), nullptr, N->h2d_stream);
        CU(cudaEventRecord(N->bev[1], N->h2d_stream));
        // the first sample's random gather over many CTAs (one CTA cannot keep
        // 8 Ki random loads in flight: ~30 us), then the policy CTA
        if (!N->fsample.ensure(s1 * 8)) throw LsortError{LSORT_ENOMEM, "first sample"};
        if (given_sample)  // a random subsample of the given sample
            launch_gather(N->segs.as<SegDesc>(), given_sample, false, seed, 0, s1, N->fsample.as<uint64_t>(), nullptr,
                          st);
        else
            launch_gather(dseg, src, f64, seed, 0, s1, N->fsample.as<uint64_t>(), nullptr, st);
        launch_first_sample(dseg, src, f64, C->models.as<uint8_t>(), dc, N->models.as<uint8_t>(), k, gate, st,
                            N->fsample.as<uint64_t>(), given_sample ? nullptr : slices);
        launched();
        CU(cudaStreamWaitEvent(st, N->bev[1], 0));
        // one distribution level over the sample with the first-sample tree
        uint64_t pref[2] = {0, ntiles};
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
        launched(2 + 9);
        // GPU policy: a root that takes the one-pass level 0 (or a multi-GPU global
        // model of that size) tries a cell table first (models.cu k_root_lut); the
        // RMI is trained only if it is rejected. (An accepted table's largest
        // bucket holds <= 2 / nb of the sample: within the rank-balance share test.)
        const uint32_t* tgate = gate;
        if (dc.lut && sp.depth == 0 && root_lut_enabled() && hseg.nb_max <= kDirectMaxBuckets &&
            n >= kDirectMinPerBucket * hseg.nb_max) {
            if (!N->lutws.ensure(root_lut_workspace_bytes() + 16)) throw LsortError{LSORT_ENOMEM, "root cell table"};
            uint32_t* train_gate = (uint32_t*)(N->lutws.as<uint8_t>() + root_lut_workspace_bytes());
            static const bool no_log = getenv("LSORT_NO_LOG_LUT") != nullptr;
            launch_root_lut(N->sample.as<uint64_t>(), s2, C->models.as<uint8_t>() + hseg.model_off, N->lutws.p, gate,
                            train_gate, st, f64 && !no_log, n < kBigRootMinKeys);
            launched(f64 && !no_log ? 6 : 2);
            tgate = train_gate;
        }
        launch_train_rmi(N->sample.as<uint64_t>(), s2, sub, C->models.as<uint8_t>() + hseg.model_off,
                         hseg.rmi_b, N->train_ws.p, tgate, st);
        launched(8);
        if (dc.quality) {  // (and the children's sample slices for the root)
            if (!N->qws.ensure(quality_workspace_bytes())) throw LsortError{LSORT_ENOMEM, "quality workspace"};
            // a big root (>= 32 Mi keys, 512 buckets) keeps a learned model up to a
            // bucket of 1/8 of the keys: such a bucket still makes progress, and the
            // learned root takes the one-pass level 0 (a tree root does not)
            const uint32_t poor_share = (sp.depth == 0 && n >= kBigRootMinKeys && !share_den) ? kPoorShare / 2 : kPoorShare;
            launch_quality_check(N->sample.as<uint64_t>(), s2, C->models.as<uint8_t>() + hseg.model_off, hseg.tree_k,
                                 N->qws.p, slices, gate, st, share_den, poor_share);
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
    // out (nullable = keys): where base cases and fills store the final keys;
    // `keys` then only serves as the ping-pong partner of the scratch buffer.
    void sort(void* keys, uint64_t n, bool f64, lsort_stats* stats, bool in_encoded = false,
              const Forward* fw = nullptr, const std::vector<SegPlan>* start = nullptr, void* out = nullptr) {
        if (!out) out = keys;
        if (n < 2) {
            if (n == 1 && out != keys) CU(cudaMemcpyAsync(out, keys, 8, cudaMemcpyDeviceToDevice, st));
            if (n == 1 && f64 && in_encoded) {
                launch_decode((uint64_t*)out, n, st);
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
            if (out != keys) CU(cudaMemcpyAsync(out, keys, n * 8, cudaMemcpyDeviceToDevice, st));
            keys = out;
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
        uint64_t* lvl_dout = nullptr;  // the padded output of the current level when it ran one-pass
        while (!segs.empty()) {
            const uint32_t ns = (uint32_t)segs.size();
            {  // bucket ids are indexed by read position: cover this level's read window
                uint64_t rmax = 0;
                for (const SegPlan& q : segs) rmax = std::max(rmax, q.rd() + q.n);
                if (!C->ids.ensure(2 * std::max<uint64_t>(rmax, 1))) throw LsortError{LSORT_ENOMEM, "bucket ids"};
            }
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
            bool padded_in = false;  // the level reads a padded level-0 output (cluster items read `begin`)
            for (const SegPlan& q : segs) padded_in |= q.rd() != q.begin;
            const bool use_cluster = level >= 1 && !src_f64 && cluster_available() &&
                                     ((cfg.flags & LSORT_FLAG_CLUSTER) || auto_cluster) && cap >= 16384 &&
                                     !(classic && level <= 1) && !padded_in;
            std::vector<uint32_t> fwd1;  // classic: level-1 segments with a forwarded model
            std::vector<BaseItem> clus;
            std::vector<SegPlan> psegs;
            psegs.reserve(ns);
            for (uint32_t i = 0; i < ns; ++i) {
                const SegPlan& s = segs[i];
                if (use_cluster && s.n > cap && s.n <= kClCap) {
                    clus.push_back(BaseItem{s.begin, s.n, (int64_t)s.begin});
                    continue;
                }
                const uint32_t j = (uint32_t)psegs.size();
                psegs.push_back(s);
                SegDesc& d = hs[j];
                d.begin = s.begin;
                d.in_begin = s.rd();
                d.n = s.n;
                d.depth = s.depth;
                d.flags = s.flags;
                d.pslice = s.pslice;
                const bool classic1 = classic && level == 1 && !(s.flags & kSegForceRadix);
                d.rmi_b = (fw && level == 0) ? fw->nb : (classic1 ? classic_B : rmi_b(s.n));
                // GPU policy: a learned root over >= 32 Mi keys partitions 512 ways (its
                // level 0 writes 8-key runs instead of 4-key runs; the children, still far
                // above the base-case capacity, take one more level either way): C5
                // 12.11 -> 11.79 ms, C2 arrays -4%; 256 ways sent C5 segments to a third level
                static const uint32_t root_cap =
                    getenv("LSORT_ROOT_B") ? (uint32_t)atoi(getenv("LSORT_ROOT_B")) : kBigRootBuckets;
                root_sub = 0;
                if (level == 0 && !fw && !classic && !(cfg.flags & LSORT_FLAG_STRICT_POLICY) &&
                    s.n >= kBigRootMinKeys && root_cap && root_cap < d.rmi_b) {
                    root_sub = d.rmi_b;  // the RMI keeps its submodels; its CDF feeds fewer buckets
                    d.rmi_b = root_cap;
                }
                max_rmi_b = std::max(max_rmi_b, root_sub);
                max_rmi_b = std::max(max_rmi_b, d.rmi_b);
                d.tree_k = tree_k(s.n);
                uint32_t payload, nb;
                if (s.flags & kSegForceRadix) {
                    payload = 0;
                    nb = 1u << kRadixBits;
                } else {
                    uint32_t tp = (uint32_t)((tree_payload_bytes(d.tree_k, d.tree_k - 1) + 15) & ~15ull);
                    payload = std::max<uint32_t>(kLearnedEntryBytes * std::max(d.rmi_b, root_sub), tp);
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
                if (classic1) {  // the root restricted to this round-1 bucket (k_forward_models)
                    fwd1.push_back(j);
                    kinds |= 1u;
                    continue;
                }
                const int mc = model_class(s);
                if (mc == 2) bigs.push_back(j);
                else if (mc == 1) mids.push_back(j);
                else hi[nsmall++] = j;
                if (s.flags & kSegForceRadix) kinds |= 4u;
                else kinds |= (s.n >= effective_min_rmi(cfg) ? (dev_cfg(cfg).lut ? 5u : 1u) : 0u) | 2u;
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
                !C->kseg.ensure(4 * (size_t)np * 4 + 16) || !C->ktp.ensure(4 * ((size_t)np + 1) * 8) ||
                !C->kplan.ensure(4 * sizeof(KindPlan)) || !C->clus.ensure(ncl * sizeof(BaseItem) + 16))
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
            // model records start zeroed: a builder that leaves a header field unset (the
            // depth-cap radix fallback once left `flags`) reads as 0 on every run, not as
            // whatever the reused memory held
            if (model_bytes) CU(cudaMemsetAsync(C->models.p, 0, model_bytes, st));
            CU(cudaMemsetAsync(&dctrl->n_rec, 0, offsetof(Ctrl, verify_first) - offsetof(Ctrl, n_rec), st));  // per-level lists and key counters

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
            // one-pass level 0 (GPU policy): a learned root with >= 64 Ki keys per bucket.
            // (A one-pass level 1 needs all of its segments learned with >= 32 samples per
            // bucket; with the 6-sigma padding of C5's 8 samples per bucket it spread the
            // writes over ~4x the keys and the level got slower, 12.3 -> 15.6 ms -- measured,
            // not kept.)
            static const bool no_direct = getenv("LSORT_NO_DIRECT") != nullptr;
            // (no cluster segments: their children sit in the level's exact output)
            const bool direct0 = !no_direct && !fw && !classic && !(cfg.flags & LSORT_FLAG_STRICT_POLICY) &&
                                 level == 0 && np == 1 && ncl == 0 && bigs.size() == 1 &&
                                 hs[0].nb_max <= kDirectMaxBuckets && n >= kDirectMinPerBucket * hs[0].nb_max;
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
                if (!fwd1.empty()) {
                    if (!C->cidx.ensure(4 * fwd1.size())) throw LsortError{LSORT_ENOMEM, "classic models"};
                    up(C->cidx.p, fwd1.data(), 4 * fwd1.size());
                    launch_forward_models(p.segs, C->cidx.as<uint32_t>(), (uint32_t)fwd1.size(), (const uint64_t*)src,
                                          classic, C->models.as<uint8_t>(), st);
                    launched();
                }
                if (trace_enabled())
                    fprintf(stderr, "    level_models host %.3f ms\n",
                            std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - th0).count());
            }
            // ---- one-pass (padded) level (k_direct): launched here, after the models;
            // the exact two-pass level below runs only if it did not (Ctrl::run_exact:
            // an ineligible model or a region that outgrew its estimate)
            uint64_t* dout = nullptr;
            uint64_t root_m = 0, alloc = 0;
            // one-pass level 1 (GPU policy): every segment a linear cell table trained on its
            // slice of the root's sorted sample -- regions sized from the slice counts
            // (C5 10.48 -> 9.80 ms, LogNormal(0,0.5) 1e8 2.30 -> 2.19); a level with another
            // model kind runs the exact two-pass level (LSORT_NO_L1_DIRECT: always)
            static const bool l1_direct = getenv("LSORT_NO_L1_DIRECT") == nullptr;
            bool direct1 = l1_direct && !fw && !classic && !(cfg.flags & LSORT_FLAG_STRICT_POLICY) && level == 1 &&
                           np >= 1 && ncl == 0 && bigs.empty() && dc.psample && !src_f64 && max_nb <= kDirectMaxBuckets;
            uint64_t alloc1 = 0;
            uint64_t* ldst = dst;  // where this level's exact kernels write (and its base cases read)
            for (uint32_t j = 0; direct1 && j < np; ++j) {
                const uint64_t m = psegs[j].pslice & 0xffffffu;
                if (m < 2) { direct1 = false; break; }
                alloc1 += direct_capacity_bound(psegs[j].n, m, hs[j].nb_max);
            }
            // the padded regions are an optimisation: without the memory for them the
            // exact two-pass level (scratch + ids only) runs instead
            const bool no_padded = (cfg.flags & LSORT_FLAG_TEST_NO_PADDED_MEM) != 0;
            if (direct1 && (no_padded || !C->scratch3.ensure(8 * (alloc1 + n)))) {
                last_alloc_error().clear();
                direct1 = false;
            }
            if (direct1) {  // (direct0 is level 0 only)
                if (timing) CU(cudaEventRecord(C->pev[6], st));
                // scratch3 = [padded regions (alloc1) | exact output of the segments the
                // exact kernels take (n)]: the next level reads both through one buffer,
                // at read positions < alloc1 + n (the id array covers them)
                if (!C->dws.ensure(direct_multi_workspace_bytes(nbuckets, np)) || !C->segd.ensure(4 * (size_t)np + 16))
                    throw LsortError{LSORT_ENOMEM, "one-pass level 1"};
                LevelParams pd = p;
                pd.dst = C->scratch3.as<uint64_t>();
                // segments of another model kind go to the exact kernels (seg_sel 2), whose
                // recursion children are then read through the padded buffer as well
                pd.seg_direct = C->segd.as<uint32_t>();
                pd.seg_sel = 1;
                p.seg_direct = C->segd.as<uint32_t>();
                p.seg_sel = 2;
                ldst = C->scratch3.as<uint64_t>() + alloc1;
                p.dst = ldst;
                p.rec_delta = (int64_t)alloc1;
                launch_direct_multi(pd, dc.psample, alloc1, C->dws.p, nbuckets,
                                    (int)std::min<uint64_t>(ntiles, (uint64_t)nsm * kPartPerSM), st,
                                    (cfg.flags & LSORT_FLAG_TEST_DIRECT_OVERFLOW) != 0, ldst);
                launched(5);
                if (timing) CU(cudaEventRecord(C->pev[7], st));
                p.gate = &dctrl->run_exact;
                dout = pd.dst;
            }
            if (direct0) {
                root_m = root_rmi_sample(n);
                // (a splitter-tree root sizes its regions from the smaller first sample)
                alloc = direct_capacity_bound(
                    n, std::min<uint64_t>(root_m, sample_size_host(cfg.sample_fraction, cfg.first_sample_cap, n)),
                    hs[0].nb_max);
                // (level 1 reads this padded output: its bucket ids are indexed by read position)
                // (without the memory for the padded regions the exact two-pass level runs)
                if (!no_padded && C->scratch2.ensure(8 * alloc) && C->ids.ensure(2 * alloc)) dout = C->scratch2.as<uint64_t>();
                else if (!C->ids.ensure(2 * std::max<uint64_t>(n, 1))) throw LsortError{LSORT_ENOMEM, "bucket ids"};
                else last_alloc_error().clear();
            }
            if (dout && direct0) {
                if (!C->dws.ensure(direct_workspace_bytes(nbuckets, np))) throw LsortError{LSORT_ENOMEM, "one-pass level"};
                LevelParams pd = p;
                pd.dst = dout;
                pd.slices = root_slices;
                if (timing) CU(cudaEventRecord(C->pev[6], st));
                launch_direct(pd, src_f64, root_m, alloc, C->dws.p, nbuckets,
                              (int)std::min<uint64_t>(ntiles, (uint64_t)nsm * kPartPerSM), st,
                              (cfg.flags & LSORT_FLAG_TEST_DIRECT_OVERFLOW) != 0, dst);
                if (timing) CU(cudaEventRecord(C->pev[7], st));
                launched(7);
                p.gate = &dctrl->run_exact;
            }
            p.ids = C->ids.as<uint16_t>();  // (the one-pass setup may have grown the id array)
            const bool direct = dout != nullptr;
            lvl_dout = dout;
            const bool next_from_dout = direct1;  // (every next-level segment reads through it)
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
                launch_cluster_sort(C->clus.as<BaseItem>(), ncl, (const uint64_t*)src, dst, out, f64, p, level + 1,
                                    st);
                launched();
            }
            if (classic && level <= 1) {  // model-based counting sort of the finished buckets
                launch_classic_base(p, dst, out, f64, classic, (int)level + 1, st);
                launched(3);
            } else {
                base_cases(p, ldst, out, f64);
            }
            mark(4);
            launch_fill(p, out, f64, nsm * 4, st);
            mark(5);
            launched(kBaseLaunches + 1);
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
            if (trace_enabled() && direct) {
                uint32_t fl = 0;
                CU(cudaMemcpy(&fl, direct_flag_ptr(C->dws.p, nbuckets, np), 4, cudaMemcpyDeviceToHost));
                fprintf(stderr, "    one-pass level %u: flag %u (0 ran, 1 overflow, 2 ineligible)\n", level, fl);
            }
            if (timing) {
                float t[5];
                for (int i = 0; i < 5; ++i) CU(cudaEventElapsedTime(&t[i], C->pev[i], C->pev[i + 1]));
                if (direct) {  // the padded one-pass level 0 is a scatter (launched inside the models mark)
                    float td = 0;
                    CU(cudaEventElapsedTime(&td, C->pev[6], C->pev[7]));
                    t[0] -= td;
                    t[2] += td;
                }
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
                stats->level0_kind = h0.kind == kLearned ? 0 : (h0.kind == kRadix && (h0.flags & kModelLut) ? 3 : 1);
            }
            if (stats) {
                stats->levels = level + 1;
                stats->segments += ns;
                uint64_t moved = 0;
                for (uint32_t i = 0; i < ns; ++i) moved += segs[i].n;
                stats->partitioned_keys += moved;
                if (hc->direct) stats->direct_keys += moved;
                stats->base_case_keys += hc->keys_base;
                stats->fill_keys += hc->keys_fill;
                stats->base_segments += (uint64_t)hc->n_base[0] + hc->n_base[1] + hc->n_base[2];
                if (classic && level == 1)  // non-empty sub-buckets after round two
                    stats->round2_buckets =
                        (uint64_t)hc->n_base[0] + hc->n_base[1] + hc->n_base[2] + hc->n_fill + hc->n_rec;
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
                                    (C->psample.p || (fw && fw->psample)) ? r[i].pslice : 0, r[i].in_begin});
                std::sort(segs.begin(), segs.end(),
                          [](const SegPlan& a, const SegPlan& b) { return a.begin < b.begin; });
            }
            // ping-pong: this level's output becomes the next level's input (a padded
            // level 0 wrote scratch2; the next level writes exact offsets into `keys`)
            src = (hc->direct || next_from_dout) ? (void*)lvl_dout : (void*)dst;
            src_f64 = false;
            dst = (dst == C->scratch.as<uint64_t>()) ? (uint64_t*)keys : C->scratch.as<uint64_t>();
            ++level;
            if (level > 64) throw LsortError{LSORT_EINTERNAL, "recursion did not terminate"};
        }
    }
};


inline int fail(lsort_ctx* ctx, const LsortError& e) {
    if (ctx) {
        ctx->err = e.msg;
        if (e.code == LSORT_ENOMEM && !last_alloc_error().empty()) ctx->err += " (" + last_alloc_error() + ")";
    }
    last_alloc_error().clear();
    return e.code;
}

inline lsort_cfg cfg_or_default(const lsort_cfg* cfg) {
    lsort_cfg c;
    if (cfg) c = *cfg;
    else lsort_cfg_default(&c);
    return c;
}

}  // namespace
