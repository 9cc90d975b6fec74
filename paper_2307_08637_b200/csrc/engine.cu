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
#include "engine_core.cuh"

using namespace lsort_host;

namespace {
constexpr uint32_t kManyWays = 3;  // concurrent sorts in lsort_cuda_sort_many
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

}  // extern "C"


extern "C" {

int lsort_cuda_sort_classic(lsort_ctx* C, void* keys, uint64_t n, int key_kind, int mem_kind, const lsort_cfg* cfgp,
                            lsort_stats* stats, uint64_t* nan_index_out) {
    if (!C) return LSORT_EINVAL;
    C->err.clear();
    if (nan_index_out) *nan_index_out = ~0ull;
    if (key_kind != LSORT_KEY_U64 && key_kind != LSORT_KEY_F64) return fail(C, {LSORT_EINVAL, "key_kind"});
    if (mem_kind != LSORT_MEM_DEVICE && mem_kind != LSORT_MEM_HOST) return fail(C, {LSORT_EINVAL, "mem_kind"});
    if (n > 0 && !keys) return fail(C, {LSORT_EINVAL, "null keys"});
    lsort_cfg cfg = cfg_or_default(cfgp);
    if (stats) std::memset(stats, 0, sizeof(*stats));
    try {
        validate_cfg(cfg);
        CU(cudaSetDevice(C->device));
        const bool f64 = key_kind == LSORT_KEY_F64;
        C->launches = 0;
        const cudaStream_t st = C->stream;
        void* dkeys = keys;
        if (mem_kind == LSORT_MEM_HOST) {
            if (!C->data.ensure(std::max<uint64_t>(n, 1) * 8)) throw LsortError{LSORT_ENOMEM, "device keys"};
            dkeys = C->data.p;
            CU(cudaMemcpyAsync(dkeys, keys, n * 8, cudaMemcpyHostToDevice, st));
        }
        CU(cudaEventRecord(C->ev[0], st));
        Engine E(C, cfg);
        if (n <= cfg.base_case_capacity) {
            E.sort(dkeys, n, f64, stats);  // one shared-memory sort: no model to train
        } else {
            // train the RMI once (§3.3: LearnedSort samples the data only once)
            const uint32_t B = cfg.rmi_bucket_count;
            const uint64_t s = sample_size_host(cfg.sample_fraction, cfg.rmi_sample_cap, n);
            const size_t mb = sizeof(ModelHdr) + kLearnedEntryBytes * (size_t)B;
            if (!C->sample.ensure(8 * s) || !C->segs.ensure(sizeof(SegDesc)) || !C->fwd_model.ensure(mb) ||
                !C->train_ws.ensure(train_workspace_bytes(s, B)))
                throw LsortError{LSORT_ENOMEM, "classic model"};
            SegDesc d{};
            d.begin = 0;
            d.n = n;
            CU(cudaMemcpyAsync(C->segs.p, &d, sizeof(d), cudaMemcpyHostToDevice, st));
            launch_gather(C->segs.as<SegDesc>(), dkeys, f64, cfg.seed, 0, s, C->sample.as<uint64_t>(), nullptr, st);
            E.nested_sort(C->sample.as<uint64_t>(), s);
            CU(cudaMemsetAsync(C->fwd_model.p, 0, sizeof(ModelHdr), st));
            launch_train_rmi(C->sample.as<uint64_t>(), s, B, C->fwd_model.as<uint8_t>(), B, C->train_ws.p, nullptr, st);
            C->launches += 10;
            Forward fw;
            fw.model = C->fwd_model.as<uint8_t>();
            fw.model_bytes = mb;
            fw.nb = B;
            fw.B = B;
            E.classic = C->fwd_model.as<uint8_t>();
            E.classic_B = B;
            E.sort(dkeys, n, f64, stats, false, &fw);
        }
        CU(cudaEventRecord(C->ev[1], st));
        if (mem_kind == LSORT_MEM_HOST) CU(cudaMemcpyAsync(keys, dkeys, n * 8, cudaMemcpyDeviceToHost, st));
        CU(cudaStreamSynchronize(st));
        if (stats) {
            float ms = 0;
            cudaEventElapsedTime(&ms, C->ev[0], C->ev[1]);
            stats->ms_total = ms;
            stats->kernel_launches = C->launches;
        }
    } catch (const LsortError& e) {
        cudaStreamSynchronize(C->stream);
        cudaGetLastError();
        if (e.code == LSORT_ENAN) {
            if (nan_index_out) *nan_index_out = std::stoull(e.msg);
            C->err = "NaN at index " + e.msg;
            return LSORT_ENAN;
        }
        return fail(C, e);
    }
    return LSORT_OK;
}

int lsort_cuda_model_counting_sort(lsort_ctx* C, const lsort_rmi_header* h, const lsort_rmi_entry* e, double cdf_lo,
                                   double cdf_hi, const uint64_t* d_keys, uint64_t n, uint64_t* d_out) {
    if (!C || !h || !e || h->submodels == 0 || h->submodels > LSORT_MAX_RMI || (n && (!d_keys || !d_out)))
        return fail(C, {LSORT_EINVAL, "model_counting_sort: bad arguments"});
    if (n > kSmallSampleCap) return fail(C, {LSORT_EINVAL, "model_counting_sort: at most 8192 keys per segment"});
    try {
        CU(cudaSetDevice(C->device));
        upload_learned(C, h, e, h->submodels, cdf_lo, cdf_hi);
        if (n) launch_model_counting_sort(C->models.as<uint8_t>(), d_keys, n, d_out, C->stream);
        CU(cudaStreamSynchronize(C->stream));
        CU(cudaGetLastError());
    } catch (const LsortError& er) {
        return fail(C, er);
    }
    return LSORT_OK;
}

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
                small[c].push_back(BaseItem{at, len, (int64_t)at});
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

}  // extern "C"
