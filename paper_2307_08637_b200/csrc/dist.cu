// dist.cu -- multi-GPU LearnedSort: the C++ driver behind lsort_cuda_sort_dist
// (one process per GPU, the library owns the NCCL communicator) and
// lsort_cuda_sort_multi (one process, several GPUs).
//
// the RMI's (or splitter tree's) buckets act as global
// splitters; one exchange moves every key to the rank that owns its bucket;
// every rank then sorts its key range locally. Per sort, on every rank:
//   1. all-gather of the shard sizes (host: sample shares);
//   2. device gather of this rank's share of the global sample, all-gather;
//   3. the global partition model, built identically on every rank from the
//      gathered sample (Engine::big_model: Alg. 5 policy, multi-CTA RMI
//      training, quality check -- a learned model whose largest bucket holds
//      more than 1/(16 p) of the sample is replaced by a splitter tree over
//      the same sample, so rank cuts can balance; PAPER.md:419 monotone F =>
//      ranks hold ordered key ranges);
//   4. level-0 classify + histogram of the local shard (k_hist), all-gather
//      of the histograms (with the NaN index and output capacity of every
//      rank -- a NaN anywhere fails every rank the same way);
//   5. host plan (dist_plan below, identical on every rank): rank cuts in
//      global position space on bucket boundaries, except inside equality
//      buckets, which may be split anywhere (all their keys are equal);
//   6. the exchange FUSED into the level-0 scatter: k_scatter's per-bucket
//      cursors are pre-set to each bucket's final position in the owner's
//      receive buffer, addressed through CUDA IPC peer pointers over NVLink
//      (no all-to-all, no regroup copy: keys land bucket-major, sources in
//      rank order inside a bucket); a stream-ordered collective barrier;
//   7. local sort from level 1: every received bucket is a segment whose
//      model trains on its slice of the sorted global sample; equality-bucket
//      pieces are fills; the final stores (decoding float64) go to the
//      caller's output buffer.
//
// Collectives go through `Comm`: NCCL (dlopen'ed at run time, so the library
// loads and its single-GPU API works without NCCL), a one-rank no-op, or an
// in-process emulation (several virtual ranks on one device, one host thread
// each, host barriers between phases -- no kernel ever waits on another) that
// lets one GPU test the multi-rank data path (lsort_cuda_dist_emulate).
#include <dlfcn.h>
#include <nccl.h>  // types only: the functions are resolved with dlsym

#include <condition_variable>

#include "engine_core.cuh"

using namespace lsort_host;

namespace {

// ------------------------------------------------------------------ NCCL
struct NcclApi {
    ncclResult_t (*getUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*commInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*commInitAll)(ncclComm_t*, int, const int*) = nullptr;
    ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*allGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*allReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                              cudaStream_t) = nullptr;
    const char* (*errStr)(ncclResult_t) = nullptr;
    bool ok = false;
};

// The process's NCCL: the copy torch already loaded (same soname) or the system one.
NcclApi* nccl() {
    static NcclApi api;
    static std::once_flag once;
    std::call_once(once, [] {
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) return;
        api.getUniqueId = (decltype(api.getUniqueId))dlsym(h, "ncclGetUniqueId");
        api.commInitRank = (decltype(api.commInitRank))dlsym(h, "ncclCommInitRank");
        api.commInitAll = (decltype(api.commInitAll))dlsym(h, "ncclCommInitAll");
        api.commDestroy = (decltype(api.commDestroy))dlsym(h, "ncclCommDestroy");
        api.allGather = (decltype(api.allGather))dlsym(h, "ncclAllGather");
        api.allReduce = (decltype(api.allReduce))dlsym(h, "ncclAllReduce");
        api.errStr = (decltype(api.errStr))dlsym(h, "ncclGetErrorString");
        api.ok = api.getUniqueId && api.commInitRank && api.commInitAll && api.commDestroy && api.allGather &&
                 api.allReduce && api.errStr;
    });
    return api.ok ? &api : nullptr;
}

#define NC(call)                                                                                       \
    do {                                                                                               \
        ncclResult_t r__ = (call);                                                                     \
        if (r__ != ncclSuccess)                                                                        \
            throw LsortError{LSORT_ENCCL, std::string(#call) + ": " + nccl()->errStr(r__)};            \
    } while (0)

// ------------------------------------------------------------------ Comm
struct Comm {
    int rank = 0, world = 1;
    virtual ~Comm() {}
    // every rank's `bytes` of device src -> device dst (world x bytes, rank order), ordered on st
    virtual void allgather(const void* src, void* dst, size_t bytes, cudaStream_t st) = 0;
    // work queued on st after the barrier sees every rank's device writes issued before it
    virtual void barrier(cudaStream_t st) = 0;
    // collective: device pointers of every rank's `mine` (peers[rank] = mine)
    virtual void share(void* mine, std::vector<void*>& peers, cudaStream_t st) = 0;
    virtual void unshare(std::vector<void*>& peers) { peers.clear(); }
};

struct SelfComm : Comm {  // one rank, no NCCL
    void allgather(const void* src, void* dst, size_t bytes, cudaStream_t st) override {
        if (bytes && src != dst) CU(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToDevice, st));
    }
    void barrier(cudaStream_t) override {}
    void share(void* mine, std::vector<void*>& peers, cudaStream_t) override { peers.assign(1, mine); }
};

struct NcclComm : Comm {
    ncclComm_t comm = nullptr;
    bool own = true;
    DevBuf tiny, hbuf;
    PinBuf hpin;
    ~NcclComm() override {
        if (comm && own && nccl()) nccl()->commDestroy(comm);
    }
    void allgather(const void* src, void* dst, size_t bytes, cudaStream_t st) override {
        NC(nccl()->allGather(src, dst, bytes, ncclUint8, comm, st));
    }
    void barrier(cudaStream_t st) override {
        if (!tiny.ensure(8)) throw LsortError{LSORT_ENOMEM, "barrier"};
        NC(nccl()->allReduce(tiny.p, tiny.p, 1, ncclInt32, ncclSum, comm, st));
    }
    void share(void* mine, std::vector<void*>& peers, cudaStream_t st) override {
        unshare(peers);
        cudaIpcMemHandle_t h;
        CU(cudaIpcGetMemHandle(&h, mine));
        const size_t hb = sizeof(h);
        if (!hbuf.ensure(hb * (world + 1)) || !hpin.ensure(hb * (world + 1))) throw LsortError{LSORT_ENOMEM, "ipc"};
        std::memcpy(hpin.p, &h, hb);
        uint8_t* d = hbuf.as<uint8_t>();
        CU(cudaMemcpyAsync(d + hb * world, hpin.p, hb, cudaMemcpyHostToDevice, st));
        allgather(d + hb * world, d, hb, st);
        CU(cudaMemcpyAsync(hpin.p, d, hb * world, cudaMemcpyDeviceToHost, st));
        CU(cudaStreamSynchronize(st));
        peers.assign(world, nullptr);
        for (int r = 0; r < world; ++r) {
            if (r == rank) { peers[r] = mine; continue; }
            cudaIpcMemHandle_t pr;
            std::memcpy(&pr, hpin.as<uint8_t>() + hb * r, hb);
            CU(cudaIpcOpenMemHandle(&peers[r], pr, cudaIpcMemLazyEnablePeerAccess));
        }
    }
    void unshare(std::vector<void*>& peers) override {
        for (int r = 0; r < (int)peers.size(); ++r)
            if (r != rank && peers[r]) cudaIpcCloseMemHandle(peers[r]);
        peers.clear();
    }
};

// In-process emulation: `world` virtual ranks on one device, one host thread
// each. Collectives = stream synchronise + host barrier + device copies.
struct LocalGroup {
    int world;
    std::mutex mu;
    std::condition_variable cv;
    int arrived = 0;
    uint64_t gen = 0;
    std::vector<const void*> slots;
    explicit LocalGroup(int w) : world(w), slots(w, nullptr) {}
    void wait() {
        std::unique_lock<std::mutex> lk(mu);
        const uint64_t g = gen;
        if (++arrived == world) {
            arrived = 0;
            ++gen;
            cv.notify_all();
        } else {
            cv.wait(lk, [&] { return gen != g; });
        }
    }
};

struct LocalComm : Comm {
    LocalGroup* g;
    explicit LocalComm(LocalGroup* grp, int r) : g(grp) {
        rank = r;
        world = grp->world;
    }
    void allgather(const void* src, void* dst, size_t bytes, cudaStream_t st) override {
        CU(cudaStreamSynchronize(st));
        g->slots[rank] = src;
        g->wait();
        for (int r = 0; r < world; ++r)
            if (bytes) CU(cudaMemcpyAsync((uint8_t*)dst + bytes * r, g->slots[r], bytes, cudaMemcpyDeviceToDevice, st));
        CU(cudaStreamSynchronize(st));
        g->wait();  // every rank has read every slot
    }
    void barrier(cudaStream_t st) override {
        CU(cudaStreamSynchronize(st));
        g->wait();
    }
    void share(void* mine, std::vector<void*>& peers, cudaStream_t) override {
        g->slots[rank] = mine;
        g->wait();
        peers.assign(world, nullptr);
        for (int r = 0; r < world; ++r) peers[r] = (void*)g->slots[r];
        g->wait();
    }
};

// ------------------------------------------------------------------ plan
struct Piece {
    uint32_t b;
    uint64_t at, n;  // local offset in the receive buffer, keys
};
struct Plan {
    std::vector<uint64_t> cuts;     // world + 1 positions in the global sorted order
    std::vector<uint64_t> recv;     // keys each rank receives
    std::vector<uint32_t> dest;     // per bucket: owner rank of a moved bucket (~0: empty / equality)
    std::vector<uint64_t> dest_off; // per bucket: position of `rank`'s first key of b in the owner's buffer
    std::vector<Piece> pieces;      // `rank`'s received buckets / equality pieces, in key order
};

// H: world x nb counts (source-major); eq: nb flags (nullable). Identical on
// every rank given the same H. Cuts: target r N / world moved to the nearer
// boundary of the bucket holding it, unless that bucket is an equality bucket
// (split exactly at the target); the deviation from the ideal share is at most
// half the largest non-equality bucket.
Plan dist_plan(uint32_t world, uint32_t nb, const uint64_t* H, const uint8_t* eq, uint32_t rank) {
    Plan p;
    std::vector<uint64_t> P(nb + 1, 0);
    for (uint32_t b = 0; b < nb; ++b) {
        uint64_t g = 0;
        for (uint32_t s = 0; s < world; ++s) g += H[(size_t)s * nb + b];
        P[b + 1] = P[b] + g;
    }
    const uint64_t N = P[nb];
    p.cuts.assign(world + 1, 0);
    p.cuts[world] = N;
    uint32_t b = 0;
    for (uint32_t r = 1; r < world; ++r) {
        const uint64_t T = (uint64_t)(((unsigned __int128)N * r + world / 2) / world);
        while (b < nb && P[b + 1] <= T) ++b;  // P[b] <= T < P[b + 1] (or b == nb)
        uint64_t c;
        if (b >= nb) c = N;
        else if (eq && eq[b]) c = T;
        else c = (T - P[b] <= P[b + 1] - T) ? P[b] : P[b + 1];
        p.cuts[r] = std::max(c, p.cuts[r - 1]);
    }
    p.recv.resize(world);
    for (uint32_t r = 0; r < world; ++r) p.recv[r] = p.cuts[r + 1] - p.cuts[r];
    p.dest.assign(nb, ~0u);
    p.dest_off.assign(nb, 0);
    uint32_t owner = 0;
    for (uint32_t q = 0; q < nb; ++q) {
        if (P[q + 1] == P[q] || (eq && eq[q])) continue;
        while (owner + 1 < world && p.cuts[owner + 1] <= P[q]) ++owner;
        uint64_t before = 0;  // keys of bucket q on lower source ranks
        for (uint32_t s = 0; s < rank; ++s) before += H[(size_t)s * nb + q];
        p.dest[q] = owner;
        p.dest_off[q] = P[q] + before - p.cuts[owner];
    }
    const uint64_t lo = p.cuts[rank], hi = p.cuts[rank + 1];
    for (uint32_t q = 0; q < nb && lo < hi; ++q) {
        const uint64_t a = std::max(P[q], lo), e = std::min(P[q + 1], hi);
        if (a < e) p.pieces.push_back(Piece{q, a - lo, e - a});
    }
    return p;
}

struct ModelInfo {
    uint32_t kind = 0, nbuckets = 0;
    std::vector<uint8_t> eq;       // per bucket
    std::vector<uint64_t> eqval;   // per bucket (encoded key)
};

ModelInfo parse_model(const uint8_t* m) {
    ModelInfo mi;
    const ModelHdr* h = (const ModelHdr*)m;
    mi.kind = h->kind;
    mi.nbuckets = h->nbuckets;
    mi.eq.assign(mi.nbuckets, 0);
    mi.eqval.assign(mi.nbuckets, 0);
    if (h->kind == kTree) {
        const uint64_t* tree = (const uint64_t*)(m + sizeof(ModelHdr));
        const uint64_t* spl = tree + h->leaf_origin;
        const uint32_t* eqo = (const uint32_t*)(spl + h->nsplit);
        for (uint32_t i = 0; i < h->nsplit; ++i)  // SplitterTree equality buckets (models.hpp:96-100)
            if (eqo[i + 1] - eqo[i] > 1 && eqo[i] + 1 < mi.nbuckets) {
                mi.eq[eqo[i] + 1] = 1;
                mi.eqval[eqo[i] + 1] = spl[i];
            }
    }
    return mi;
}

constexpr uint32_t kDistTreeK = 256;   // splitter-tree fallback of the global model
constexpr uint32_t kDistShare = 16;    // poor global model: a bucket > 1 / (16 world) of the sample

}  // namespace

// ====================================================================== handle
struct lsort_dist {
    lsort_ctx* ctx = nullptr;
    std::unique_ptr<Comm> comm;
    int device = 0;
    std::string err;
    DevBuf recv;             // receive buffer, shared with the peers
    uint64_t recv_cap = 0;   // keys, identical on every rank
    uint64_t last_n = 0;     // keys of the last sort left in `recv` (no output buffer given)
    std::vector<void*> peers;
    DevBuf dseg, msg, allmsg, lsamp, gsamp, small;
    PinBuf hmsg, hmodel, hpin;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    ~lsort_dist() {
        if (ctx) {
            cudaSetDevice(device);
            cudaStreamSynchronize(ctx->stream);
            if (comm) comm->unshare(peers);
            if (ev0) cudaEventDestroy(ev0);
            if (ev1) cudaEventDestroy(ev1);
            lsort_cuda_ctx_destroy(ctx);
        }
    }
};

namespace {

uint64_t share_of(const std::vector<uint64_t>& n_all, uint64_t s_total, int r) {
    // per-rank sample sizes proportional to the shard sizes (sum == s_total)
    uint64_t N = 0;
    for (uint64_t v : n_all) N += v;
    if (N == 0) return 0;
    std::vector<uint64_t> sh(n_all.size());
    uint64_t tot = 0;
    for (size_t i = 0; i < n_all.size(); ++i) {
        sh[i] = (uint64_t)(((unsigned __int128)s_total * n_all[i]) / N);
        tot += sh[i];
    }
    for (size_t i = 0; tot < s_total; i = (i + 1) % n_all.size())
        if (n_all[i]) { ++sh[i]; ++tot; }
    return std::min(sh[r], n_all[r]);
}

struct DistResult {
    uint64_t n_out = 0, nan = ~0ull;
    int nan_rank = -1;
    uint32_t kind = 0, nb = 0;
    uint64_t n_global = 0, sample = 0;
    std::vector<uint64_t> recv;
};

// The per-rank driver (see the file comment). Throws LsortError.
void dist_sort(lsort_dist* D, void* keys, uint64_t n, int key_kind, void* out, uint64_t out_cap,
               const lsort_cfg& cfg, lsort_stats* stats, DistResult& res) {
    lsort_ctx* C = D->ctx;
    Comm& comm = *D->comm;
    const cudaStream_t st = C->stream;
    const int world = comm.world, rank = comm.rank;
    const bool f64 = key_kind == LSORT_KEY_F64;
    C->launches = 0;
    // pinned host words: [0,64) scalars, [64,80) two SegDescs, [80,82) tile prefix, [128, 128+world) sizes
    if (!D->hpin.ensure(8 * (256 + (size_t)world)) || !D->small.ensure(8 * (2 + (size_t)world)))
        throw LsortError{LSORT_ENOMEM, "dist control"};
    uint64_t* hp = D->hpin.as<uint64_t>();
    uint64_t* ds = D->small.as<uint64_t>();

    // ---- 1. shard sizes
    hp[0] = n;
    CU(cudaMemcpyAsync(ds + world, hp, 8, cudaMemcpyHostToDevice, st));
    comm.allgather(ds + world, ds, 8, st);
    CU(cudaMemcpyAsync(hp + 128, ds, 8 * (size_t)world, cudaMemcpyDeviceToHost, st));
    CU(cudaStreamSynchronize(st));
    std::vector<uint64_t> n_all(hp + 128, hp + 128 + world);
    uint64_t N = 0;
    for (uint64_t v : n_all) N += v;
    res.n_global = N;
    if (N == 0) return;

    // ---- 2. sample shares, local gather, all-gather (padded to the largest share)
    const uint64_t s_total = sample_size_host(cfg.sample_fraction, cfg.rmi_sample_cap, N);
    std::vector<uint64_t> sh(world);
    uint64_t smax = 1;
    for (int r = 0; r < world; ++r) {
        sh[r] = share_of(n_all, s_total, r);
        smax = std::max(smax, sh[r]);
    }
    uint64_t s_all = 0;
    for (uint64_t v : sh) s_all += v;
    res.sample = s_all;
    if (!D->lsamp.ensure(8 * smax) || !D->gsamp.ensure(8 * smax * world + 8 * s_all + 64) ||
        !D->dseg.ensure(2 * sizeof(SegDesc)))
        throw LsortError{LSORT_ENOMEM, "dist sample"};
    SegDesc* hseg = (SegDesc*)(hp + 64);  // [0] local shard, [1] the global segment (model building)
    std::memset(hseg, 0, 2 * sizeof(SegDesc));
    hseg[0].n = n;
    const uint64_t seed_r = splitmix64(cfg.seed ^ splitmix64(0x6A09E667F3BCC908ull + (uint64_t)rank));
    CU(cudaMemcpyAsync(D->dseg.p, hseg, sizeof(SegDesc), cudaMemcpyHostToDevice, st));
    if (sh[rank]) {
        launch_gather(D->dseg.as<SegDesc>(), keys, f64, seed_r, 0, sh[rank], D->lsamp.as<uint64_t>(), nullptr, st);
        ++C->launches;
    }
    uint64_t* gpad = D->gsamp.as<uint64_t>();
    uint64_t* gs = gpad + smax * world;
    comm.allgather(D->lsamp.p, gpad, 8 * smax, st);
    uint64_t at = 0;
    for (int r = 0; r < world; ++r) {
        if (sh[r]) CU(cudaMemcpyAsync(gs + at, gpad + smax * r, 8 * sh[r], cudaMemcpyDeviceToDevice, st));
        at += sh[r];
    }

    // ---- 3. global partition model from the gathered sample (identical on every rank)
    Engine E(C, cfg);
    const uint32_t B = fanout(N, cfg.rmi_bucket_count, 0);
    const uint32_t tk = world > 1 ? std::max<uint32_t>(kDistTreeK, cfg.tree_bucket_count) : cfg.tree_bucket_count;
    const uint32_t nb_max = std::max<uint32_t>(B, 2 * tk - 1);
    const size_t model_bytes =
        sizeof(ModelHdr) + std::max<size_t>(kLearnedEntryBytes * (size_t)B, (tree_payload_bytes(tk, tk - 1) + 15) & ~15ull);
    if (!C->models.ensure(model_bytes + 16) || !C->slices.ensure(4 * ((size_t)nb_max + 2)) ||
        !C->buckets.ensure(8 * (size_t)nb_max + 8) || !C->ctrl.ensure(sizeof(Ctrl)) ||
        !C->hctrl.ensure(sizeof(Ctrl)) || !C->hmodel.ensure(sizeof(ModelHdr)) || !C->segs.ensure(sizeof(SegDesc)) ||
        !C->tile_prefix.ensure(16) || !C->kseg.ensure(16) || !C->ktp.ensure(64) ||
        !C->kplan.ensure(3 * sizeof(KindPlan)) || !C->ids.ensure(2 * std::max<uint64_t>(n, 1)))
        throw LsortError{LSORT_ENOMEM, "dist workspace"};
    hseg[1].begin = 0;
    hseg[1].n = N;
    hseg[1].rmi_b = B;
    hseg[1].tree_k = tk;
    hseg[1].nb_max = nb_max;
    hseg[1].model_off = 0;
    hseg[0].rmi_b = B;
    hseg[0].tree_k = tk;
    hseg[0].nb_max = nb_max;
    CU(cudaMemcpyAsync(D->dseg.p, hseg, 2 * sizeof(SegDesc), cudaMemcpyHostToDevice, st));
    CU(cudaMemsetAsync(C->models.p, 0, sizeof(ModelHdr), st));
    CU(cudaMemsetAsync(C->slices.p, 0, 4 * ((size_t)nb_max + 2), st));
    E.given_sample = gs;
    E.given_n = s_all;
    E.share_den = world > 1 ? kDistShare * (uint32_t)world : 0;
    DevCfg dc = dev_cfg(cfg);
    {
        std::vector<SegPlan> gseg{SegPlan{0, N, 0, 0}};
        E.level_models({0u}, D->dseg.as<SegDesc>() + 1, gseg, &hseg[1], nullptr, false, nullptr, 0, 0, dc,
                       C->slices.as<uint32_t>());
    }

    // ---- 4. level-0 classify + histogram of the local shard
    Ctrl* dctrl = C->ctrl.as<Ctrl>();
    CU(cudaMemsetAsync(dctrl, 0, sizeof(Ctrl), st));
    CU(cudaMemsetAsync(&dctrl->nan_index, 0xff, 8, st));
    CU(cudaMemsetAsync(C->buckets.p, 0, 8 * (size_t)nb_max, st));
    const uint64_t ntiles = (n + kTileKeys - 1) / kTileKeys;
    uint64_t* pref = hp + 80;
    pref[0] = 0;
    pref[1] = ntiles;
    CU(cudaMemcpyAsync(C->segs.p, &hseg[0], sizeof(SegDesc), cudaMemcpyHostToDevice, st));
    CU(cudaMemcpyAsync(C->tile_prefix.p, pref, 16, cudaMemcpyHostToDevice, st));
    LevelParams p{};
    p.segs = C->segs.as<SegDesc>();
    p.nsegs = 1;
    p.tile_prefix = C->tile_prefix.as<uint64_t>();
    p.ntiles = ntiles;
    p.models = C->models.as<uint8_t>();
    p.buckets = C->buckets.as<unsigned long long>();
    p.src = keys;
    p.ids = C->ids.as<uint16_t>();
    p.ctrl = dctrl;
    p.kseg = C->kseg.as<uint32_t>();
    p.ktp = C->ktp.as<uint64_t>();
    p.kplan = C->kplan.as<KindPlan>();
    p.kstride = 1;
    p.remote = 1u;  // cursors preset by the rank plan (no k_scan_children); peers' buffers for world > 1
    const int grid = (int)std::max<uint64_t>(1, std::min<uint64_t>(ntiles, (uint64_t)num_sms() * kPartPerSM));
    if (n) {
        launch_kind_plan(p, st);
        launch_hist(p, f64, 7u, B, grid, st);  // learned, tree or cell table
        C->launches += 3;
    }

    // ---- all-gather: histogram | n | nan index | output capacity
    const size_t mw = (size_t)nb_max + 4;
    if (!D->msg.ensure(8 * mw) || !D->allmsg.ensure(8 * mw * world) || !D->hmsg.ensure(8 * mw * world) ||
        !D->hmodel.ensure(model_bytes + 16))
        throw LsortError{LSORT_ENOMEM, "dist histograms"};
    uint64_t* dm = D->msg.as<uint64_t>();
    CU(cudaMemcpyAsync(dm, C->buckets.p, 8 * (size_t)nb_max, cudaMemcpyDeviceToDevice, st));
    CU(cudaMemcpyAsync(dm + nb_max + 1, &dctrl->nan_index, 8, cudaMemcpyDeviceToDevice, st));
    hp[1] = n;
    hp[2] = out ? out_cap : ~0ull;
    CU(cudaMemcpyAsync(dm + nb_max, hp + 1, 8, cudaMemcpyHostToDevice, st));
    CU(cudaMemcpyAsync(dm + nb_max + 2, hp + 2, 8, cudaMemcpyHostToDevice, st));
    comm.allgather(dm, D->allmsg.p, 8 * mw, st);
    CU(cudaMemcpyAsync(D->hmsg.p, D->allmsg.p, 8 * mw * world, cudaMemcpyDeviceToHost, st));
    CU(cudaMemcpyAsync(D->hmodel.p, C->models.p, model_bytes, cudaMemcpyDeviceToHost, st));
    CU(cudaStreamSynchronize(st));
    const uint64_t* M = D->hmsg.as<uint64_t>();
    for (int r = 0; r < world; ++r) {
        const uint64_t nan = M[mw * r + nb_max + 1];
        if (nan != ~0ull && res.nan_rank < 0) {
            res.nan_rank = r;
            res.nan = nan;
        }
    }
    if (res.nan_rank >= 0) {
        if (res.nan_rank != rank) res.nan = ~0ull;
        throw LsortError{LSORT_ENAN, "NaN in rank " + std::to_string(res.nan_rank) + "'s shard"};
    }
    const ModelInfo mi = parse_model(D->hmodel.as<uint8_t>());
    const uint32_t nb = mi.nbuckets;
    res.kind = mi.kind;
    res.nb = nb;
    std::vector<uint64_t> H((size_t)world * nb);
    for (int r = 0; r < world; ++r) std::memcpy(&H[(size_t)r * nb], M + mw * r, 8 * (size_t)nb);

    // ---- 5. plan (identical on every rank)
    const Plan pl = dist_plan((uint32_t)world, nb, H.data(), mi.eq.data(), (uint32_t)rank);
    res.recv = pl.recv;
    res.n_out = pl.recv[rank];
    uint64_t need = 0;
    bool short_out = false;
    for (int r = 0; r < world; ++r) {
        need = std::max(need, pl.recv[r]);
        if (M[mw * r + nb_max + 2] < pl.recv[r]) short_out = true;
    }
    if (short_out)  // every rank learns this from the same data: all fail alike
        throw LsortError{LSORT_ENOMEM, "an output buffer is smaller than its rank's key range (n_out)"};
    if (need > D->recv_cap || D->peers.empty()) {  // collective re-registration
        const uint64_t cap = std::max<uint64_t>(need + need / 16 + 1024, D->recv_cap);
        if (!D->peers.empty()) {  // every rank closes its peer mappings before any buffer is freed
            comm.unshare(D->peers);
            comm.barrier(st);
            CU(cudaStreamSynchronize(st));
        }
        {
            DevBuf old;
            old.swap(D->recv);
        }
        if (!D->recv.ensure(8 * cap)) throw LsortError{LSORT_ENOMEM, "receive buffer"};
        D->recv_cap = cap;
        comm.share(D->recv.p, D->peers, st);
    }

    // ---- 6. exchange fused into the level-0 scatter (cursor = final position in the owner's buffer)
    uint64_t* recv = D->recv.as<uint64_t>();
    if (n) {
        uint64_t* cur = (uint64_t*)D->hmsg.p;  // (the gathered messages are consumed)
        for (uint32_t q = 0; q < nb; ++q) {
            cur[q] = 0;
            if (pl.dest[q] == ~0u || H[(size_t)rank * nb + q] == 0) continue;
            const int64_t base = ((intptr_t)D->peers[pl.dest[q]] - (intptr_t)recv) / 8;
            cur[q] = (uint64_t)(base + (int64_t)pl.dest_off[q]);
        }
        CU(cudaMemcpyAsync(C->buckets.p, cur, 8 * (size_t)nb, cudaMemcpyHostToDevice, st));
        p.dst = recv;
        launch_scatter(p, f64, nb_max, grid, st);
        ++C->launches;
    }
    comm.barrier(st);

    // ---- 7. local sort of the received range, final stores into `out`
    void* dst = out ? out : (void*)recv;
    const uint64_t nr = pl.recv[rank];
    if (nr == 0) return;
    const uint32_t cap = cfg.base_case_capacity;
    const uint32_t cls_cap[3] = {std::min<uint32_t>(kWarpBaseCap, cap), std::min<uint32_t>(4096, cap), cap};
    std::vector<uint32_t> offs(nb + 1, 0);
    CU(cudaMemcpyAsync(offs.data(), C->slices.p, 4 * ((size_t)nb + 1), cudaMemcpyDeviceToHost, st));
    CU(cudaStreamSynchronize(st));
    std::vector<SegPlan> big;
    std::vector<BaseItem> small[3];
    std::vector<FillItem> fills;
    for (const Piece& pc : pl.pieces) {
        if (mi.eq[pc.b]) {
            fills.push_back(FillItem{pc.at, pc.n, mi.eqval[pc.b], 0});
        } else if (pc.n > cap) {
            uint64_t ps = 0;
            const uint32_t o = offs[pc.b], l = offs[pc.b + 1] - o;
            if (!(cfg.flags & LSORT_FLAG_STRICT_POLICY) && l >= kMinSlice) ps = (uint64_t)o << 24 | std::min<uint32_t>(l, 0xffffffu);
            big.push_back(SegPlan{pc.at, pc.n, 1, 0, ps});
        } else {
            const int c = pc.n <= cls_cap[0] ? 0 : (pc.n <= cls_cap[1] ? 1 : 2);
            small[c].push_back(BaseItem{pc.at, pc.n, (int64_t)pc.at});
        }
    }
    if (stats) {
        for (auto& v : small) for (auto& it : v) stats->base_case_keys += it.n;
        for (auto& f : fills) stats->fill_keys += f.n;
        stats->base_segments += small[0].size() + small[1].size() + small[2].size();
    }
    if (!small[0].empty() || !small[1].empty() || !small[2].empty() || !fills.empty()) {
        size_t maxl = std::max<size_t>(1, fills.size());
        for (auto& v : small) maxl = std::max(maxl, v.size());
        if (!C->base[0].ensure(maxl * sizeof(BaseItem)) || !C->base[1].ensure(maxl * sizeof(BaseItem)) ||
            !C->base[2].ensure(maxl * sizeof(BaseItem)) || !C->fill.ensure(maxl * sizeof(FillItem)))
            throw LsortError{LSORT_ENOMEM, "dist base cases"};
        Ctrl* hc = C->hctrl.as<Ctrl>();
        std::memset(hc, 0, sizeof(Ctrl));
        hc->nan_index = ~0ull;
        LevelParams q{};
        q.ctrl = dctrl;
        for (int c = 0; c < 3; ++c) {
            hc->n_base[c] = (unsigned)small[c].size();
            if (!small[c].empty())
                CU(cudaMemcpyAsync(C->base[c].p, small[c].data(), small[c].size() * sizeof(BaseItem),
                                   cudaMemcpyHostToDevice, st));
            q.base[c] = C->base[c].as<BaseItem>();
        }
        hc->n_fill = (unsigned)fills.size();
        if (!fills.empty())
            CU(cudaMemcpyAsync(C->fill.p, fills.data(), fills.size() * sizeof(FillItem), cudaMemcpyHostToDevice, st));
        q.fill = C->fill.as<FillItem>();
        q.list_cap = (uint32_t)maxl;
        CU(cudaMemcpyAsync(dctrl, hc, sizeof(Ctrl), cudaMemcpyHostToDevice, st));
        launch_base_cases(q, recv, dst, f64, st);
        launch_fill(q, dst, f64, num_sms() * 4, st);
        C->launches += 4;
        CU(cudaStreamSynchronize(st));  // the host control block is reused by the engine
    }
    if (!big.empty()) {
        lsort_stats sti{};
        E.given_sample = nullptr;
        E.share_den = 0;
        E.sort(recv, nr, f64, stats ? &sti : nullptr, true, nullptr, &big, dst);
        if (stats) {
            stats->levels += sti.levels;
            stats->partitioned_keys += sti.partitioned_keys;
            stats->base_case_keys += sti.base_case_keys;
            stats->fill_keys += sti.fill_keys;
            stats->segments += sti.segments;
            stats->base_segments += sti.base_segments;
        }
    }
    if (stats) {
        stats->levels += 1;  // the distributed level 0
        stats->level0_kind = mi.kind == kLearned ? 0 : (mi.kind == kRadix ? 3 : 1);
        stats->partitioned_keys += n;
        stats->segments += 1;
    }
}

int dist_fail(lsort_dist* D, const LsortError& e) {
    if (D) {
        D->err = e.msg;
        if (e.code == LSORT_ENOMEM && !last_alloc_error().empty()) D->err += " (" + last_alloc_error() + ")";
    }
    last_alloc_error().clear();
    return e.code;
}

lsort_dist* new_dist(int device, std::unique_ptr<Comm> comm, int* rc) {
    lsort_ctx* c = nullptr;
    *rc = lsort_cuda_ctx_create(&c, device, nullptr, 0);
    if (*rc != LSORT_OK) return nullptr;
    lsort_dist* D = new lsort_dist();
    D->ctx = c;
    D->device = device;
    D->comm = std::move(comm);
    if (cudaEventCreate(&D->ev0) != cudaSuccess || cudaEventCreate(&D->ev1) != cudaSuccess) {
        cudaGetLastError();
        delete D;
        *rc = LSORT_ECUDA;
        return nullptr;
    }
    return D;
}

int run_dist(lsort_dist* D, void* keys, uint64_t n, int key_kind, void* out, uint64_t out_cap, uint64_t* n_out,
             const lsort_cfg* cfgp, lsort_stats* stats, uint64_t* nan_index_out) {
    if (!D) return LSORT_EINVAL;
    D->err.clear();
    if (nan_index_out) *nan_index_out = ~0ull;
    if (n_out) *n_out = 0;
    if (key_kind != LSORT_KEY_U64 && key_kind != LSORT_KEY_F64) return dist_fail(D, {LSORT_EINVAL, "key_kind"});
    if (n && !keys) return dist_fail(D, {LSORT_EINVAL, "null keys"});
    lsort_cfg cfg = cfg_or_default(cfgp);
    if (stats) std::memset(stats, 0, sizeof(*stats));
    DistResult res;
    try {
        validate_cfg(cfg);
        CU(cudaSetDevice(D->device));
        CU(cudaEventRecord(D->ev0, D->ctx->stream));
        dist_sort(D, keys, n, key_kind, out, out_cap, cfg, stats, res);
        CU(cudaEventRecord(D->ev1, D->ctx->stream));
        CU(cudaStreamSynchronize(D->ctx->stream));
        CU(cudaGetLastError());
        if (n_out) *n_out = res.n_out;
        D->last_n = out ? 0 : res.n_out;
        if (stats) {
            float ms = 0;
            cudaEventElapsedTime(&ms, D->ev0, D->ev1);
            stats->ms_total = ms;
            stats->kernel_launches = D->ctx->launches;
        }
    } catch (const LsortError& e) {
        cudaStreamSynchronize(D->ctx->stream);
        cudaGetLastError();
        if (n_out) *n_out = res.n_out;
        if (e.code == LSORT_ENAN && nan_index_out) *nan_index_out = res.nan;
        return dist_fail(D, e);
    }
    return LSORT_OK;
}

}  // namespace

// ======================================================================= C-ABI
extern "C" {

int lsort_nccl_available(void) { return nccl() ? 1 : 0; }

int lsort_nccl_unique_id(void* out128) {
    if (!out128) return LSORT_EINVAL;
    NcclApi* api = nccl();
    if (!api) return LSORT_ENCCL;
    ncclUniqueId id;
    if (api->getUniqueId(&id) != ncclSuccess) return LSORT_ENCCL;
    std::memcpy(out128, &id, sizeof(id));
    return LSORT_OK;
}

int lsort_cuda_dist_create(lsort_dist** out, int device, int world, int rank, const void* nccl_id) {
    if (!out || world < 1 || rank < 0 || rank >= world) return LSORT_EINVAL;
    *out = nullptr;
    std::unique_ptr<Comm> comm;
    if (world == 1 && !nccl_id) {
        comm.reset(new SelfComm());
    } else {
        if (!nccl_id) return LSORT_EINVAL;
        NcclApi* api = nccl();
        if (!api) return LSORT_ENCCL;
        if (cudaSetDevice(device) != cudaSuccess) { cudaGetLastError(); return LSORT_ECUDA; }
        std::unique_ptr<NcclComm> nc(new NcclComm());
        ncclUniqueId id;
        std::memcpy(&id, nccl_id, sizeof(id));
        if (api->commInitRank(&nc->comm, world, id, rank) != ncclSuccess) return LSORT_ENCCL;
        nc->rank = rank;
        nc->world = world;
        comm = std::move(nc);
    }
    int rc = LSORT_OK;
    lsort_dist* D = new_dist(device, std::move(comm), &rc);
    if (!D) return rc;
    *out = D;
    return LSORT_OK;
}

int lsort_cuda_dist_destroy(lsort_dist* D) {
    delete D;
    return LSORT_OK;
}

const char* lsort_cuda_dist_last_error(const lsort_dist* D) { return D ? D->err.c_str() : "null handle"; }

int lsort_cuda_dist_set_stream(lsort_dist* D, void* stream) {
    if (!D) return LSORT_EINVAL;
    return lsort_cuda_set_stream(D->ctx, stream);
}

int lsort_cuda_sort_dist(lsort_dist* D, void* d_keys, uint64_t n, int key_kind, void* d_out, uint64_t out_cap,
                         uint64_t* n_out, const lsort_cfg* cfg, lsort_stats* stats, uint64_t* nan_index_out) {
    return run_dist(D, d_keys, n, key_kind, d_out, out_cap, n_out, cfg, stats, nan_index_out);
}

int lsort_cuda_dist_result(lsort_dist* D, void** d_keys, uint64_t* n) {
    if (!D || !d_keys || !n) return LSORT_EINVAL;
    *d_keys = D->recv.p;
    *n = D->last_n;
    return LSORT_OK;
}

int lsort_dist_plan(uint32_t world, uint32_t nb, const uint64_t* H, const uint8_t* eq, uint32_t rank, uint64_t* cuts,
                    uint64_t* recv, uint32_t* dest, uint64_t* dest_off, uint64_t* pieces, uint32_t* npieces) {
    if (world == 0 || nb == 0 || !H || rank >= world || !cuts || !recv) return LSORT_EINVAL;
    const Plan p = dist_plan(world, nb, H, eq, rank);
    std::memcpy(cuts, p.cuts.data(), 8 * ((size_t)world + 1));
    std::memcpy(recv, p.recv.data(), 8 * (size_t)world);
    if (dest) std::memcpy(dest, p.dest.data(), 4 * (size_t)nb);
    if (dest_off) std::memcpy(dest_off, p.dest_off.data(), 8 * (size_t)nb);
    if (pieces) {
        for (size_t i = 0; i < p.pieces.size(); ++i) {
            pieces[3 * i] = p.pieces[i].b;
            pieces[3 * i + 1] = p.pieces[i].at;
            pieces[3 * i + 2] = p.pieces[i].n;
        }
    }
    if (npieces) *npieces = (uint32_t)p.pieces.size();
    return LSORT_OK;
}

// Several ranks in this process: NCCL over `ndev` devices (lsort_cuda_sort_multi),
// or `world` virtual ranks on one device (lsort_cuda_dist_emulate, test).
static int run_group(const std::vector<int>& devs, bool emulate, void* const* shards, const uint64_t* n,
                     int key_kind, void* const* outs, const uint64_t* out_caps, uint64_t* n_outs,
                     const lsort_cfg* cfg, lsort_stats* stats, uint64_t* nan_index_out, char* err, size_t errlen) {
    const int world = (int)devs.size();
    std::vector<std::unique_ptr<Comm>> comms(world);
    std::unique_ptr<LocalGroup> grp;
    if (emulate) {
        grp.reset(new LocalGroup(world));
        for (int r = 0; r < world; ++r) comms[r].reset(new LocalComm(grp.get(), r));
    } else if (world == 1) {
        comms[0].reset(new SelfComm());
    } else {
        NcclApi* api = nccl();
        if (!api) return LSORT_ENCCL;
        std::vector<ncclComm_t> cs(world);
        if (api->commInitAll(cs.data(), world, devs.data()) != ncclSuccess) return LSORT_ENCCL;
        for (int r = 0; r < world; ++r) {
            NcclComm* nc = new NcclComm();
            nc->comm = cs[r];
            nc->rank = r;
            nc->world = world;
            comms[r].reset(nc);
        }
    }
    std::vector<lsort_dist*> D(world, nullptr);
    int rc = LSORT_OK;
    for (int r = 0; r < world && rc == LSORT_OK; ++r) D[r] = new_dist(devs[r], std::move(comms[r]), &rc);
    std::vector<int> rcs(world, LSORT_OK);
    if (rc == LSORT_OK) {
        std::vector<std::thread> th;
        for (int r = 0; r < world; ++r)
            th.emplace_back([&, r] {
                rcs[r] = run_dist(D[r], shards[r], n[r], key_kind, outs ? outs[r] : nullptr,
                                  out_caps ? out_caps[r] : ~0ull, n_outs ? &n_outs[r] : nullptr, cfg,
                                  stats ? &stats[r] : nullptr, nan_index_out ? &nan_index_out[r] : nullptr);
            });
        for (auto& t : th) t.join();
        for (int r = 0; r < world; ++r)
            if (rcs[r] != LSORT_OK && rc == LSORT_OK) {
                rc = rcs[r];
                if (err && errlen) snprintf(err, errlen, "rank %d: %s", r, D[r]->err.c_str());
            }
    }
    for (auto* d : D) delete d;
    return rc;
}

int lsort_cuda_sort_multi(uint32_t ndev, const int* devices, void* const* d_shards, const uint64_t* n, int key_kind,
                          void* const* d_outs, const uint64_t* out_caps, uint64_t* n_outs, const lsort_cfg* cfg,
                          lsort_stats* stats, uint64_t* nan_index_out, char* err, size_t errlen) {
    if (ndev == 0 || !devices || !d_shards || !n || !d_outs || !out_caps) return LSORT_EINVAL;
    std::vector<int> devs(devices, devices + ndev);
    return run_group(devs, false, d_shards, n, key_kind, d_outs, out_caps, n_outs, cfg, stats, nan_index_out, err,
                     errlen);
}

int lsort_cuda_dist_emulate(int device, uint32_t world, void* const* d_shards, const uint64_t* n, int key_kind,
                            void* const* d_outs, const uint64_t* out_caps, uint64_t* n_outs, const lsort_cfg* cfg,
                            lsort_stats* stats, uint64_t* nan_index_out, char* err, size_t errlen) {
    if (world == 0 || !d_shards || !n || !d_outs || !out_caps) return LSORT_EINVAL;
    std::vector<int> devs(world, device);
    return run_group(devs, true, d_shards, n, key_kind, d_outs, out_caps, n_outs, cfg, stats, nan_index_out, err,
                     errlen);
}

}  // extern "C"
