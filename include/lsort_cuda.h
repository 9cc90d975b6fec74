/*
 * lsort_cuda.h -- C-ABI of the B200-native parallel LearnedSort (AIPS2o)
 * library liblsort_cuda.so (hand-written sm_100a CUDA kernels + C++ host
 * orchestrator). Plain pointers and sizes only; no torch or CUDA types.
 *
 * Reference interfaces each entry point replaces (paths under
 * /root/reference; the reference ships only the model layer in code, the sort
 * entry point is declared by its SPEC):
 *   lsort_cuda_sort          <- sort(a, cfg)
 *                               (+ encode_doubles/decode_doubles keys.hpp:36-46
 *                               for LSORT_KEY_F64: NaN -> first index, keys.hpp:34-42)
 *   lsort_cfg                <- SortConfig
 *   lsort_cuda_build_model   <- build_partition_model
 *   lsort_cuda_rmi_train     <- Rmi::train + enforce_monotonic
 *                                                             proj/src/models.cpp:39-131
 *   lsort_cuda_classify_rmi  <- PartitionModel::bucket_index (learned) + Rmi::predict
 *                                                             proj/src/models.hpp:34-65,162-171
 *   lsort_cuda_tree_build    <- SplitterTree::build          proj/src/models.cpp:133-185
 *   lsort_cuda_classify_tree <- SplitterTree::classify       proj/src/models.hpp:92-101
 *   lsort_cuda_verify        <- verify_sorted, multiset_hash proj/src/verify.hpp:17-29
 *   lsort_cuda_learned_pivots / lsort_cuda_pivot_quality / lsort_cuda_eta
 *                            <- learned_pivots_for_samplesort, pivot_quality, eta
 *                               SPEC.md:236-262 (Alg. 4, Table 1)
 *   lsort_gen_keys           <- data.generate
 *   lsort_read_keys / lsort_write_keys <- data.read_keys / write_keys SPEC.md:480-497
 *   (lsort_cli, csrc/cli.cpp  <- bench-cli generate / bench / verify SPEC.md:521-590)
 *   lsort_cuda_sort_dist / lsort_cuda_sort_multi
 *                            <- sort(a, cfg) with `workers` spanning GPUs;
 *                               the multi-GPU layer itself is new (SURVEY.md 8(b),(e))
 *
 * Conventions: return 0 (LSORT_OK) or an LSORT_E* code; the message is
 * available from lsort_cuda_last_error(ctx). LSORT_EINVAL mirrors the
 * reference's std::invalid_argument (models.cpp:40-43,135-138). A context is
 * single-threaded; concurrent sorts use separate contexts.
 * Calls are synchronous on return. The caller owns `keys`; the library owns
 * every workspace buffer (allocated per context, reused across calls).
 */
#ifndef LSORT_CUDA_H
#define LSORT_CUDA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define LSORT_OK 0
#define LSORT_EINVAL 1
#define LSORT_ENAN 2
#define LSORT_ENOMEM 3
#define LSORT_ECUDA 4
#define LSORT_ENCCL 5
#define LSORT_EINTERNAL 6
#define LSORT_EIO 7

#define LSORT_KEY_U64 0
#define LSORT_KEY_F64 1
/* keys already encoded as u64 (keys.hpp:36-42), result decoded to float64 in
 * place (lsort_cuda_sort only; the distributed local sort) */
#define LSORT_KEY_ENC_F64 2

#define LSORT_MEM_DEVICE 0
#define LSORT_MEM_HOST 1

#define LSORT_MAX_TREE 1024     /* max SplitterTree bucket budget */
#define LSORT_MAX_RMI 2048      /* max RMI submodels / output buckets on the GPU */

/* SortConfig plus GPU extensions. */
typedef struct lsort_cfg {
    uint32_t rmi_bucket_count;      /* 1024 */
    uint32_t tree_bucket_count;     /* 256 */
    uint64_t min_rmi_input;         /* 1e5 */
    double max_duplicate_fraction;  /* 0.10 */
    uint32_t radix_base_case;       /* 4096 (CPU reference; unused on the GPU) */
    uint32_t insertion_base_case;   /* 16 */
    uint32_t first_sample_cap;      /* 2*tree_bucket_count*16 = 8192 */
    uint32_t rmi_sample_cap;        /* 1<<20 */
    double sample_fraction;         /* 0.01 */
    uint64_t seed;
    uint32_t workers;               /* CPU reference only */
    /* --- GPU extensions --- */
    uint32_t base_case_capacity;    /* segments <= this go to the shared-memory base case (<=16384) */
    uint32_t bucket_target;         /* adaptive fan-out: ~keys per output bucket; 0 = fixed fan-out */
    uint32_t flags;                 /* reserved, 0 */
} lsort_cfg;

typedef struct lsort_rmi_header {
    double root_slope, root_intercept;
    double key_base, key_scale;     /* models.hpp:71-72 */
    uint32_t submodels;
    uint32_t reserved;
} lsort_rmi_header;

typedef struct lsort_rmi_entry {    /* LinearModel + clamp bounds, models.hpp:17-22,68-70 */
    double slope, intercept, lo, hi;
} lsort_rmi_entry;

typedef struct lsort_tree {         /* SplitterTree, models.hpp:110-116 */
    uint32_t levels, leaf_origin, nsplitters, bucket_count;
    uint64_t tree[LSORT_MAX_TREE];        /* implicit heap, 1-based */
    uint64_t splitters[LSORT_MAX_TREE];   /* strictly increasing */
    uint32_t eq_offset[LSORT_MAX_TREE + 1];
} lsort_tree;

/* Partition model chosen by the Alg. 5 policy for one segment. */
typedef struct lsort_model_info {
    uint32_t kind;                  /* 0 learned, 1 tree */
    uint32_t nbuckets;
    uint64_t first_sample;          /* s1 */
    uint64_t rmi_sample;            /* s2 (learned only) */
    double duplicate_fraction;      /* of the first sample */
} lsort_model_info;

typedef struct lsort_stats {
    double ms_total;                /* device time of the sort (events) */
    double ms_h2d, ms_d2h;          /* LSORT_MEM_HOST transfers */
    uint32_t levels;                /* distribution levels run (batch / many: summed over the arrays) */
    uint32_t level0_kind;           /* 0 learned (RMI), 1 tree, 2 base case only, 3 learned cell table (GPU policy) */
    uint64_t partitioned_keys;      /* keys moved by distribution passes (all levels) */
    uint64_t base_case_keys;
    uint64_t fill_keys;             /* keys written by equality/homogeneous fills */
    uint64_t segments;              /* segments partitioned */
    uint64_t base_segments;
    uint64_t kernel_launches;
    uint64_t h2d_bytes, d2h_bytes;
    /* per-phase device time (CUDA events between launch groups), filled when
     * cfg->flags has LSORT_FLAG_PHASE_TIMING; summed over levels */
    double ms_models, ms_classify, ms_scatter, ms_base, ms_fill;
    double ms_level0_classify, ms_level0_scatter;
    uint64_t level0_keys;
    uint64_t round2_buckets;        /* lsort_cuda_sort_classic: non-empty sub-buckets after round two */
    uint64_t direct_keys;           /* keys partitioned by the padded one-pass level 0 (no classify pass) */
} lsort_stats;

#define LSORT_FLAG_PHASE_TIMING 1u
/* cfg->flags: build every model exactly by the reference's Alg. 5 policy
 * (PAPER.md:389-415). Without it the GPU policy (1) lets segments of
 * >= min(min_rmi_input, 32768) keys take the learned branch (a learned model
 * classifies faster than a splitter-tree descent on the GPU) and (2) replaces
 * a learned model that puts more than 1/16 of its own sorted sample into one
 * bucket by a splitter tree over that sample (bucket imbalance costs whole
 * extra passes). The sorted output is identical either way;
 * lsort_cuda_build_model always runs strict. */
#define LSORT_FLAG_STRICT_POLICY 2u
/* cfg->flags: run every level >= 1 segment of 16 Ki..128 Ki keys through the
 * last distribution level fused with the base case in distributed shared
 * memory (thread-block clusters, cluster.cu). Without the flag the GPU policy
 * does so only when such segments hold at most 4 Mi keys in total (a few
 * leftovers: cheaper than a whole partition level); for a full level the
 * classify + scatter + base-case path is faster. */
#define LSORT_FLAG_CLUSTER 4u
/* cfg->flags, TEST ONLY: size the padded level-0 regions below their expected
 * counts so they overflow and the exact two-pass level runs instead (checks
 * the fallback of the one-pass level 0 that large learned roots take). */
#define LSORT_FLAG_TEST_DIRECT_OVERFLOW 8u
/* cfg->flags, TEST ONLY: behave as if the padded one-pass buffers (~1.2 N keys for
 * level 0, ~5 N for level 1) could not be allocated: the exact two-pass levels,
 * which need only the N-key scratch array and the bucket ids, run instead. */
#define LSORT_FLAG_TEST_NO_PADDED_MEM 16u

typedef struct lsort_ctx lsort_ctx;

void lsort_cfg_default(lsort_cfg* cfg);

int lsort_cuda_ctx_create(lsort_ctx** out, int device, void* cuda_stream /* nullable */,
                          size_t workspace_hint /* keys; 0 = grow on demand */);
int lsort_cuda_ctx_destroy(lsort_ctx* ctx);
const char* lsort_cuda_last_error(const lsort_ctx* ctx);
/* Set the stream for subsequent calls (nullable = the context's own
 * non-blocking stream, which is NOT ordered after work on the legacy default
 * stream: the caller synchronises that work first). */
int lsort_cuda_set_stream(lsort_ctx* ctx, void* cuda_stream);

/* In-place ascending sort of n keys (uint64 or float64). mem_kind DEVICE:
 * keys is device memory; HOST: host memory, copied in and out inside the
 * call. F64 keys containing NaN: returns LSORT_ENAN with the first NaN index
 * in *nan_index_out and leaves the array unmodified. */
int lsort_cuda_sort(lsort_ctx* ctx, void* keys, uint64_t n, int key_kind, int mem_kind,
                    const lsort_cfg* cfg, lsort_stats* stats, uint64_t* nan_index_out);

/* sort(a, cfg) over `count` independent HOST arrays in one call -- the
 * reference sorts each array with its own sort() (the
 * C2/C4 configs are three arrays). The copies are pipelined on two copy
 * streams against the sorts: array i+1 is copied in and array i-1 out while
 * array i sorts (three device buffers in flight; pinned host memory makes the
 * copies asynchronous). Arrays holding a NaN are left untouched and reported
 * in nan_index_out[i] (~0 otherwise); the call then returns LSORT_ENAN after
 * sorting all other arrays. stats (nullable) sums over the batch; ms_total is
 * the device time from the first copy-in to the last copy-out. */
int lsort_cuda_sort_batch(lsort_ctx* ctx, void* const* keys, const uint64_t* n, uint32_t count, int key_kind,
                          const lsort_cfg* cfg, lsort_stats* stats, uint64_t* nan_index_out);

/* sort(a, cfg) over `count` independent DEVICE arrays in one call: up to three
 * sorts run concurrently, each on its own internal context (stream +
 * workspace) driven by its own host thread, so one array's latency-bound
 * phases (model building, level hand-over) overlap another's partition and
 * base-case kernels. Synchronous on return; the same NaN / error contract as
 * lsort_cuda_sort_batch; stats (nullable) sums over the arrays (ms_total
 * is not filled). */
int lsort_cuda_sort_many(lsort_ctx* ctx, void* const* keys, const uint64_t* n, uint32_t count, int key_kind,
                         const lsort_cfg* cfg, lsort_stats* stats, uint64_t* nan_index_out);

/* ---- unit entry points (parity tests; device pointers) ---- */
int lsort_cuda_rmi_train(lsort_ctx* ctx, const uint64_t* d_sorted_sample, uint64_t s,
                         uint32_t submodels, lsort_rmi_header* h_out,
                         lsort_rmi_entry* h_entries_out);
int lsort_cuda_classify_rmi(lsort_ctx* ctx, const lsort_rmi_header* h,
                            const lsort_rmi_entry* entries, uint32_t bucket_count, double cdf_lo,
                            double cdf_hi, const void* d_keys, uint64_t n, int key_kind,
                            uint32_t* d_ids_opt, uint64_t* d_hist_opt);
int lsort_cuda_tree_build(lsort_ctx* ctx, const uint64_t* d_sorted_sample, uint64_t s,
                          uint32_t bucket_budget, int equality_mode, lsort_tree* h_out);
int lsort_cuda_classify_tree(lsort_ctx* ctx, const lsort_tree* t, const void* d_keys, uint64_t n,
                             int key_kind, uint32_t* d_ids_opt, uint64_t* d_hist_opt);
/* Alg. 5 on a whole device array (level 0): first sample, duplicate
 * fraction, RMI or tree. Learned params / tree are returned when non-null. */
int lsort_cuda_build_model(lsort_ctx* ctx, const void* d_keys, uint64_t n, int key_kind,
                           const lsort_cfg* cfg, lsort_model_info* info,
                           lsort_rmi_header* h_out, lsort_rmi_entry* entries_out,
                           lsort_tree* tree_out);
/* Device sort of a small device sample (the shared-memory block sort), n <= 8192. */
int lsort_cuda_block_sort(lsort_ctx* ctx, uint64_t* d_keys, uint64_t n);
/* verify_sorted + multiset_hash on device keys (F64 keys hashed encoded). */
int lsort_cuda_verify(lsort_ctx* ctx, const void* d_keys, uint64_t n, int key_kind,
                      uint64_t* first_violation /* 0 = sorted */, uint64_t* multiset_hash);

/* ---- pivot analysis ----
 * lsort_cuda_learned_pivots <- learned_pivots_for_samplesort (Alg. 4): the
 *   largest key of every learned cell i < b-1 under the given RMI (b output
 *   buckets, cdf range [0,1]); cells never hit are dropped; ascending,
 *   deduplicated. pivots_out (host) needs b-1 slots; keys in key_kind's
 *   representation (float64 bit patterns for LSORT_KEY_F64).
 * lsort_cuda_pivot_quality <- pivot_quality: sum_i |P(A <= p_i) - (i+1)/b| over
 *   the device-resident SORTED keys; LSORT_EINVAL unless np + 1 == b
 *   (SPEC.md:249). ranks_out (nullable, host, np) gets #keys <= p_i.
 * lsort_cuda_eta <- eta: max(P(A <= p), 1 - P(A <= p)) - 1/2. */
int lsort_cuda_learned_pivots(lsort_ctx* ctx, const lsort_rmi_header* h, const lsort_rmi_entry* entries,
                              uint32_t b, const void* d_keys, uint64_t n, int key_kind,
                              uint64_t* pivots_out, uint32_t* cells_out /* nullable: cell of each pivot */,
                              uint32_t* count_out);
int lsort_cuda_pivot_quality(lsort_ctx* ctx, const void* d_sorted, uint64_t n, int key_kind,
                             const uint64_t* pivots, uint32_t np, uint32_t b, double* distance_out,
                             uint64_t* ranks_out);
int lsort_cuda_eta(lsort_ctx* ctx, const void* d_sorted, uint64_t n, int key_kind, uint64_t pivot,
                   double* eta_out);

/* ---- host-side synthetic generators (BASELINE.json configs) ---- */
/* dist: 0 uniform, 1 normal, 2 lognormal(0,0.5), 3 exponential(2),
 * 4 mixgauss, 5 rootdups, 6 twodups, 7 zipf(0.75), 8 lognormal(0,2).
 * Writes elements [first, first+count) of the length-`total` dataset to host
 * memory `out` (double for 0-4,8; uint64 for 5-7). */
int lsort_gen_keys(int dist, uint64_t total, uint64_t seed, uint64_t first, uint64_t count,
                   void* out, int threads);

/* ---- key files (SPEC.md data module :480-497): an 8-byte little-endian count,
 * then count 8-byte little-endian keys. Host-only; no context needed. ---- */
/* read_keys: with keys == NULL only validates the file and returns its count
 * in *n_out; a truncated / oversized file is LSORT_EIO with the expected and
 * actual byte ranges in `err`. */
int lsort_read_keys(const char* path, uint64_t* keys, uint64_t capacity, uint64_t* n_out, char* err,
                    size_t errlen);
/* write_keys: inverse of read_keys (n == 0 writes the 8-byte zero count). */
int lsort_write_keys(const char* path, const uint64_t* keys, uint64_t n, char* err, size_t errlen);

/* LearnedSort 2.0 classic path (learned_sort_classic; PAPER.md
 * §2.2, §3.3): one RMI (cfg->rmi_bucket_count submodels) trained once on a
 * sample of min(sample_fraction n, rmi_sample_cap) keys drawn with
 * Rng(cfg->seed); round 1 partitions into B buckets, round 2 every bucket of
 * more than base_case_capacity keys into B sub-buckets with the SAME model
 * restricted to the bucket's CDF range (no sampling, no training); every
 * finished (sub-)bucket is placed by model-based counting sort and its
 * collisions fixed (the reference's insertion-sort sweep). Sub-buckets still
 * above the capacity (a poorly fitting model) continue with the AIPS2o
 * recursion. Same in-place / NaN / host-memory contract as lsort_cuda_sort. */
int lsort_cuda_sort_classic(lsort_ctx* ctx, void* keys, uint64_t n, int key_kind, int mem_kind,
                            const lsort_cfg* cfg, lsort_stats* stats, uint64_t* nan_index_out);
/* model_counting_sort of one device segment (n <= 8192):
 * d_out[] = d_keys[] placed by predicted position floor(n F(x)) over the CDF
 * range [cdf_lo, cdf_hi) (PartitionModel::bucket_index with n buckets,
 * models.hpp:128-138,162-171), stable for equal positions; sorted iff the
 * model is monotone and collision-free on the segment, else almost sorted. */
int lsort_cuda_model_counting_sort(lsort_ctx* ctx, const lsort_rmi_header* h, const lsort_rmi_entry* entries,
                                   double cdf_lo, double cdf_hi, const uint64_t* d_keys, uint64_t n,
                                   uint64_t* d_out);

/* Model forwarding (LearnedSort 2.0 classic path; Learned
 * cdf_lo / cdf_hi, models.hpp:128-138): sort device keys known to fall in
 * buckets [b_lo, b_hi) of the learned model (h, entries) with h->submodels
 * buckets. The root level reuses that model restricted to the CDF range
 * [b_lo/B, b_hi/B) with b_hi - b_lo buckets -- no sampling, no training;
 * with d_sorted_sample (the sorted sample the model was trained on, device)
 * the children train on their slices of it. The sorted output is the same as
 * lsort_cuda_sort's; keys outside the range are still sorted correctly (they
 * land in the first / last bucket). key_kind may be LSORT_KEY_ENC_F64. */
int lsort_cuda_sort_forward(lsort_ctx* ctx, void* d_keys, uint64_t n, int key_kind, const lsort_cfg* cfg,
                            const lsort_rmi_header* h, const lsort_rmi_entry* entries, uint32_t b_lo,
                            uint32_t b_hi, const uint64_t* d_sorted_sample, uint64_t sample_n,
                            lsort_stats* stats, uint64_t* nan_index_out);

/* Local sort of a rank's received keys when they are already grouped by the
 * global model's buckets [b_lo, b_hi) (bucket_sizes[b - b_lo] keys each, in
 * bucket order): buckets within the base-case capacity are sorted in place, the
 * others start the recursion at level 1 (children train on their slice of the
 * sorted global sample) -- no second level-0 pass. key_kind LSORT_KEY_U64 or
 * LSORT_KEY_ENC_F64 (decoded to float64 in the final stores). */
int lsort_cuda_sort_buckets(lsort_ctx* ctx, void* d_keys, uint64_t n, int key_kind, const lsort_cfg* cfg,
                            const lsort_rmi_header* h, const lsort_rmi_entry* entries, uint32_t b_lo,
                            uint32_t b_hi, const uint64_t* bucket_sizes /* host */,
                            const uint64_t* d_sorted_sample, uint64_t sample_n, lsort_stats* stats);
/* Decode encoded keys to float64 in place (after a distributed sort). */
int lsort_cuda_decode_inplace(lsort_ctx* ctx, uint64_t* d_keys, uint64_t n);

/* ---- multi-GPU driver (dist.cu; SURVEY.md 8(b),(e)) --------------------------
 * The distributed form of sort(a, cfg) (`workers` across
 * GPUs): every rank holds a shard; afterwards rank r holds the r-th key range
 * of the global sorted order (variable length), so the concatenation over
 * ranks is the sorted input. The library owns the NCCL communicator (NCCL is
 * loaded at run time; the single-GPU API does not need it). Per sort: the
 * global partition model (RMI, or a splitter tree when the RMI cannot balance
 * the ranks) is trained on a gathered global sample; rank cuts are chosen on
 * the all-gathered level-0 histograms; the exchange is fused into the level-0
 * scatter as NVLink stores into the owners' receive buffers (CUDA IPC); each
 * rank then sorts its range from level 1. A NaN in any shard fails every rank
 * with LSORT_ENAN (the owning rank gets the index). Collective: every rank
 * makes the same sequence of calls. */
typedef struct lsort_dist lsort_dist;

/* 1 when an NCCL library could be loaded into this process. */
int lsort_nccl_available(void);
/* ncclGetUniqueId into out[128] (rank 0; broadcast it to the other ranks). */
int lsort_nccl_unique_id(void* out128);
/* One rank of a `world`-rank group on `device`. nccl_id: the 128-byte id from
 * lsort_nccl_unique_id, or NULL with world == 1 (no NCCL needed). */
int lsort_cuda_dist_create(lsort_dist** out, int device, int world, int rank, const void* nccl_id);
int lsort_cuda_dist_destroy(lsort_dist* d);
const char* lsort_cuda_dist_last_error(const lsort_dist* d);
int lsort_cuda_dist_set_stream(lsort_dist* d, void* cuda_stream);
/* Globally sort the device shard d_keys[n] (LSORT_KEY_U64 / LSORT_KEY_F64).
 * The rank's key range (*n_out keys) is written to d_out (capacity out_cap;
 * d_out may equal d_keys). If any rank's out_cap is below its range, every
 * rank returns LSORT_ENOMEM with *n_out set. d_out == NULL: the range stays
 * in a library buffer (lsort_cuda_dist_result). stats (nullable): this rank's
 * counters; ms_total = device time on this rank. */
int lsort_cuda_sort_dist(lsort_dist* d, void* d_keys, uint64_t n, int key_kind, void* d_out, uint64_t out_cap,
                         uint64_t* n_out, const lsort_cfg* cfg, lsort_stats* stats, uint64_t* nan_index_out);
/* The library buffer holding the last range sorted with d_out == NULL
 * (encoded keys for LSORT_KEY_F64 are decoded; valid until the next call). */
int lsort_cuda_dist_result(lsort_dist* d, void** d_keys, uint64_t* n);
/* One process, `ndev` GPUs (ncclCommInitAll; one host thread per device):
 * shard i on devices[i], output range i into d_outs[i] (capacity out_caps[i]).
 * stats / nan_index_out / n_outs: per device, nullable. err (nullable): first
 * failing rank's message. */
int lsort_cuda_sort_multi(uint32_t ndev, const int* devices, void* const* d_shards, const uint64_t* n, int key_kind,
                          void* const* d_outs, const uint64_t* out_caps, uint64_t* n_outs, const lsort_cfg* cfg,
                          lsort_stats* stats, uint64_t* nan_index_out, char* err, size_t errlen);
/* TEST ENTRY: `world` virtual ranks on ONE device, one host thread each,
 * collectives emulated by host barriers + device copies (no kernel waits on
 * another). Runs the multi-GPU driver's data path -- global model, rank cuts,
 * exchange fused into the scatter, local sorts -- at world > 1 on one GPU. */
int lsort_cuda_dist_emulate(int device, uint32_t world, void* const* d_shards, const uint64_t* n, int key_kind,
                            void* const* d_outs, const uint64_t* out_caps, uint64_t* n_outs, const lsort_cfg* cfg,
                            lsort_stats* stats, uint64_t* nan_index_out, char* err, size_t errlen);
/* Host-only: the driver's rank plan from the world x nb bucket counts H
 * (source-major) and per-bucket equality flags eq (nullable). cuts[world+1]:
 * positions in the global order (bucket boundaries, or anywhere inside an
 * equality bucket); recv[world]: keys per rank; dest[nb] / dest_off[nb]
 * (nullable): owner rank of each moved bucket (~0 for empty / equality) and
 * the position of `rank`'s first key of it in the owner's buffer; pieces
 * (nullable, 3 x nb): `rank`'s received (bucket, local offset, count). */
int lsort_dist_plan(uint32_t world, uint32_t nb, const uint64_t* H, const uint8_t* eq, uint32_t rank, uint64_t* cuts,
                    uint64_t* recv, uint32_t* dest, uint64_t* dest_off, uint64_t* pieces, uint32_t* npieces);

#ifdef __cplusplus
}
#endif
#endif
