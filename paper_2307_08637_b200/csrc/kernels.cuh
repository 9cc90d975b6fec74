// kernels.cuh -- shared declarations between kernels.cu and engine.cu.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "lsort_device.cuh"

namespace lsort_dev {

// One segment being partitioned at the current level.
struct SegDesc {
    uint64_t begin, n;       // absolute key range
    uint64_t model_off;      // byte offset in the model arena (16-aligned)
    uint64_t bucket_off;     // index into the per-bucket counter/cursor arena
    uint32_t depth, flags;   // flags: kSegForceRadix
    uint32_t nb_max, rmi_b;  // bucket slots reserved, learned fan-out
    uint32_t tree_k, pad;    // tree bucket budget
    uint64_t pslice;         // GPU policy: (offset << 24 | len) of this segment's keys in the
                             // parent level's sorted sample (DevCfg::psample), 0 = draw a sample
    uint64_t in_begin;       // where the segment's keys are READ (the level's input buffer);
                             // == begin except after a padded level-0 partition (k_direct),
                             // whose buckets sit at estimated offsets while `begin` (the write
                             // coordinates of this level's output) is exact
};
constexpr uint32_t kSegForceRadix = 1u;

// Child segment emitted for the next level.
struct SegOut {
    uint64_t begin, n;
    uint32_t depth, flags;
    uint64_t pslice;    // see SegDesc::pslice
    uint64_t in_begin;  // see SegDesc::in_begin
};
struct BaseItem {
    uint64_t begin, n;
    int64_t rd;  // read position, relative to the base kernels' source pointer (== begin
                 // except for the children of the padded one-pass level 0)
};
struct FillItem {
    uint64_t begin, n, value, pad;
};

// Device control block (zeroed per level, nan_index once per sort).
struct Ctrl {
    unsigned long long nan_index;   // first NaN index, ~0 if none
    unsigned int n_rec;
    unsigned int n_base[3];
    unsigned int n_fill;
    unsigned int err;
    unsigned int direct;            // level 0 ran the padded one-pass partition (k_direct)
    unsigned int run_exact;         // gate of the exact two-pass level (0 when k_direct succeeded)
    unsigned long long keys_fill, keys_base, keys_rec;
    unsigned long long verify_first;
    unsigned long long verify_hash;
    unsigned long long pad[4];
};

// Per-kind (learned / tree / radix) segment lists of a level.
struct KindPlan {
    uint32_t nsegs, pad;
    uint64_t ntiles;
};

// Parameters shared by the level kernels.
struct LevelParams {
    const SegDesc* segs;
    uint32_t nsegs;
    const uint64_t* tile_prefix;   // nsegs+1
    uint64_t ntiles;
    const uint8_t* models;         // model arena
    unsigned long long* buckets;   // counters -> cursors
    const void* src;               // keys in (level 0 may be f64)
    uint64_t* dst;                 // partitioned keys out (encoded)
    uint16_t* ids;                 // per key of src: bucket id written by k_hist, read by k_scatter
    const uint32_t* slices;        // level 0 only: [nb+1] offsets of each bucket's keys in the sorted
                                   // model sample (children train on them), or nullptr
                                   // (kNoMove: equality / fill bucket, the key is not moved)
    Ctrl* ctrl;
    SegOut* rec;
    BaseItem* base[3];
    FillItem* fill;
    uint32_t base_cap[3];          // size classes: n <= base_cap[c]
    uint32_t depth_cap;
    uint32_t list_cap;             // capacity of rec/base/fill lists
    const uint32_t* gate;          // nullptr, or: level runs only if *gate != 0
    uint32_t* kseg;                // [3][kstride] segment indices per kind
    uint64_t* ktp;                 // [3][kstride+1] tile prefixes per kind
    KindPlan* kplan;               // [3]
    uint32_t kstride;
    uint32_t remote;               // k_scatter: cursors preset by the multi-GPU rank plan, addressing
                                   // peer GPUs' receive buffers (exchange fused into the scatter, dist.cu)
    // one-pass level 1 over part of a level: seg_direct[j] = 1 when segment j is
    // handled by the one-pass kernels; seg_sel 1 = process only those, 2 = only the
    // others (the exact two-pass kernels), 0 = every segment
    const uint32_t* seg_direct;
    uint32_t seg_sel;
    int64_t rec_delta;             // k_scan_children: SegOut::in_begin = begin + rec_delta
};

// Sort configuration as seen by kernels.
struct DevCfg {
    uint64_t min_rmi_input;
    double max_dup;
    double sample_fraction;
    uint32_t first_sample_cap, rmi_sample_cap;
    uint64_t seed;
    uint32_t quality;  // 1: GPU policy -- a learned model that puts > 1/kPoorShare of its own
                       // sample into one bucket is replaced by a splitter tree over that sample
    const uint64_t* psample;  // GPU policy: the parent level's sorted sample (children's
                              // models train on their slice of it instead of drawing)
    uint32_t lut;             // GPU policy: learned-eligible segments below the root get a
                              // cell-table model (kModelLut) instead of an RMI
};
constexpr uint32_t kMinSlice = 64;  // shorter slices: draw a fresh sample
constexpr uint32_t kPoorShare = 16;
// GPU policy quality test: a learned model is poor when its largest bucket
// holds more than 1/kPoorShare of the sample AND more than kPoorMean times the
// mean bucket share (with 16 buckets, 1/16 alone would reject every model whose
// largest bucket is merely above average)
constexpr uint32_t kPoorMean = 4;
__host__ __device__ __forceinline__ bool poor_model(uint64_t mx, uint64_t s, uint32_t nb) {
    return mx * kPoorShare > s && mx * nb > (uint64_t)kPoorMean * s;
}

constexpr int kTileKeys = 4096;     // keys per classify/scatter tile
constexpr uint16_t kNoMove = 0xffff;
constexpr int kPartNT = 512;        // threads per classify/scatter CTA
constexpr int kPartPerSM = 2;       // resident classify/scatter CTAs per SM
constexpr int kRadixBits = 10;      // fallback radix model: 1024 buckets
constexpr uint32_t kSmallSampleCap = 8192;   // samples sortable in one model CTA
// cluster.cu: last level fused with the base case in distributed shared memory
constexpr int kClNT = 512;          // threads per CTA
constexpr int kClSize = 8;          // CTAs per cluster (portable maximum)
constexpr int kClRecv = 20480;      // keys an owner CTA can receive (160 KB)
constexpr int kClSub = 128;         // max sub-buckets per segment (kClCap / kClTarget <= 128)
constexpr int kClSortCap = 4096;    // max keys of a sub-bucket sorted in shared memory
constexpr uint32_t kClTarget = 1536;               // sub-bucket size target (upper bound of the mean)
constexpr uint32_t kClCap = kClSize * (kClRecv - kClSortCap);  // max keys per cluster segment
constexpr uint32_t kModelSmallCap = 2048;    // samples of the small model CTA

// Host-visible launchers.
// models.cu
// mid = 0: samples <= kModelSmallCap (256 threads); 1: <= kSmallSampleCap (512 threads)
void launch_build_models(const SegDesc* segs, const uint32_t* idx, uint32_t count, const void* src,
                         int in_f64, uint8_t* models, const DevCfg& cfg, int mid, cudaStream_t st);
// pre (nullable): the first sample already gathered (launch_gather draws [0, s1))
// dslices (nullable): when the policy builds a splitter tree (dup-heavy root), its
// buckets' offsets in the sorted first sample (the one-pass level 0 sizes regions from them)
void launch_first_sample(const SegDesc* seg, const void* src, int in_f64, uint8_t* models,
                         const DevCfg& cfg, uint8_t* aux, uint32_t aux_budget, uint32_t* gate,
                         cudaStream_t st, const uint64_t* pre = nullptr, uint32_t* dslices = nullptr);
void launch_gather(const SegDesc* seg, const void* src, int in_f64, uint64_t seed, uint64_t j0,
                   uint64_t s, uint64_t* out, const uint32_t* gate, cudaStream_t st);
size_t train_workspace_bytes(uint64_t s, uint32_t B);
// GPU policy (DevCfg::quality) for a big segment's learned model trained on the
// sorted sample: classify the sample, fall back to a splitter tree if poor.
// offs (nullable): also returns the final model's bucket offsets in the sample
// share_den > 0: also poor when the largest bucket holds more than 1/share_den of the sample;
// poor_share: the poor_model share test (1/poor_share of the sample, default kPoorShare)
void launch_quality_check(const uint64_t* sorted, uint64_t s, uint8_t* model, uint32_t tree_k, void* ws,
                          uint32_t* offs, const uint32_t* gate, cudaStream_t st, uint32_t share_den = 0,
                          uint32_t poor_share = kPoorShare);
size_t quality_workspace_bytes();
// GPU policy: a learned root becomes a cell-table model (kModelLut) when the
// table balances its sorted sample within 2x the mean bucket (models.cu)
size_t root_lut_workspace_bytes();
// (before the RMI training, which runs gated on *train_gate: skipped when the table is accepted)
// log_table: also try a binade-indexed table (float keys) -- first when log_first (a
// linear table classifies faster, a log table is accepted more often), else when
// the linear one is rejected
void launch_root_lut(const uint64_t* sorted, uint64_t s, uint8_t* model, void* ws, const uint32_t* gate,
                     uint32_t* train_gate, cudaStream_t st, bool log_table, bool log_first);
// offsets[b] = first index of the sorted sample whose bucket (under `model`) is >= b, b <= nb
void launch_sample_slices(const uint64_t* sorted, uint64_t s, const uint8_t* model, uint32_t* offsets,
                          uint32_t nb_cap, const uint32_t* gate, cudaStream_t st);
void launch_train_rmi(const uint64_t* sample, uint64_t s, uint32_t B, uint8_t* model, uint32_t nbuckets,
                      void* ws, const uint32_t* gate, cudaStream_t st);
void launch_tree_build(const uint64_t* sorted, uint64_t s, uint32_t budget, int eq_mode, uint8_t* model,
                       cudaStream_t st);
void launch_block_sort(uint64_t* keys, uint64_t n, cudaStream_t st);
// partition.cu
void launch_kind_plan(const LevelParams& p, cudaStream_t st);
void launch_hist(const LevelParams& p, int in_f64, uint32_t kinds, uint32_t max_rmi_b, int grid, cudaStream_t st);
void launch_scan_children(const LevelParams& p, uint32_t max_nb, cudaStream_t st);
// scatter of every segment of the level (all kinds), bucket ids from k_hist in p.ids
void launch_scatter(const LevelParams& p, int in_f64, uint32_t nb_cap, int grid, cudaStream_t st);
// One-pass (padded) level (k_direct, partition.cu): level 0 with the root
// sample's bucket offsets in p.slices (root_m samples). dw: direct_workspace_bytes(slots, nsegs)
// bytes (slots: the level's bucket counter slots); alloc_keys: capacity of
// p.dst (keys). Ctrl::direct / run_exact report the outcome on the device.
size_t direct_workspace_bytes(uint64_t slots, uint32_t nsegs);
// the one-pass level's outcome flag in its workspace (2: ineligible, 1: a region overflowed)
const uint32_t* direct_flag_ptr(const void* dw, uint64_t slots, uint32_t nsegs);
constexpr uint64_t kDirectMinPerBucket = 4096;   // mean keys per root bucket for the padded level 0
constexpr uint32_t kDirectMaxBuckets = 1024;     // buckets per segment a one-pass level handles
// One-pass level >= 1 over many segments (each a linear cell table with a slice of
// the parent's sorted sample psample); p.dst: the padded output (alloc_keys)
size_t direct_multi_workspace_bytes(uint64_t slots, uint32_t nsegs);
void launch_direct_multi(const LevelParams& p, const uint64_t* psample, uint64_t alloc_keys, void* dw, uint64_t slots,
                         int grid, cudaStream_t st, bool test_overflow, const uint64_t* base_src);
// base_src: the source pointer the level's base-case kernels are launched with (the
// direct children that go to the base cases read p.dst through it)
void launch_direct(const LevelParams& p, int in_f64, uint64_t root_m, uint64_t alloc_keys, void* dw, uint64_t slots,
                   int grid, cudaStream_t st, bool test_overflow, const uint64_t* base_src);
// bound on one segment's padded output: n keys, a model sample of m, nb buckets
uint64_t direct_capacity_bound(uint64_t n, uint64_t m, uint32_t nb);
// basecase.cu
void launch_base_cases(const LevelParams& p, const uint64_t* src, void* out, int out_f64, cudaStream_t st);
// cls 0: <= 1 Ki keys, 1: <= 4 Ki, 2: list 2 items > 8 Ki, 3: list 2 items <= 8 Ki
void launch_base_class(const LevelParams& p, int cls, const uint64_t* src, void* out, int out_f64, cudaStream_t st);
constexpr int kBaseLaunches = 4;
void launch_fill(const LevelParams& p, void* out, int out_f64, int grid, cudaStream_t st);
void launch_small_sort(void* keys, uint64_t n, int f64, Ctrl* ctrl, cudaStream_t st);
// classic.cu (LearnedSort 2.0 classic path)
void launch_forward_models(const SegDesc* segs, const uint32_t* idx, uint32_t count, const uint64_t* src,
                           const uint8_t* root, uint8_t* models, cudaStream_t st);
void launch_classic_base(const LevelParams& p, const uint64_t* src, void* out, int out_f64, const uint8_t* model,
                         int round, cudaStream_t st);
void launch_model_counting_sort(const uint8_t* model, const uint64_t* keys, uint64_t n, uint64_t* out,
                                cudaStream_t st);
// cluster.cu
bool cluster_available();
void launch_cluster_sort(const BaseItem* segs, uint32_t nsegs, const uint64_t* src, uint64_t* dst, void* out,
                         int out_f64, const LevelParams& p, uint32_t depth, cudaStream_t st);
// util.cu
void launch_classify_ids(const uint8_t* model, const void* keys, uint64_t n, int in_f64,
                         uint32_t* ids, uint16_t* ids16, unsigned long long* hist, int payload, cudaStream_t st);
void launch_verify(const void* keys, uint64_t n, int f64, Ctrl* ctrl, cudaStream_t st);
// Alg. 4 per-cell maxima (gmax / ghit zeroed by the caller, nbuckets cells)
void launch_learned_pivots(const uint8_t* model, const void* keys, uint64_t n, int in_f64, unsigned long long* gmax,
                           unsigned int* ghit, int payload, cudaStream_t st);
// ranks[i] = #keys <= pivots[i] (pivots encoded when f64)
void launch_rank_le(const void* sorted, uint64_t n, int f64, const uint64_t* pivots, uint32_t np, uint64_t* ranks,
                    cudaStream_t st);
void launch_copy_bytes(void* dst, const void* src, size_t bytes, cudaStream_t st);  // UVA pointers
void launch_decode(uint64_t* keys, uint64_t n, cudaStream_t st);
int num_sms();
void kernels_init();   // shared-memory opt-in for every kernel

constexpr uint32_t kWarpBaseCap = 1024;  // segments <= this: smallest base-case class

}  // namespace lsort_dev
