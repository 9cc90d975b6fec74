// classic.cu -- the LearnedSort 2.0 "classic" path (PAPER.md
// §2.2, §3.3): one RMI trained once on a 1% sample, two partition rounds with
// that SAME model, model-based counting sort of the sub-buckets, and a fix-up
// of the model's mistakes.
//
//   k_forward_models   round 2: every round-1 bucket b gets the root RMI
//                      restricted to its CDF range [b/B, (b+1)/B) with B output
//                      buckets (Learned cdf_lo / inv_span, models.hpp:128-138),
//                      compiled for the partition kernels -- no sampling, no
//                      training ("LearnedSort samples data only once").
//   k_classic_base     model_counting_sort + fix-up of a finished bucket: each
//                      key's digit is its predicted position within the
//                      bucket's CDF range (round 1: [b/B, (b+1)/B), round 2:
//                      [b/B + j/B^2, b/B + (j+1)/B^2)), counted into shared
//                      memory; keys that share a position are ordered by the
//                      collision fix-up (sorting networks / insertion sort for
//                      <= 16 keys, a range pass for larger groups) -- the GPU
//                      form of the reference's final insertion-sort sweep.
//   k_model_counting_sort  the unit: stable counting
//                      placement of one segment by predicted position, no
//                      fix-up (almost sorted where the model collides).
#include "kernels_common.cuh"
#include "smemsort.cuh"

namespace lsort_dev {

// models + off[idx[i]] <- root restricted to the round-1 bucket of the segment's keys
__global__ void __launch_bounds__(256) k_forward_models(const SegDesc* segs, const uint32_t* idx, const uint64_t* src,
                                                        const uint8_t* root, uint8_t* models) {
    griddep_wait();
    const SegDesc sd = segs[idx[blockIdx.x]];
    const ModelHdr& rh = *(const ModelHdr*)root;
    const RmiEntry* re = (const RmiEntry*)(root + sizeof(ModelHdr));
    const uint32_t B = rh.B;
    uint8_t* m = models + sd.model_off;
    ModelHdr* h = (ModelHdr*)m;
    RmiEntry* e = (RmiEntry*)(m + sizeof(ModelHdr));
    for (uint32_t i = threadIdx.x; i < B; i += 256) e[i] = re[i];
    if (threadIdx.x == 0) {
        // every key of the segment lies in one round-1 bucket: read it off the first
        const uint32_t b = learned_bucket(rh, re, src[sd.begin]);
        ModelHdr x = rh;
        x.nbuckets = B;
        x.cdf_lo = (double)b / (double)B;
        x.inv_span = (double)B;  // 1 / (1/B), exact for a power-of-two B
        *h = x;
    }
    __syncthreads();
    compile_learned(m, threadIdx.x, 256);
}

// CDF range of a finished bucket from its first key: round 1 -> [b/B, (b+1)/B),
// round 2 -> the sub-bucket j of b under the restricted model
__device__ __forceinline__ void classic_range(const ModelHdr& h, const RmiEntry* e, uint64_t x0, int round,
                                              double& lo, double& inv_span) {
    const double B = (double)h.B;
    const double f = rmi_predict(h, e, x0);
    const uint32_t b = cdf_bucket(f, 0.0, 1.0, h.B);
    lo = (double)b / B;
    inv_span = B;
    if (round == 2) {
        const uint32_t j = cdf_bucket(f, lo, B, h.B);
        lo = __dadd_rn(lo, (double)j / (B * B));
        inv_span = B * B;
    }
}

template <int IT, class SS, bool OUT_F64>
__device__ __forceinline__ void classic_one(uint64_t* g, uint32_t n, typename SS::SmemR& S, void* out, uint64_t begin,
                                            const ModelHdr& h, const RmiEntry* e, int round) {
    constexpr int NT = SS::kThreads;
    uint64_t k[IT];
#pragma unroll
    for (int i = 0; i < IT; ++i) {
        const uint32_t j = threadIdx.x + i * NT;
        k[i] = j < n ? __ldcs((const unsigned long long*)g + j) : 0ull;
    }
    double lo, inv;
    classic_range(h, e, g[0], round, lo, inv);
    constexpr uint32_t kNb = SS::kNbMax;
    const uint32_t lgnb = min(32u - __clz(max(n, 2u) - 1u), 31u - __clz(kNb));
    const uint32_t nb = 1u << lgnb;
    uint32_t dg[IT];
#pragma unroll
    for (int i = 0; i < IT; ++i) {  // predicted position, scaled to nb digits (monotone in the key)
        const uint32_t j = threadIdx.x + i * NT;
        dg[i] = j < n ? cdf_bucket(rmi_predict(h, e, k[i]), lo, inv, nb) : 0u;
    }
    SS::template sort_digits<IT, typename SS::SmemR, false>(k, dg, n, nb, S, g);
    for (uint32_t i = threadIdx.x; i < n; i += NT) {
        const uint64_t v = S.B[i];
        if (OUT_F64) __stcs((double*)out + begin + i, decode(v));
        else __stcs((unsigned long long*)out + begin + i, (unsigned long long)v);
    }
    __syncthreads();  // S.B is read before the next segment's placement
}

template <int NT, int CAP, int NBMAX, int MINB, bool OUT_F64>
__global__ void __launch_bounds__(NT, MINB) k_classic_base(const BaseItem* items, const unsigned int* count,
                                                           uint64_t* src, void* out, Ctrl* ctrl, uint32_t list_cap,
                                                           const uint8_t* model, int round) {
    griddep_wait();
    using SS = SmemSort<NT, CAP, NBMAX>;
    extern __shared__ uint4 smem_u4[];
    typename SS::SmemR& S = *(typename SS::SmemR*)smem_u4;
    if (ctrl->nan_index != ~0ull) return;
    const ModelHdr h = *(const ModelHdr*)model;
    const RmiEntry* e = (const RmiEntry*)(model + sizeof(ModelHdr));
    const uint32_t ni = min(*count, list_cap);
    for (uint32_t it = blockIdx.x; it < ni; it += gridDim.x) {
        const BaseItem b = items[it];
        const uint32_t n = (uint32_t)b.n;
        if (n <= (uint32_t)CAP / 2) classic_one<SS::ITEMS / 2, SS, OUT_F64>(src + b.begin, n, S, out, b.begin, h, e, round);
        else classic_one<SS::ITEMS, SS, OUT_F64>(src + b.begin, n, S, out, b.begin, h, e, round);
    }
}

// Unit (n <= 8192): stable counting placement by predicted position: the
// composite (position << 32 | input index) sorted in shared memory is the
// stable order.
using McsSS = SmemSort<512, 8192, 4096>;
__global__ void __launch_bounds__(512) k_model_counting_sort(const uint8_t* model, const uint64_t* keys, uint32_t n,
                                                            uint64_t* out) {
    griddep_wait();
    extern __shared__ uint4 smem_u4[];
    McsSS::Smem& S = *(McsSS::Smem*)smem_u4;
    const ModelHdr h = *(const ModelHdr*)model;
    const RmiEntry* e = (const RmiEntry*)(model + sizeof(ModelHdr));
    for (uint32_t i = threadIdx.x; i < n; i += 512) {
        const uint32_t p = cdf_bucket(rmi_predict(h, e, keys[i]), h.cdf_lo, h.inv_span, n);
        S.A[i] = (uint64_t)p << 32 | i;
    }
    __syncthreads();
    if (n > 1) {
        McsSS::sort_fast(S.A, n, S);
        for (uint32_t i = threadIdx.x; i < n; i += 512) out[i] = keys[(uint32_t)S.B[i]];
    } else if (n == 1 && threadIdx.x == 0) {
        out[0] = keys[0];
    }
}

// ------------------------------------------------------------- launchers
using ClsSmall = SmemSort<128, 1024, 1024>;
using ClsMid = SmemSort<256, 4096, 4096>;
using ClsBig = SmemSort<1024, 16384, 8192>;

void classic_init(int optin) {
    allow_smem(k_classic_base<128, 1024, 1024, 6, true>, optin);
    allow_smem(k_classic_base<128, 1024, 1024, 6, false>, optin);
    allow_smem(k_classic_base<256, 4096, 4096, 3, true>, optin);
    allow_smem(k_classic_base<256, 4096, 4096, 3, false>, optin);
    allow_smem(k_classic_base<1024, 16384, 8192, 1, true>, optin);
    allow_smem(k_classic_base<1024, 16384, 8192, 1, false>, optin);
    allow_smem(k_model_counting_sort, optin);
}

void launch_forward_models(const SegDesc* segs, const uint32_t* idx, uint32_t count, const uint64_t* src,
                           const uint8_t* root, uint8_t* models, cudaStream_t st) {
    if (count) pdl(k_forward_models, count, 256, 0, st, segs, idx, src, root, models);
}

void launch_classic_base(const LevelParams& p, const uint64_t* src, void* out, int out_f64, const uint8_t* model,
                         int round, cudaStream_t st) {
    const int nsm = num_sms();
    uint64_t* s = (uint64_t*)src;
    unsigned int* cnt = &p.ctrl->n_base[0];
    const size_t s0 = sizeof(ClsSmall::SmemR), s1 = sizeof(ClsMid::SmemR), s2 = sizeof(ClsBig::SmemR);
    if (out_f64) {
        pdl(k_classic_base<128, 1024, 1024, 6, true>, nsm * 6, 128, s0, st, p.base[0], cnt, s, out, p.ctrl, p.list_cap, model, round);
        pdl(k_classic_base<256, 4096, 4096, 3, true>, nsm * 3, 256, s1, st, p.base[1], cnt + 1, s, out, p.ctrl, p.list_cap, model, round);
        pdl(k_classic_base<1024, 16384, 8192, 1, true>, nsm, 1024, s2, st, p.base[2], cnt + 2, s, out, p.ctrl, p.list_cap, model, round);
    } else {
        pdl(k_classic_base<128, 1024, 1024, 6, false>, nsm * 6, 128, s0, st, p.base[0], cnt, s, out, p.ctrl, p.list_cap, model, round);
        pdl(k_classic_base<256, 4096, 4096, 3, false>, nsm * 3, 256, s1, st, p.base[1], cnt + 1, s, out, p.ctrl, p.list_cap, model, round);
        pdl(k_classic_base<1024, 16384, 8192, 1, false>, nsm, 1024, s2, st, p.base[2], cnt + 2, s, out, p.ctrl, p.list_cap, model, round);
    }
}

void launch_model_counting_sort(const uint8_t* model, const uint64_t* keys, uint64_t n, uint64_t* out,
                                cudaStream_t st) {
    pdl(k_model_counting_sort, 1, 512, sizeof(McsSS::Smem), st, model, keys, (uint32_t)n, out);
}

}  // namespace lsort_dev
