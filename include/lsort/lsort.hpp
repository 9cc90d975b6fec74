// lsort/lsort.hpp -- C++20 drop-in for the reference's sort entry point
// (`sort(a, cfg)` in place over a contiguous range of keys,
// float64 pre-encoded with keys.hpp:36-42), backed by liblsort_cuda.so
// through the C-ABI in lsort_cuda.h. Header-only; link with -llsort_cuda.
//
//   lsort::SortConfig cfg;                 // SPEC.md:369-372 defaults
//   lsort::sort(std::span<lsort::Key>(v)); // host uint64 keys (copied in/out)
//   lsort::sort(std::span<double>(d));     // host float64; NaN -> lsort::nan_error
//   lsort::sort(lsort::device_span<double>{dptr, n});  // keys already in HBM
//   lsort::dist_sorter ds(dev, world, rank, &id);    // multi-GPU (one process per GPU)
//   size_t m = ds.sort(device_span<double>{shard, n}, device_span<double>{out, cap});
//
// Errors mirror the reference: invalid configuration -> std::invalid_argument
// (models.cpp:40-43), NaN -> lsort::nan_error (derived from
// std::invalid_argument) carrying the first NaN index (keys.hpp:34-42),
// CUDA / allocation failures -> lsort::cuda_error. One context per thread
// (thread_local), so concurrent sorts on disjoint arrays are safe
// (SPEC.md:445).
#ifndef LSORT_LSORT_HPP
#define LSORT_LSORT_HPP

#include <array>
#include <cstddef>
#include <cstdint>
#include <span>
#include <stdexcept>
#include <string>
#include <type_traits>
#include <vector>

#include "../lsort_cuda.h"

namespace lsort {

using Key = std::uint64_t;  // keys.hpp:18

struct SortConfig {
    std::uint32_t rmi_bucket_count = 1024;
    std::uint32_t tree_bucket_count = 256;
    std::uint64_t min_rmi_input = 100000;
    double max_duplicate_fraction = 0.10;
    std::uint32_t radix_base_case = 4096;
    std::uint32_t insertion_base_case = 16;
    std::uint32_t first_sample_cap = 2 * 256 * 16;
    std::uint32_t rmi_sample_cap = 1u << 20;
    double sample_fraction = 0.01;
    std::uint64_t seed = 0x5EED;
    std::uint32_t workers = 0;
    // GPU extensions
    std::uint32_t base_case_capacity = 16384;
    std::uint32_t bucket_target = 4096;
    int device = 0;

    lsort_cfg to_c() const {
        lsort_cfg c;
        lsort_cfg_default(&c);
        c.rmi_bucket_count = rmi_bucket_count;
        c.tree_bucket_count = tree_bucket_count;
        c.min_rmi_input = min_rmi_input;
        c.max_duplicate_fraction = max_duplicate_fraction;
        c.radix_base_case = radix_base_case;
        c.insertion_base_case = insertion_base_case;
        c.first_sample_cap = first_sample_cap;
        c.rmi_sample_cap = rmi_sample_cap;
        c.sample_fraction = sample_fraction;
        c.seed = seed;
        c.workers = workers;
        c.base_case_capacity = base_case_capacity;
        c.bucket_target = bucket_target;
        return c;
    }
};

class nan_error : public std::invalid_argument {
public:
    explicit nan_error(std::uint64_t index)
        : std::invalid_argument("lsort::sort: NaN at index " + std::to_string(index)), index_(index) {}
    std::uint64_t index() const noexcept { return index_; }

private:
    std::uint64_t index_;
};

class cuda_error : public std::runtime_error {
public:
    cuda_error(int code, const std::string& msg) : std::runtime_error(msg), code_(code) {}
    int code() const noexcept { return code_; }

private:
    int code_;
};

// Keys resident in device memory (HBM).
template <class T>
struct device_span {
    T* data;
    std::size_t size;
};

namespace detail {
struct Context {
    lsort_ctx* h = nullptr;
    int device = -1;
    ~Context() {
        if (h) lsort_cuda_ctx_destroy(h);
    }
    lsort_ctx* get(int dev) {
        if (h && device == dev) return h;
        if (h) lsort_cuda_ctx_destroy(h);
        h = nullptr;
        int rc = lsort_cuda_ctx_create(&h, dev, nullptr, 0);
        if (rc != LSORT_OK) throw cuda_error(rc, "lsort: cannot create a context on device " + std::to_string(dev));
        device = dev;
        return h;
    }
};
inline Context& context() {
    thread_local Context c;
    return c;
}
inline void run(void* keys, std::size_t n, int kind, int mem, const SortConfig& cfg) {
    lsort_ctx* h = context().get(cfg.device);
    lsort_cfg c = cfg.to_c();
    std::uint64_t nan_index = ~0ull;
    int rc = lsort_cuda_sort(h, keys, n, kind, mem, &c, nullptr, &nan_index);
    if (rc == LSORT_OK) return;
    if (rc == LSORT_ENAN) throw nan_error(nan_index);
    std::string msg = lsort_cuda_last_error(h);
    if (rc == LSORT_EINVAL) throw std::invalid_argument("lsort::sort: " + msg);
    throw cuda_error(rc, "lsort::sort: " + msg);
}
}  // namespace detail

// Several independent host arrays in one call (copies pipelined against the
// sorts). Throws nan_error for the first array holding a NaN (that array is
// left untouched, the others are sorted).
template <class T>
inline void sort_batch(std::span<std::span<T>> arrays, const SortConfig& cfg = {}) {
    static_assert(std::is_same_v<T, Key> || std::is_same_v<T, double>, "uint64 or double keys");
    lsort_ctx* h = detail::context().get(cfg.device);
    lsort_cfg c = cfg.to_c();
    std::vector<void*> ptrs;
    std::vector<std::uint64_t> ns, nans(arrays.size());
    for (auto& a : arrays) {
        ptrs.push_back(a.data());
        ns.push_back(a.size());
    }
    const int kind = std::is_same_v<T, double> ? LSORT_KEY_F64 : LSORT_KEY_U64;
    int rc = lsort_cuda_sort_batch(h, ptrs.data(), ns.data(), (std::uint32_t)arrays.size(), kind, &c, nullptr,
                                   nans.data());
    if (rc == LSORT_OK) return;
    if (rc == LSORT_ENAN)
        for (auto v : nans)
            if (v != ~0ull) throw nan_error(v);
    std::string msg = lsort_cuda_last_error(h);
    if (rc == LSORT_EINVAL) throw std::invalid_argument("lsort::sort_batch: " + msg);
    throw cuda_error(rc, "lsort::sort_batch: " + msg);
}

// sort(a, cfg) -- SPEC.md:384-392. Ascending, unstable.
inline void sort(std::span<Key> a, const SortConfig& cfg = {}) {
    detail::run(a.data(), a.size(), LSORT_KEY_U64, LSORT_MEM_HOST, cfg);
}
inline void sort(std::span<double> a, const SortConfig& cfg = {}) {
    detail::run(a.data(), a.size(), LSORT_KEY_F64, LSORT_MEM_HOST, cfg);
}
inline void sort(device_span<Key> a, const SortConfig& cfg = {}) {
    detail::run(a.data, a.size, LSORT_KEY_U64, LSORT_MEM_DEVICE, cfg);
}
inline void sort(device_span<double> a, const SortConfig& cfg = {}) {
    detail::run(a.data, a.size, LSORT_KEY_F64, LSORT_MEM_DEVICE, cfg);
}

// learned_sort_classic(a, cfg) -- SPEC.md:402-410 (the LearnedSort 2.0 path:
// one RMI, two partition rounds with it, model-based counting sort + fix-up).
template <class T>
inline void learned_sort_classic(std::span<T> a, const SortConfig& cfg = {}) {
    static_assert(std::is_same_v<T, Key> || std::is_same_v<T, double>, "uint64 or double keys");
    lsort_ctx* h = detail::context().get(cfg.device);
    lsort_cfg c = cfg.to_c();
    std::uint64_t nan_index = ~0ull;
    const int kind = std::is_same_v<T, double> ? LSORT_KEY_F64 : LSORT_KEY_U64;
    int rc = lsort_cuda_sort_classic(h, a.data(), a.size(), kind, LSORT_MEM_HOST, &c, nullptr, &nan_index);
    if (rc == LSORT_OK) return;
    if (rc == LSORT_ENAN) throw nan_error(nan_index);
    std::string msg = lsort_cuda_last_error(h);
    if (rc == LSORT_EINVAL) throw std::invalid_argument("lsort::learned_sort_classic: " + msg);
    throw cuda_error(rc, "lsort::learned_sort_classic: " + msg);
}

// ---- multi-GPU (lsort_cuda_sort_dist, one process per GPU) ----------------
// The distributed sort(a, cfg): every rank of a `world`-rank group holds a
// device shard; after sort() this rank holds the rank-th key range of the
// global order in `out`. The library owns the NCCL communicator: rank 0 calls
// nccl_unique_id() and the caller ships the 128 bytes to the other ranks (MPI,
// a file, torch.distributed ...). world == 1 needs no id. Collective: every
// rank calls sort() with its shard. A NaN anywhere -> nan_error on every rank
// (index() is meaningful on the owning rank only, ~0 elsewhere).
using nccl_id = std::array<char, 128>;
inline nccl_id nccl_unique_id() {
    nccl_id id{};
    int rc = lsort_nccl_unique_id(id.data());
    if (rc != LSORT_OK) throw cuda_error(rc, "lsort: NCCL is not available");
    return id;
}

class dist_sorter {
public:
    dist_sorter(int device, int world, int rank, const nccl_id* id = nullptr) {
        int rc = lsort_cuda_dist_create(&h_, device, world, rank, id ? id->data() : nullptr);
        if (rc != LSORT_OK) throw cuda_error(rc, "lsort::dist_sorter: cannot join the group");
    }
    ~dist_sorter() {
        if (h_) lsort_cuda_dist_destroy(h_);
    }
    dist_sorter(const dist_sorter&) = delete;
    dist_sorter& operator=(const dist_sorter&) = delete;
    // Returns the number of keys of this rank's range written to out.data.
    template <class T>
    std::size_t sort(device_span<T> shard, device_span<T> out, const SortConfig& cfg = {}) {
        static_assert(std::is_same_v<T, Key> || std::is_same_v<T, double>, "uint64 or double keys");
        lsort_cfg c = cfg.to_c();
        std::uint64_t n_out = 0, nan = ~0ull;
        const int kind = std::is_same_v<T, double> ? LSORT_KEY_F64 : LSORT_KEY_U64;
        int rc = lsort_cuda_sort_dist(h_, shard.data, shard.size, kind, out.data, out.size, &n_out, &c, nullptr, &nan);
        if (rc == LSORT_OK) return n_out;
        if (rc == LSORT_ENAN) throw nan_error(nan);
        std::string msg = lsort_cuda_dist_last_error(h_);
        if (rc == LSORT_EINVAL) throw std::invalid_argument("lsort::dist_sorter::sort: " + msg);
        throw cuda_error(rc, "lsort::dist_sorter::sort: " + msg + " (range " + std::to_string(n_out) + " keys)");
    }

private:
    lsort_dist* h_ = nullptr;
};

}  // namespace lsort

#endif
