// CPU baselines (TEST / BENCH INFRASTRUCTURE ONLY -- the product never links
// this): the sorts BASELINE.md section 3 times beside the GPU path.
//   lso_std_sort_u64       std::sort, one thread (the paper's sequential
//                          baseline)
//   lso_parallel_sort_u64  libstdc++ parallel mode __gnu_parallel::sort
//                          (OpenMP) on `threads` threads: the stand-in for
//                          std::sort(std::execution::par_unseq, ...)
//                          (TBB is absent, so GCC's par_unseq
//                          would run serially)
// Both sort encoded uint64 keys (keys.hpp:36-42), i.e. the same order the
// LearnedSort port and the GPU produce.
#include <algorithm>
#include <cstdint>
#include <parallel/algorithm>
#include <omp.h>

extern "C" {

void lso_std_sort_u64(uint64_t* a, uint64_t n) { std::sort(a, a + n); }

void lso_parallel_sort_u64(uint64_t* a, uint64_t n, int threads) {
    if (threads <= 0) threads = omp_get_max_threads();
    omp_set_num_threads(threads);
    __gnu_parallel::sort(a, a + n, __gnu_parallel::default_parallel_tag(threads));
}

int lso_max_threads(void) { return omp_get_max_threads(); }

}  // extern "C"
