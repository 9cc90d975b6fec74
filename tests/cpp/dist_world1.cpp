// The multi-GPU entry points driven from C++ without torch:
// lsort::dist_sorter over an NCCL communicator the library owns (world 1 on
// the one GPU of the test box), lsort_cuda_sort_multi on one device, and the
// multi-rank data path through the in-process emulation (4 virtual ranks).
// Built and run by tests/test_cpp_dropin.py.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <random>
#include <vector>

#include "lsort/lsort.hpp"

static bool check(const std::vector<double>& got, std::vector<double> ref) {
    std::sort(ref.begin(), ref.end());
    return got == ref;
}

int main() {
    std::mt19937_64 g(11);
    std::lognormal_distribution<double> ln(0.0, 2.0);
    const size_t n = 3'000'000;
    std::vector<double> h(n);
    for (auto& v : h) v = ln(g);
    double *d_in = nullptr, *d_out = nullptr;
    cudaMalloc(&d_in, n * 8);
    cudaMalloc(&d_out, 2 * n * 8);
    // 1. dist_sorter, NCCL communicator of one rank
    lsort::nccl_id id = lsort::nccl_unique_id();
    {
        lsort::dist_sorter ds(0, 1, 0, &id);
        for (int rep = 0; rep < 2; ++rep) {
            cudaMemcpy(d_in, h.data(), n * 8, cudaMemcpyHostToDevice);
            size_t m = ds.sort(lsort::device_span<double>{d_in, n}, lsort::device_span<double>{d_out, 2 * n});
            std::vector<double> got(m);
            cudaMemcpy(got.data(), d_out, m * 8, cudaMemcpyDeviceToHost);
            if (m != n || !check(got, h)) { std::puts("dist_sorter mismatch"); return 1; }
        }
        // in place (out == shard)
        cudaMemcpy(d_in, h.data(), n * 8, cudaMemcpyHostToDevice);
        size_t m = ds.sort(lsort::device_span<double>{d_in, n}, lsort::device_span<double>{d_in, n});
        std::vector<double> got(m);
        cudaMemcpy(got.data(), d_in, m * 8, cudaMemcpyDeviceToHost);
        if (!check(got, h)) { std::puts("dist_sorter in-place mismatch"); return 1; }
    }
    // 2. lsort_cuda_sort_multi over one device
    {
        cudaMemcpy(d_in, h.data(), n * 8, cudaMemcpyHostToDevice);
        int dev = 0;
        void* shards[1] = {d_in};
        void* outs[1] = {d_out};
        uint64_t ns[1] = {n}, caps[1] = {2 * n}, nouts[1] = {0};
        char err[256] = {0};
        int rc = lsort_cuda_sort_multi(1, &dev, shards, ns, LSORT_KEY_F64, outs, caps, nouts, nullptr, nullptr,
                                       nullptr, err, sizeof(err));
        std::vector<double> got(nouts[0]);
        cudaMemcpy(got.data(), d_out, nouts[0] * 8, cudaMemcpyDeviceToHost);
        if (rc != LSORT_OK || !check(got, h)) { std::printf("sort_multi failed: %d %s\n", rc, err); return 1; }
    }
    // 3. four virtual ranks on this GPU (emulated collectives, real fused scatter)
    {
        const int W = 4;
        std::vector<void*> shards(W), outs(W);
        std::vector<uint64_t> ns(W), caps(W), nouts(W);
        const size_t per = n / W;
        for (int r = 0; r < W; ++r) {
            ns[r] = r == W - 1 ? n - per * (W - 1) : per;
            cudaMalloc(&shards[r], ns[r] * 8);
            cudaMemcpy(shards[r], h.data() + per * r, ns[r] * 8, cudaMemcpyHostToDevice);
            caps[r] = n;
            cudaMalloc(&outs[r], caps[r] * 8);
        }
        char err[256] = {0};
        int rc = lsort_cuda_dist_emulate(0, W, shards.data(), ns.data(), LSORT_KEY_F64, outs.data(), caps.data(),
                                         nouts.data(), nullptr, nullptr, nullptr, err, sizeof(err));
        if (rc != LSORT_OK) { std::printf("emulate failed: %d %s\n", rc, err); return 1; }
        std::vector<double> got;
        for (int r = 0; r < W; ++r) {
            std::vector<double> part(nouts[r]);
            cudaMemcpy(part.data(), outs[r], nouts[r] * 8, cudaMemcpyDeviceToHost);
            got.insert(got.end(), part.begin(), part.end());
            cudaFree(shards[r]);
            cudaFree(outs[r]);
        }
        if (!check(got, h)) { std::puts("emulated 4-rank sort mismatch"); return 1; }
    }
    cudaFree(d_in);
    cudaFree(d_out);
    std::puts("dist ok");
    return 0;
}
