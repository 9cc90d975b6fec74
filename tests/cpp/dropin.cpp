// Drop-in check of include/lsort/lsort.hpp: host uint64 / float64 sorts,
// NaN error with index, invalid config error. Built and run by
// tests/test_cpp_dropin.py (compile on CPU, run on the GPU box).
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <random>
#include <vector>

#include "lsort/lsort.hpp"

int main() {
    std::mt19937_64 g(7);
    std::vector<lsort::Key> k(2'000'000);
    for (auto& v : k) v = g() >> (g() & 31);
    std::vector<lsort::Key> ref = k;
    std::sort(ref.begin(), ref.end());
    lsort::sort(std::span<lsort::Key>(k));
    if (k != ref) { std::puts("u64 mismatch"); return 1; }

    std::normal_distribution<double> nd;
    std::vector<double> d(1'500'000);
    for (auto& v : d) v = nd(g);
    std::vector<double> dref = d;
    std::sort(dref.begin(), dref.end());
    lsort::sort(std::span<double>(d));
    if (d != dref) { std::puts("f64 mismatch"); return 1; }

    d[123] = std::nan("");
    d[77777] = std::nan("");
    try {
        lsort::sort(std::span<double>(d));
        std::puts("expected nan_error");
        return 1;
    } catch (const lsort::nan_error& e) {
        if (e.index() != 123) { std::puts("wrong NaN index"); return 1; }
    }
    // several host arrays in one call (copies pipelined against the sorts)
    std::vector<std::vector<double>> arrs(3);
    std::vector<std::span<double>> spans;
    for (size_t a = 0; a < arrs.size(); ++a) {
        arrs[a].resize(700'000 + 1000 * a);
        for (auto& v : arrs[a]) v = nd(g) * (double)(a + 1);
        spans.emplace_back(arrs[a]);
    }
    std::vector<std::vector<double>> aref = arrs;
    for (auto& r : aref) std::sort(r.begin(), r.end());
    lsort::sort_batch(std::span<std::span<double>>(spans));
    if (arrs != aref) { std::puts("batch mismatch"); return 1; }

    // LearnedSort 2.0 classic path
    std::vector<double> cd(1'200'000);
    for (auto& v : cd) v = nd(g);
    std::vector<double> cref = cd;
    std::sort(cref.begin(), cref.end());
    lsort::learned_sort_classic(std::span<double>(cd));
    if (cd != cref) { std::puts("classic mismatch"); return 1; }

    lsort::SortConfig bad;
    bad.rmi_bucket_count = 1000;  // not a power of two
    try {
        lsort::sort(std::span<lsort::Key>(k), bad);
        std::puts("expected invalid_argument");
        return 1;
    } catch (const std::invalid_argument&) {
    }
    std::puts("dropin ok");
    return 0;
}
