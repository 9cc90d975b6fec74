// cli.cpp -- lsort_cli, the command-line harness around the GPU sort
// (SPEC.md bench-cli module :521-590 and data module :458-519):
//
//   lsort_cli generate <name> <n> <seed> <out.bin> [--raw-f64]
//   lsort_cli sort <in.bin> <out.bin> [--f64] [--device D]
//   lsort_cli verify <file> [--f64]
//   lsort_cli bench --dataset <name|file> [--n N] [--runs R] [--seed S] [--warmup W]
//                   [--algo gpu-aips2o|reference]... [--csv out.csv] [--resident] [--device D]
//   lsort_cli pivot-quality <dataset> <n> <pivots> <trials> <seed> [csv_out] [--device D]
//
// Key files: 8-byte little-endian count + count 8-byte keys (lsort_read_keys /
// lsort_write_keys). Float datasets are written as encoded keys (keys.hpp:36-42,
// ordered as u64) unless --raw-f64. bench: per run a fresh copy of the input,
// a monotonic-clock timer around exactly the sort call (training included,
// SPEC.md:544), verify_sorted + multiset hash against the input, one CSV row
// `algorithm,dataset,n,workers,run,elapsed_ns,keys_per_second,verified`, then a
// summary block per algorithm; a failed verification fails the exit status.
// pivot-quality (Table 1): per trial, random-sampling
// pivots (IPS4o-style oversampling) and the RMI's implicit pivots (Alg. 4,
// lsort_cuda_learned_pivots) scored by pivot_quality against the sorted data;
// CSV `trial,method,requested,pivots,distance,flagged` plus a mean row per method
// (flagged: Alg. 4 dropped empty cells; the RMI set is still scored against b,
// an empty cell's boundary taking the last pivot below it).
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <map>
#include <string>
#include <vector>

#include "lsort/lsort.hpp"

namespace {

struct Dist {
    int id;
    bool f64;
};
const std::map<std::string, Dist>& registry() {
    static const std::map<std::string, Dist> r = {
        {"uniform", {0, true}},      {"normal", {1, true}},    {"lognormal", {2, true}},
        {"lognormal05", {2, true}},  {"exponential", {3, true}}, {"exponential2", {3, true}},
        {"mixgauss", {4, true}},     {"rootdups", {5, false}}, {"twodups", {6, false}},
        {"zipf", {7, false}},        {"lognormal2", {8, true}}};
    return r;
}
std::string registry_names() {
    std::string s;
    for (auto& kv : registry()) s += (s.empty() ? "" : ", ") + kv.first;
    return s;
}

uint64_t encode(double x) {  // keys.hpp:24-27
    uint64_t b;
    std::memcpy(&b, &x, 8);
    return (b & (1ull << 63)) ? ~b : (b ^ (1ull << 63));
}
uint64_t splitmix(uint64_t x) {  // rng.hpp:13-18 (multiset hash, verify.hpp:25-29)
    x += 0x9e3779b97f4a7c15ull;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
    return x ^ (x >> 31);
}

int usage() {
    std::fprintf(stderr,
                 "usage:\n"
                 "  lsort_cli generate <name> <n> <seed> <out.bin> [--raw-f64]\n"
                 "  lsort_cli sort <in.bin> <out.bin> [--f64] [--device D]\n"
                 "  lsort_cli verify <file> [--f64]\n"
                 "  lsort_cli bench --dataset <name|file> [--n N] [--runs R] [--seed S]\n"
                 "                  [--algo gpu-aips2o|reference]... [--csv out.csv] [--resident] [--device D]\n"
                 "                  [--warmup W]\n"
                 "  lsort_cli pivot-quality <dataset> <n> <pivots> <trials> <seed> [csv_out] [--device D]\n"
                 "generators: %s\n",
                 registry_names().c_str());
    return 2;
}

bool read_file(const std::string& path, std::vector<uint64_t>& keys) {
    char err[512] = {0};
    uint64_t n = 0;
    if (lsort_read_keys(path.c_str(), nullptr, 0, &n, err, sizeof err) != LSORT_OK) {
        std::fprintf(stderr, "%s\n", err);
        return false;
    }
    keys.resize(n);
    if (lsort_read_keys(path.c_str(), keys.data(), n, &n, err, sizeof err) != LSORT_OK) {
        std::fprintf(stderr, "%s\n", err);
        return false;
    }
    return true;
}
bool write_file(const std::string& path, const std::vector<uint64_t>& keys) {
    char err[512] = {0};
    if (lsort_write_keys(path.c_str(), keys.data(), keys.size(), err, sizeof err) != LSORT_OK) {
        std::fprintf(stderr, "%s\n", err);
        return false;
    }
    return true;
}

// the dataset in memory: u64 keys, or doubles when f64
struct Data {
    bool f64 = false;
    std::vector<uint64_t> u;
    std::vector<double> d;
    size_t size() const { return f64 ? d.size() : u.size(); }
};

bool generate(const std::string& name, uint64_t n, uint64_t seed, Data& out) {
    auto it = registry().find(name);
    if (it == registry().end()) {
        std::fprintf(stderr, "unknown generator '%s'; registry: %s\n", name.c_str(), registry_names().c_str());
        return false;
    }
    out.f64 = it->second.f64;
    void* p;
    if (out.f64) {
        out.d.resize(n);
        p = out.d.data();
    } else {
        out.u.resize(n);
        p = out.u.data();
    }
    if (n && lsort_gen_keys(it->second.id, n, seed, 0, n, p, 0) != LSORT_OK) {
        std::fprintf(stderr, "generate: bad arguments\n");
        return false;
    }
    return true;
}

int cmd_generate(int argc, char** argv) {
    if (argc < 6) return usage();
    const std::string name = argv[2], out = argv[5];
    const uint64_t n = std::strtoull(argv[3], nullptr, 10), seed = std::strtoull(argv[4], nullptr, 10);
    bool raw = false;
    for (int i = 6; i < argc; ++i) raw |= !std::strcmp(argv[i], "--raw-f64");
    Data d;
    if (!generate(name, n, seed, d)) return 2;
    std::vector<uint64_t> keys(d.size());
    for (size_t i = 0; i < keys.size(); ++i) {
        if (!d.f64) keys[i] = d.u[i];
        else if (raw) std::memcpy(&keys[i], &d.d[i], 8);
        else keys[i] = encode(d.d[i]);
    }
    return write_file(out, keys) ? 0 : 1;
}

int cmd_sort(int argc, char** argv) {
    if (argc < 4) return usage();
    bool f64 = false;
    lsort::SortConfig cfg;
    for (int i = 4; i < argc; ++i) {
        if (!std::strcmp(argv[i], "--f64")) f64 = true;
        else if (!std::strcmp(argv[i], "--device") && i + 1 < argc) cfg.device = std::atoi(argv[++i]);
    }
    std::vector<uint64_t> keys;
    if (!read_file(argv[2], keys)) return 2;
    try {
        if (f64) lsort::sort(std::span<double>(reinterpret_cast<double*>(keys.data()), keys.size()), cfg);
        else lsort::sort(std::span<lsort::Key>(keys), cfg);
    } catch (const lsort::nan_error& e) {
        std::fprintf(stderr, "NaN at index %llu\n", (unsigned long long)e.index());
        return 1;
    } catch (const std::exception& e) {
        std::fprintf(stderr, "%s\n", e.what());
        return 1;
    }
    return write_file(argv[3], keys) ? 0 : 1;
}

int cmd_verify(int argc, char** argv) {
    if (argc < 3) return usage();
    bool f64 = false;
    for (int i = 3; i < argc; ++i) f64 |= !std::strcmp(argv[i], "--f64");
    std::vector<uint64_t> keys;
    if (!read_file(argv[2], keys)) return 2;
    for (size_t i = 1; i < keys.size(); ++i) {
        uint64_t a = keys[i - 1], b = keys[i];
        if (f64) {
            double x, y;
            std::memcpy(&x, &a, 8);
            std::memcpy(&y, &b, 8);
            a = encode(x);
            b = encode(y);
        }
        if (b < a) {
            std::printf("violation at index %zu\n", i);
            return 1;
        }
    }
    std::printf("sorted (%zu keys)\n", keys.size());
    return 0;
}

// verify_sorted + multiset hash of encoded keys (verify.hpp:17-29)
bool check(const Data& in, const Data& out) {
    uint64_t h_in = 0, h_out = 0;
    const size_t n = in.size();
    for (size_t i = 0; i < n; ++i) {
        const uint64_t a = in.f64 ? encode(in.d[i]) : in.u[i];
        const uint64_t b = out.f64 ? encode(out.d[i]) : out.u[i];
        h_in += splitmix(a);
        h_out += splitmix(b);
        if (i) {
            const uint64_t p = out.f64 ? encode(out.d[i - 1]) : out.u[i - 1];
            if (b < p) {
                std::fprintf(stderr, "verification failed: violation at index %zu\n", i);
                return false;
            }
        }
    }
    if (h_in != h_out) std::fprintf(stderr, "verification failed: multiset hash mismatch\n");
    return h_in == h_out;
}

int cmd_bench(int argc, char** argv) {
    std::string dataset, csv;
    uint64_t n = 1000000, seed = 42;
    int runs = 10, warmup = 1;
    bool resident = false;
    std::vector<std::string> algos;
    lsort::SortConfig cfg;
    for (int i = 2; i < argc; ++i) {
        const std::string a = argv[i];
        auto next = [&]() -> std::string { return i + 1 < argc ? argv[++i] : ""; };
        if (a == "--dataset") dataset = next();
        else if (a == "--n") n = std::strtoull(next().c_str(), nullptr, 10);
        else if (a == "--runs") runs = std::atoi(next().c_str());
        else if (a == "--warmup") warmup = std::atoi(next().c_str());
        else if (a == "--seed") seed = std::strtoull(next().c_str(), nullptr, 10);
        else if (a == "--algo") algos.push_back(next());
        else if (a == "--csv") csv = next();
        else if (a == "--resident") resident = true;
        else if (a == "--device") cfg.device = std::atoi(next().c_str());
        else return usage();
    }
    if (dataset.empty() || runs < 1) return usage();
    if (algos.empty()) algos = {"gpu-aips2o", "reference"};
    for (auto& a : algos)
        if (a != "gpu-aips2o" && a != "reference") {
            std::fprintf(stderr, "unknown algorithm '%s'; registry: gpu-aips2o, reference\n", a.c_str());
            return 2;
        }
    Data input;
    if (registry().count(dataset)) {
        if (!generate(dataset, n, seed, input)) return 2;
    } else {
        if (!read_file(dataset, input.u)) return 2;
        n = input.u.size();
    }
    FILE* out = csv.empty() ? stdout : std::fopen(csv.c_str(), "w");
    if (!out) {
        std::fprintf(stderr, "cannot open %s\n", csv.c_str());
        return 2;
    }
    std::fprintf(out, "algorithm,dataset,n,workers,run,elapsed_ns,keys_per_second,verified\n");
    bool all_ok = true;
    struct Sum { std::vector<double> rate; };
    std::map<std::string, Sum> sums;
    const size_t bytes = input.size() * 8;
    void* dbuf = nullptr;
    if (resident && bytes) cudaMalloc(&dbuf, bytes);
    for (const auto& algo : algos) {
        for (int r = -warmup; r < runs; ++r) {  // r < 0: untimed warm-up (context, workspace)
            Data w = input;  // fresh copy per run (not timed)
            if (algo == "gpu-aips2o" && resident && dbuf)
                cudaMemcpy(dbuf, input.f64 ? (const void*)input.d.data() : (const void*)input.u.data(), bytes,
                           cudaMemcpyHostToDevice);
            const auto t0 = std::chrono::steady_clock::now();
            try {
                if (algo == "reference") {  // the host standard library's unstable sort
                    if (w.f64) std::sort(w.d.begin(), w.d.end(), [](double a, double b) { return encode(a) < encode(b); });
                    else std::sort(w.u.begin(), w.u.end());
                } else if (resident && dbuf) {
                    if (w.f64) lsort::sort(lsort::device_span<double>{(double*)dbuf, w.size()}, cfg);
                    else lsort::sort(lsort::device_span<lsort::Key>{(lsort::Key*)dbuf, w.size()}, cfg);
                } else {
                    if (w.f64) lsort::sort(std::span<double>(w.d), cfg);
                    else lsort::sort(std::span<lsort::Key>(w.u), cfg);
                }
            } catch (const std::exception& e) {
                std::fprintf(stderr, "%s: %s\n", algo.c_str(), e.what());
                return 1;
            }
            const auto t1 = std::chrono::steady_clock::now();
            if (algo == "gpu-aips2o" && resident && dbuf)
                cudaMemcpy(w.f64 ? (void*)w.d.data() : (void*)w.u.data(), dbuf, bytes, cudaMemcpyDeviceToHost);
            const double ns = (double)std::chrono::duration_cast<std::chrono::nanoseconds>(t1 - t0).count();
            const bool ok = check(input, w);
            all_ok &= ok;
            if (r < 0) continue;
            const double rate = (double)n / (ns * 1e-9);
            std::fprintf(out, "%s,%s,%llu,%d,%d,%.0f,%.1f,%s\n", algo.c_str(), dataset.c_str(),
                         (unsigned long long)n, 1, r, ns, rate, ok ? "true" : "false");
            if (ok) sums[algo].rate.push_back(rate);
        }
    }
    std::fprintf(out, "# summary\nalgorithm,dataset,n,workers,runs,mean_keys_per_second,stddev_keys_per_second\n");
    for (const auto& algo : algos) {
        const auto& v = sums[algo].rate;
        double m = 0, s = 0;
        for (double x : v) m += x;
        m = v.empty() ? 0 : m / v.size();
        for (double x : v) s += (x - m) * (x - m);
        s = v.size() > 1 ? std::sqrt(s / (v.size() - 1)) : 0;
        std::fprintf(out, "%s,%s,%llu,%d,%zu,%.1f,%.1f\n", algo.c_str(), dataset.c_str(), (unsigned long long)n, 1,
                     v.size(), m, s);
    }
    if (out != stdout) std::fclose(out);
    if (dbuf) cudaFree(dbuf);
    return all_ok ? 0 : 1;
}

// SPEC.md:550-558 cmd_pivot_quality
int cmd_pivot_quality(int argc, char** argv) {
    if (argc < 7) return usage();
    const std::string dataset = argv[2];
    const uint64_t n = std::strtoull(argv[3], nullptr, 10);
    const uint32_t want = (uint32_t)std::strtoul(argv[4], nullptr, 10);
    const int trials = std::atoi(argv[5]);
    const uint64_t seed = std::strtoull(argv[6], nullptr, 10);
    std::string csv;
    int device = 0;
    for (int i = 7; i < argc; ++i) {
        if (!std::strcmp(argv[i], "--device") && i + 1 < argc) device = std::atoi(argv[++i]);
        else csv = argv[i];
    }
    const uint32_t b = want + 1;
    if (n < 2 || want < 1 || trials < 1 || b > 2048) {
        std::fprintf(stderr, "pivot-quality: need n >= 2, 1 <= pivots <= 2047, trials >= 1\n");
        return 2;
    }
    Data data;
    if (!generate(dataset, n, seed, data)) return 2;
    std::vector<uint64_t> keys(n);  // encoded keys (keys.hpp:36-42): the model's domain
    for (uint64_t i = 0; i < n; ++i) keys[i] = data.f64 ? encode(data.d[i]) : data.u[i];
    lsort_ctx* ctx = nullptr;
    if (lsort_cuda_ctx_create(&ctx, device, nullptr, 0) != LSORT_OK) {
        std::fprintf(stderr, "pivot-quality: no CUDA device\n");
        return 1;
    }
    uint64_t *d_keys = nullptr, *d_sorted = nullptr, *d_smp = nullptr;
    const uint64_t smax = std::max<uint64_t>(2, std::min<uint64_t>((n + 99) / 100, 1ull << 20));
    cudaMalloc(&d_keys, n * 8);
    cudaMalloc(&d_sorted, n * 8);
    cudaMalloc(&d_smp, smax * 8);
    cudaMemcpy(d_keys, keys.data(), n * 8, cudaMemcpyHostToDevice);
    cudaMemcpy(d_sorted, keys.data(), n * 8, cudaMemcpyHostToDevice);
    int rc = lsort_cuda_sort(ctx, d_sorted, n, LSORT_KEY_U64, LSORT_MEM_DEVICE, nullptr, nullptr, nullptr);
    FILE* out = csv.empty() ? stdout : std::fopen(csv.c_str(), "w");
    if (!out) {
        std::fprintf(stderr, "cannot write %s\n", csv.c_str());
        return 1;
    }
    std::fprintf(out, "trial,method,requested,pivots,distance,flagged\n");
    // IPS4o oversampling factor alpha = 0.2 log2 n (at least 1)
    const uint32_t alpha = std::max<uint32_t>(1, (uint32_t)(0.2 * std::log2((double)n)));
    double sum[2] = {0, 0};
    std::vector<lsort_rmi_entry> ent(b);
    for (int t = 0; t < trials && rc == LSORT_OK; ++t) {
        const uint64_t st = splitmix(seed + 1 + (uint64_t)t);
        // random-sampling pivots: alpha * b keys, every alpha-th of the sorted sample
        std::vector<uint64_t> smp((size_t)alpha * b);
        for (size_t j = 0; j < smp.size(); ++j) smp[j] = keys[splitmix(st + j) % n];
        std::sort(smp.begin(), smp.end());
        std::vector<uint64_t> rp;
        for (uint32_t i = 0; i + 1 < b; ++i) {
            const uint64_t v = smp[(size_t)alpha * (i + 1) - 1];
            if (rp.empty() || v > rp.back()) rp.push_back(v);
        }
        // the RMI's pivots: model on a sorted sample (SPEC.md:438 size), Alg. 4 over all keys
        const uint64_t s = smax;
        std::vector<uint64_t> rs(s);
        const uint64_t st2 = splitmix(st ^ 0x5a3c9e1f0b7d2468ull);
        for (uint64_t j = 0; j < s; ++j) rs[j] = keys[splitmix(st2 + j) % n];
        std::sort(rs.begin(), rs.end());
        cudaMemcpy(d_smp, rs.data(), s * 8, cudaMemcpyHostToDevice);
        lsort_rmi_header h{};
        std::vector<uint64_t> lp(b);
        std::vector<uint32_t> cells(b);
        uint32_t nlp = 0;
        rc = lsort_cuda_rmi_train(ctx, d_smp, s, b, &h, ent.data());
        if (rc == LSORT_OK)
            rc = lsort_cuda_learned_pivots(ctx, &h, ent.data(), b, d_keys, n, LSORT_KEY_U64, lp.data(), cells.data(),
                                           &nlp);
        lp.resize(nlp);
        const std::vector<uint64_t>* sets[2] = {&rp, &lp};
        const char* names[2] = {"random", "rmi"};
        for (int m = 0; m < 2 && rc == LSORT_OK; ++m) {
            const auto& pv = *sets[m];
            double d = 0;
            std::vector<uint64_t> rk(pv.size() + 1);
            rc = lsort_cuda_pivot_quality(ctx, d_sorted, n, LSORT_KEY_U64, pv.data(), (uint32_t)pv.size(),
                                          (uint32_t)pv.size() + 1, &d, rk.data());
            if (rc == LSORT_OK && m == 1 && pv.size() != want) {
                // dropped cells: the pivot of boundary (g+1)/b is the largest key with
                // F < (g+1)/b (Alg. 4's definition) = the last pivot of a cell <= g
                // (rank 0 before the first one); scored against b
                d = 0;
                size_t j = 0;
                uint64_t r = 0;
                for (uint32_t g = 0; g + 1 < b; ++g) {
                    while (j < pv.size() && cells[j] <= g) r = rk[j++];
                    const double c = (double)r / (double)n, tg = (double)(g + 1) / (double)b;
                    d += c > tg ? c - tg : tg - c;
                }
            }
            sum[m] += d;
            std::fprintf(out, "%d,%s,%u,%zu,%.6f,%d\n", t, names[m], want, pv.size(), d, (int)(pv.size() != want));
        }
    }
    if (rc == LSORT_OK)
        for (int m = 0; m < 2; ++m)
            std::fprintf(out, "mean,%s,%u,,%.6f,\n", m ? "rmi" : "random", want, sum[m] / trials);
    else
        std::fprintf(stderr, "pivot-quality: %s\n", lsort_cuda_last_error(ctx));
    if (out != stdout) std::fclose(out);
    cudaFree(d_keys);
    cudaFree(d_sorted);
    cudaFree(d_smp);
    lsort_cuda_ctx_destroy(ctx);
    return rc == LSORT_OK ? 0 : 1;
}

}  // namespace

int main(int argc, char** argv) {
    if (argc < 2) return usage();
    const std::string cmd = argv[1];
    if (cmd == "generate") return cmd_generate(argc, argv);
    if (cmd == "sort") return cmd_sort(argc, argv);
    if (cmd == "verify") return cmd_verify(argc, argv);
    if (cmd == "bench") return cmd_bench(argc, argv);
    if (cmd == "pivot-quality") return cmd_pivot_quality(argc, argv);
    return usage();
}
