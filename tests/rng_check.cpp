// tests/test_rng.py: the block mt19937_64 pair draw (knnj_rng.hpp) against the std types
// the reference uses (std::mt19937_64 + std::uniform_int_distribution<uint64_t>).
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <random>
#include <unordered_map>
#include <vector>

#include "knnj_rng.hpp"

static int check(uint64_t N, uint64_t pairs, uint64_t seed) {
    std::vector<uint64_t> a(2 * pairs), b(2 * pairs);
    kj::draw_pairs_stream(N, pairs, seed, a.data());
    std::mt19937_64 rng(seed);
    std::uniform_int_distribution<uint64_t> pick(0, N - 1);
    for (uint64_t p = 0; p < pairs; ++p) {
        uint64_t i = pick(rng), j = pick(rng);
        while (j == i) j = pick(rng);
        b[2 * p] = i;
        b[2 * p + 1] = j;
    }
    // the stream must also continue identically afterwards
    kj::Mt64Stream s2(seed);
    std::mt19937_64 r2(seed);
    for (int k = 0; k < 50000; ++k)
        if (s2() != r2()) {
            std::printf("raw stream differs at %d (seed %llu)\n", k, (unsigned long long)seed);
            return 1;
        }
    for (uint64_t k = 0; k < 2 * pairs; ++k)
        if (a[k] != b[k]) {
            std::printf("N=%llu pairs=%llu seed=%llu: differs at %llu (%llu vs %llu)\n",
                        (unsigned long long)N, (unsigned long long)pairs, (unsigned long long)seed,
                        (unsigned long long)k, (unsigned long long)a[k], (unsigned long long)b[k]);
            return 1;
        }
    return 0;
}

// sample_without_replacement exactly as proj/include/knnjoin/util.hpp:70-92 writes it
static std::vector<uint64_t> ref_sample(uint64_t n, uint64_t k, uint64_t seed) {
    std::mt19937_64 rng(seed);
    if (k >= n) {
        std::vector<uint64_t> all(n);
        for (uint64_t i = 0; i < n; ++i) all[i] = i;
        return all;
    }
    std::vector<uint64_t> picked;
    std::unordered_map<uint64_t, uint64_t> remap;
    for (uint64_t i = 0; i < k; ++i) {
        std::uniform_int_distribution<uint64_t> dist(i, n - 1);
        uint64_t j = dist(rng);
        auto ji = remap.find(j);
        uint64_t jv = ji == remap.end() ? j : ji->second;
        auto ii = remap.find(i);
        uint64_t iv = ii == remap.end() ? i : ii->second;
        picked.push_back(jv);
        remap[j] = iv;
    }
    std::sort(picked.begin(), picked.end());
    return picked;
}

static int check_sample(uint64_t n, uint64_t k, uint64_t seed) {
    using clk = std::chrono::steady_clock;
    auto t0 = clk::now();
    std::vector<uint64_t> ref = ref_sample(n, k, seed);
    auto t1 = clk::now();
    std::vector<uint64_t> got(std::min(n, k));
    kj::sample_fast(n, k, seed, got.data());
    // unsorted mode: the same multiset
    std::vector<uint64_t> uns(got.size());
    kj::sample_fast(n, k, seed, uns.data(), false);
    std::sort(uns.begin(), uns.end());
    if (uns != ref) {
        std::printf("unsorted sample n=%llu k=%llu differs\n", (unsigned long long)n, (unsigned long long)k);
        return 1;
    }
    auto t2 = clk::now();
    if (k >= 100000)
        std::printf("sample n=%llu k=%llu: reference loop %.1f ms, sample_fast %.1f ms\n",
                    (unsigned long long)n, (unsigned long long)k,
                    std::chrono::duration<double, std::milli>(t1 - t0).count(),
                    std::chrono::duration<double, std::milli>(t2 - t1).count());
    if (ref != got) {
        std::printf("sample n=%llu k=%llu seed=%llu differs\n", (unsigned long long)n,
                    (unsigned long long)k, (unsigned long long)seed);
        return 1;
    }
    return 0;
}

int main() {
    int bad = 0;
    const uint64_t Ns[] = {2, 3, 7, 1000, 100000, 5000000, 20000000, (1ULL << 32) + 15,
                           (1ULL << 63) + 12345, 0xFFFFFFFFFFFFFFF0ULL};
    const uint64_t seeds[] = {0, 1, 12345, 0x9E3779B97F4A7C15ULL};
    for (uint64_t N : Ns)
        for (uint64_t sd : seeds) bad |= check(N, 30011, sd);
    bad |= check(5000000, 1000000, 987654321);
    // the histogram / parameter-search sampler: dense (k close to n), sparse, k >= n
    const uint64_t sn[][2] = {{1, 1}, {5, 10}, {100, 100}, {100, 99}, {1000, 1}, {1000, 700},
                              {100000, 1000}, {100000, 99990}, {5000000, 50000},
                              {(1ULL << 33) + 7, 20000}, {100000000, 1000000}};
    for (auto& c : sn)
        for (uint64_t sd : {0ull, 1ull, 77ull}) bad |= check_sample(c[0], c[1], sd);
    std::printf(bad ? "FAIL\n" : "OK\n");
    return bad;
}
