// tests/test_rng.py: the block mt19937_64 pair draw (knnj_rng.hpp) against the std types
// the reference uses (std::mt19937_64 + std::uniform_int_distribution<uint64_t>).
#include <cstdio>
#include <random>
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

int main() {
    int bad = 0;
    const uint64_t Ns[] = {2, 3, 7, 1000, 100000, 5000000, 20000000, (1ULL << 32) + 15,
                           (1ULL << 63) + 12345, 0xFFFFFFFFFFFFFFF0ULL};
    const uint64_t seeds[] = {0, 1, 12345, 0x9E3779B97F4A7C15ULL};
    for (uint64_t N : Ns)
        for (uint64_t sd : seeds) bad |= check(N, 30011, sd);
    bad |= check(5000000, 1000000, 987654321);
    std::printf(bad ? "FAIL\n" : "OK\n");
    return bad;
}
