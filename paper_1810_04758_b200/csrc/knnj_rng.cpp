// Host-compiled (g++) home of the block mt19937_64 draws (knnj_rng.hpp), so the
// AVX2 clone dispatch stays out of nvcc's host pass.
#include "knnj_rng.hpp"

#include <algorithm>
#include <memory>
#include <vector>

namespace kj {
void draw_pairs_fast(uint64_t N, uint64_t pairs, uint64_t seed, uint64_t* ij) {
    draw_pairs_stream(N, pairs, seed, ij);
}

// sample_without_replacement (proj/include/knnjoin/util.hpp:70-92) with the same output
// for the same mt19937_64 seed, restructured for memory-level parallelism:
//  * the draws j_i = uniform_int_distribution(i, n-1) do not depend on the index map, so
//    they are generated first, in one pass over the block engine;
//  * the map's keys below k (every i, and the j that land there) live in a dense array;
//    keys >= k in an open-addressing table whose slots are prefetched 32 draws ahead;
//  * the ascending sort (an LSD radix sort) is skipped when the caller does not need the
//    order: the histogram's counts do not depend on the order of its queries.
// The reference's loop does three unordered_map probes per draw, nearly all cache misses
// at k = 1e6 (~1 s at C5). `w` keeps the buffers across calls.
void sample_fast(uint64_t n, uint64_t k, uint64_t seed, uint64_t* out, bool sorted,
                 SampleWork* w) {
    if (k >= n) {
        for (uint64_t i = 0; i < n; ++i) out[i] = i;
        return;
    }
    std::unique_ptr<SampleWork> own;
    if (!w) {
        own = std::make_unique<SampleWork>();
        w = own.get();
    }
    std::vector<uint64_t>& J = w->J;
    std::vector<uint64_t>& D = w->D;
    J.resize(k);
    {
        auto st = std::make_unique<Mt64Stream>(seed);
        for (uint64_t i = 0; i < k; ++i) J[i] = i + st->below(n - i);
    }
    D.resize(k);
    for (uint64_t i = 0; i < k; ++i) D[i] = i;
    uint64_t cap = 16;
    while (cap < 2 * k + 16) cap <<= 1;
    std::vector<SampleWork::Slot>& T = w->T;
    T.assign(cap, SampleWork::Slot{~0ull, 0});
    const auto home = [&](uint64_t key) { return ((key * 0x9E3779B97F4A7C15ull) >> 17) & (cap - 1); };
    constexpr uint64_t PF = 32;
    for (uint64_t i = 0; i < k; ++i) {
        if (i + PF < k) {
            const uint64_t jp = J[i + PF];
            if (jp >= k) __builtin_prefetch(&T[home(jp)], 1);
            else __builtin_prefetch(&D[jp], 1);
        }
        const uint64_t j = J[i];
        const uint64_t iv = D[i];
        uint64_t jv;
        if (j < k) {
            jv = D[j];
            D[j] = iv;
        } else {
            uint64_t h = home(j);
            while (T[h].key != ~0ull && T[h].key != j) h = (h + 1) & (cap - 1);
            jv = T[h].key == j ? T[h].val : j;
            T[h].key = j;
            T[h].val = iv;
        }
        out[i] = jv;
    }
    if (!sorted) return;
    // ascending: LSD radix sort, 11-bit digits over the bits n - 1 needs
    int bits = 1;
    while (bits < 64 && ((n - 1) >> bits)) ++bits;
    std::vector<uint64_t>& tmp = w->J;  // the draws are consumed
    uint64_t* a = out;
    uint64_t* b = tmp.data();
    for (int sh = 0; sh < bits; sh += 11) {
        uint64_t cnt[2048] = {0};
        for (uint64_t i = 0; i < k; ++i) ++cnt[(a[i] >> sh) & 2047];
        uint64_t run = 0;
        for (int d = 0; d < 2048; ++d) {
            const uint64_t c = cnt[d];
            cnt[d] = run;
            run += c;
        }
        for (uint64_t i = 0; i < k; ++i) b[cnt[(a[i] >> sh) & 2047]++] = a[i];
        std::swap(a, b);
    }
    if (a != out) std::copy(a, a + k, out);
}
SampleWork* sample_work_new() { return new SampleWork(); }
void sample_work_free(SampleWork* w) { delete w; }
}  // namespace kj
