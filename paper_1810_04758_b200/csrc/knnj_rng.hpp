// Block-generated mt19937_64 and the reference's pair draw (estimate_eps_mean,
// proj/src/epsilon.cpp:14-44: std::mt19937_64 + std::uniform_int_distribution<uint64_t>).
//
// The output stream is std::mt19937_64's, bit for bit (the standard fixes the
// engine). The state is regenerated 312 words at a time in two dependency-free loops
// (vectorised, AVX2 where the CPU has it) instead of one word per call, and the
// values are mapped to [0, N) with libstdc++'s nearly-divisionless method, which is
// what std::uniform_int_distribution<uint64_t> runs for a 64-bit engine
// (bits/uniform_int_dist.h, _S_nd with unsigned __int128). tests/test_rng.py checks the
// pair stream against the std types for small, large and near-2^63 ranges.
#pragma once
#include <cstdint>
#include <vector>

namespace kj {

struct Mt64Block {
    static constexpr int NN = 312, MM = 156;
    static constexpr uint64_t MATRIX_A = 0xB5026F5AA96619E9ULL;
    static constexpr uint64_t UM = 0xFFFFFFFF80000000ULL, LM = 0x7FFFFFFFULL;
    uint64_t mt[NN];

    explicit Mt64Block(uint64_t seed) {
        mt[0] = seed;
        for (int i = 1; i < NN; ++i) mt[i] = 6364136223846793005ULL * (mt[i - 1] ^ (mt[i - 1] >> 62)) + (uint64_t)i;
    }
    // the next NN outputs (tempered) into out[0, NN)
    __attribute__((target_clones("avx2", "default"))) void next_block(uint64_t* out) {
        for (int i = 0; i < NN - MM; ++i) {
            const uint64_t y = (mt[i] & UM) | (mt[i + 1] & LM);
            mt[i] = mt[i + MM] ^ (y >> 1) ^ ((mt[i + 1] & 1ULL) ? MATRIX_A : 0ULL);
        }
        for (int i = NN - MM; i < NN - 1; ++i) {
            const uint64_t y = (mt[i] & UM) | (mt[i + 1] & LM);
            mt[i] = mt[i + MM - NN] ^ (y >> 1) ^ ((mt[i + 1] & 1ULL) ? MATRIX_A : 0ULL);
        }
        const uint64_t y = (mt[NN - 1] & UM) | (mt[0] & LM);
        mt[NN - 1] = mt[MM - 1] ^ (y >> 1) ^ ((mt[0] & 1ULL) ? MATRIX_A : 0ULL);
        for (int i = 0; i < NN; ++i) {
            uint64_t x = mt[i];
            x ^= (x >> 29) & 0x5555555555555555ULL;
            x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
            x ^= (x << 37) & 0xFFF7EEE000000000ULL;
            x ^= x >> 43;
            out[i] = x;
        }
    }
};

// Sequential consumer of the block stream (same order as repeated engine calls).
class Mt64Stream {
  public:
    explicit Mt64Stream(uint64_t seed) : g_(seed) {}
    uint64_t operator()() {
        if (at_ == kBuf) refill();
        return buf_[at_++];
    }
    // std::uniform_int_distribution<uint64_t>(0, range - 1) for 1 <= range < 2^64
    uint64_t below(uint64_t range) {
        unsigned __int128 prod = (unsigned __int128)(*this)() * range;
        uint64_t low = (uint64_t)prod;
        if (low < range) {
            const uint64_t threshold = (0 - range) % range;
            while (low < threshold) {
                prod = (unsigned __int128)(*this)() * range;
                low = (uint64_t)prod;
            }
        }
        return (uint64_t)(prod >> 64);
    }

  private:
    static constexpr int kBlocks = 64, kBuf = Mt64Block::NN * kBlocks;
    void refill() {
        for (int b = 0; b < kBlocks; ++b) g_.next_block(buf_ + b * Mt64Block::NN);
        at_ = 0;
    }
    Mt64Block g_;
    uint64_t buf_[kBuf];
    int at_ = kBuf;
};

// estimate_eps_mean's sampled pairs: i, j uniform in [0, N), j redrawn while j == i
inline void draw_pairs_stream(uint64_t N, uint64_t pairs, uint64_t seed, uint64_t* ij) {
    auto* st = new Mt64Stream(seed);  // ~160 KB buffer: heap, not the caller's stack
    for (uint64_t p = 0; p < pairs; ++p) {
        const uint64_t i = st->below(N);
        uint64_t j = st->below(N);
        while (j == i) j = st->below(N);
        ij[2 * p] = i;
        ij[2 * p + 1] = j;
    }
    delete st;
}

// buffers of sample_fast (knnj_rng.cpp), kept across calls by the caller
struct SampleWork {
    struct Slot {
        uint64_t key, val;
    };
    std::vector<uint64_t> J, D;
    std::vector<Slot> T;
};
// sample_without_replacement(n, k, std::mt19937_64(seed)) (util.hpp:70-92); ascending
// when `sorted`, else in an order that depends only on (n, k, seed)
void sample_fast(uint64_t n, uint64_t k, uint64_t seed, uint64_t* out, bool sorted = true,
                 SampleWork* w = nullptr);
SampleWork* sample_work_new();
void sample_work_free(SampleWork* w);

}  // namespace kj
