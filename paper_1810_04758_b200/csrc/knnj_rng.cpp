// Host-compiled (g++) home of the block mt19937_64 pair draw (knnj_rng.hpp), so the
// AVX2 clone dispatch stays out of nvcc's host pass.
#include "knnj_rng.hpp"

namespace kj {
void draw_pairs_fast(uint64_t N, uint64_t pairs, uint64_t seed, uint64_t* ij) {
    draw_pairs_stream(N, pairs, seed, ij);
}
}  // namespace kj
