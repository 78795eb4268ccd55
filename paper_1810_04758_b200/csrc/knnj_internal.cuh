// Internal declarations shared by the device kernels (knnj_kernels.cu) and the
// host runtime / C ABI (knnj_capi.cu). Not part of the public ABI.
#pragma once

#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <map>
#include <utility>
#include <stdexcept>
#include <string>
#include <vector>

namespace kj {

// ---------------------------------------------------------------- errors
struct Error : std::runtime_error {
    int code;
    Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

#define KJ_CUDA(call)                                                                 \
    do {                                                                              \
        cudaError_t e_ = (call);                                                      \
        if (e_ != cudaSuccess)                                                        \
            throw ::kj::Error(9, std::string("CUDA error: ") + cudaGetErrorString(e_) + \
                                     " at " + __FILE__ + ":" + std::to_string(__LINE__)); \
    } while (0)

// ---------------------------------------------------------------- device buffer
// Device memory of a ctx never goes back to the driver between calls: blocks are
// recycled through the ctx's BlockCache (best fit, stream-ordered on the ctx's one
// stream), so a steady-state run performs no cudaMalloc at all. (Large
// cudaMallocAsync calls from a fragmented pool were measured at up to ~1 s.)
struct BlockCache {
    std::multimap<size_t, void*> free_blocks;       // bytes -> block
    std::vector<std::pair<void*, size_t>> owned;    // every block, freed at ctx destroy
    void* get(size_t bytes, size_t& got, cudaStream_t s);
    void put(void* p, size_t bytes) { free_blocks.emplace(bytes, p); }
    BlockCache() = default;
    BlockCache(const BlockCache&) = delete;
    ~BlockCache();
};
cudaStream_t& alloc_stream();
BlockCache*& alloc_cache();
template <class T>
struct DBuf {
    T* p = nullptr;
    size_t n = 0;      // capacity in elements
    size_t bytes = 0;  // size of the block behind p
    BlockCache* cache = nullptr;
    cudaStream_t s = nullptr;
    DBuf() = default;
    DBuf(const DBuf&) = delete;
    DBuf& operator=(const DBuf&) = delete;
    ~DBuf() { release(); }
    void release() {
        if (p) {
            if (cache) cache->put(p, bytes);
            else cudaFreeAsync(p, s);
        }
        p = nullptr;
        n = bytes = 0;
    }
    T* ensure(size_t count) {
        if (count == 0) count = 1;
        if (count > n) {
            release();
            s = alloc_stream();
            cache = alloc_cache();
            size_t got = count * sizeof(T);
            if (cache) {
                p = static_cast<T*>(cache->get(count * sizeof(T), got, s));
            } else {
                KJ_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&p), got, s));
            }
            bytes = got;
            n = got / sizeof(T);
        }
        return p;
    }
    T* get() const { return p; }
    void swap(DBuf& o) {
        std::swap(p, o.p);
        std::swap(n, o.n);
        std::swap(bytes, o.bytes);
        std::swap(cache, o.cache);
        std::swap(s, o.s);
    }
};

// ---------------------------------------------------------------- constants
constexpr int JB = 128;          // threads (= queries) per join / histogram block
constexpr uint32_t OVF = 0xFFFFFFFFu;
constexpr uint32_t SKIP = 0xFFFFFFFEu;
constexpr uint32_t FB = 128;     // positions per candidate block of the box filter  // list count of a row whose item was split into parts

// Status bits written by the finalize kernel, per query.
enum : uint8_t {
    ST_HAS_K = 1,      // >= K candidates (non-self) in the candidate set
    ST_IN_EPS = 2,     // K-th exact sq <= eps^2 (dense "solved" rule, dense_engine.cpp:182)
    ST_CERT = 4,       // K-th exact sq < coverage^2 (1-eta): globally exact
    ST_OVF = 8,        // screen list overflowed (many near-ties): needs the exact slow path
    ST_MISS = 16,      // radius-bounded pass: fewer than K candidates within the bound, or
                       // the list overflowed; the row is re-run without the bound
};

// One grid level over all points (level 0 is the reference ε-grid; level L
// has cell width ε·2^L, nested exactly in level 0).
struct Level {
    bool built = false;
    uint32_t m = 0;
    double w = 0.0;
    double prec_w = 0.0;  // width the tcgen05 precision rule compares the screen band with
                          // (w; a radius-bounded fine grid keeps level 0's: its cut is a
                          // K-th distance, not a cell width)
    std::vector<double> mins, maxs;
    std::vector<uint64_t> cpd, strides;
    uint64_t ncells = 0;
    uint64_t npts = 0;   // points in the tables (all N, or a slice: the histogram's shard grid)
    uint32_t key_bits = 0;
    DBuf<uint64_t> B;    // ncells: sorted non-empty linear cell ids
    DBuf<uint2> G;       // ncells: [begin,end) into A
    DBuf<uint32_t> A;    // N: sorted position -> point id
    DBuf<uint32_t> slot; // N: point id -> cell index
    DBuf<uint32_t> posOf;// N: point id -> sorted position
    DBuf<uint32_t> J;    // N: join-order position -> point id (cells contiguous, Morton inside)
    DBuf<uint32_t> posJ; // N: point id -> join-order position
    DBuf<float> Xs;      // n x Npad SoA, sorted order, centred floats (SIMT join; lazy)
    bool xs_ready = false;
    bool tc_ready = false;
    uint32_t row_halfs = 0, split = 0;
    DBuf<__half> Bh;     // N x row_halfs: tensor-core B operand (knnj_tc.cu)
    const __half* bh_zero_p = nullptr;  // Bh block whose row padding an earlier build zeroed
    uint32_t bh_zero_halfs = 0;         // ... beyond this many halfs, for rows of this width
    uint64_t bh_zero_rows = 0;          // ... in its first this many rows
    DBuf<float> bbox;    // 2n x ceil(N/FB): FP32 boxes (outward) of FB-position blocks (J order)
    bool bbox_ready = false;
    DBuf<double> XJ;     // N x n: FP64 rows in join order (finalize gathers; lazy)
    bool xj_ready = false;
};

// Work description of one join pass (queries of one level grid).
struct Pass {
    uint64_t nq = 0;
    uint64_t nitems = 0;
    uint64_t nadj = 0;
    uint64_t candidates = 0;  // sum over queries of candidate-set size
    uint64_t candidates_dense = 0;  // the same over dense queries (when flags were given)
    uint64_t screened = 0;    // candidate pairs left after the box filter (join work)
    uint64_t row_begin = 0;   // first owned position in the cell-ordered query list (shards)
    uint64_t nq_all = 0;      // queries before sharding
    uint32_t chunk = 128;     // queries per work item
    DBuf<uint32_t> qpos;      // nq: sorted positions of the queries (grouped by cell)
    DBuf<uint32_t> qrow;      // nq: output row of each query
    DBuf<uint4> items;        // nitems: qbeg, qend, abeg, aend
    DBuf<uint2> adj;          // nadj: candidate position ranges
    // Items too large for the schedule are split into candidate-range parts. Parts run
    // on virtual launch rows [nq, nv) (qpos copied from their real row, vsrc[v - nq]);
    // splits[i] = (first real row, queries, parts, first virtual row - nq).
    uint64_t nv = 0, nsplits = 0;
    DBuf<uint32_t> vsrc;
    DBuf<uint4> splits;
    // Launch chunks (passes built with stream_chunks > 1 and no split items): chunk c is
    // items [chunk_item[c], chunk_item[c+1]) over the contiguous launch rows
    // [chunk_row[c], chunk_row[c+1]); items are LPT-ordered inside each chunk. Empty: one
    // launch over everything.
    std::vector<uint64_t> chunk_item, chunk_row;
    // mixed pass (knnj_capi.cu pass_mixed): items on the tensor cores where their own data
    // radius (item_r2, absolute units, from the box filter) allows, the rest SIMT
    bool mixed = false, has_r2 = false;
    DBuf<float> item_r2;
};

struct JoinArgs {
    const float* Xs;
    uint64_t Npad;
    uint32_t n;
    const uint32_t* qpos;
    const uint4* items;
    const uint2* adj;
    const float* init_cut;   // per launch row, may be null
    uint32_t K, L;
    uint32_t* out_cnt;       // per launch row
    uint32_t* out_pos;       // per launch row * L
    float gam;               // 2.02 * gamma_{n+2} (float32 unit roundoff)
    float erg;               // 2*u1*Rg: input-rounding part of E
    float eab;               // u(1+2u): (A+B) coefficient of E
    float e64;               // (n+3) * 2^-52: FP64 accumulation slack
};

struct TcJoinArgs {
    const __half* Bh;        // level's B operand rows (sorted order)
    uint32_t row_halfs, n;
    uint32_t ksteps;         // K=16 UMMA steps holding the 3n+2 non-zero columns
    const uint32_t* qpos;
    const uint4* items;
    const uint2* adj;
    const float* init_cut;   // per launch row (scaled units), may be null
    uint32_t K, L;
    uint32_t* out_cnt;       // per launch row
    uint32_t* out_pos;       // per launch row * L
    float delta;             // |key - sq64/S^2| bound (scaled units)
    const float* item_delta; // optional per work item bound (radius of the item's own data)
    float* dbg;              // test hook: block 0 dumps its first accumulator tile [128][128]
    unsigned long long* stats;  // dev hook (KNNJ_JOIN_STATS): slabs, rare slabs, bits, inserts, compactions
    // histogram epilogue (HIST kernels only)
    uint32_t n_bins;
    uint32_t n_count;        // bins [0, n_count) are counted (n_count < n_bins: capped histogram)
    const float* tables;     // LO[n_bins+1], HI[n_bins+1] in scaled units
    float inv_width_scaled;  // S / bin_width
    const double* X64;
    const uint32_t* A;       // HIST: candidate/query position -> point id (null: identity)
    double eps_mean, limit_sq, inv_width;
    unsigned long long* counts;
};

struct FinalArgs {
    const double* X64;
    uint32_t n;
    const uint32_t* A;       // sorted pos -> pid (level)
    const uint32_t* qpos;
    const uint32_t* qrow;
    const uint32_t* cnt;
    const uint32_t* pos;     // launch row * L
    uint64_t nrows;
    uint32_t K, L;
    double eps2;             // dense rule threshold (level 0) or -1
    double cover2;           // certification: kth < cover2 (already scaled by 1-eta); inf = all
    uint32_t* out_ids;       // [qrow * K]
    double* out_dist;
    double* out_kth;         // [qrow]
    uint8_t* out_status;     // [qrow]
    double* out_sq;          // optional [qrow * K]: exact sq (split-part rows, for the merge)
    uint32_t* out_count;     // optional [qrow]: entries written (min(candidates, K))
    const double* XJ;        // optional: X64 rows in A order (row p = point A[p]); locality
    double bound2;           // > 0: radius-bounded pass (every candidate with sq <= bound2 was
                             // screened); rows whose K-th is not within it get ST_MISS only
};

struct HistArgs {
    const float* Xf;         // n x Npad SoA, id order
    uint64_t Npad, N;
    uint32_t n;
    const double* X64;
    const uint32_t* q;       // query ids
    uint64_t nq;
    uint64_t cand_begin_stride;  // candidate slab length
    uint32_t n_bins;
    uint32_t n_count;        // bins [0, n_count) are counted; pairs beyond bin n_count's edge skipped
    const float* SU;         // n_bins+1: lower edge rounded up   (SU[0] = -inf)
    const float* SD;         // n_bins+1: lower edge rounded down (SD[n_bins] = end)
    double eps_mean, limit_sq, inv_width;
    unsigned long long* counts;  // n_bins (u64)
    float gam, erg, eab, e64;
};

// Capped histogram over a grid whose cell width covers the counted radius
// (k_hist_grid, knnj_kernels.cu): queries by their sorted position in that grid.
struct HistGridArgs {
    const float* Xs;         // n x Npad SoA, the grid's sorted order, centred
    uint64_t Npad;
    const double* X64;       // working FP64 rows, id order
    const uint32_t* A;       // sorted position -> point id
    const uint32_t* slot;    // point id -> cell index
    const uint64_t* B;       // ncells sorted linear ids
    const uint2* G;          // ncells position ranges
    uint64_t ncells;
    const uint64_t* cpd;     // m
    const uint64_t* strides; // m
    uint32_t n, m;
    const uint32_t* qpos;    // nq sorted query positions
    uint64_t nq;
    uint32_t n_bins, n_count;
    const float* SU;
    const float* SD;
    double eps_mean, limit_sq, inv_width;
    unsigned long long* counts;
    float gam, erg, eab, e64;
    // candidate-slice grids (a shard's points only): queries are point ids (qids), their
    // cell from the coordinates with the grid's mins / width, FP32 coords from Xf (id order)
    const uint32_t* qids;    // non-null selects this mode (qpos unused)
    const float* Xf;
    const double* mins;      // m
    double w;
};
void launch_hist_grid(const HistGridArgs& a, cudaStream_t s);

// ---------------------------------------------------------------- launchers
extern std::atomic<unsigned long long> g_launches;  // our kernels launched so far
double measure_ffma_tflops(cudaStream_t s);
void launch_morton_keys(const double* X64, const uint32_t* A, const uint32_t* slot, uint64_t N,
                        uint32_t n, uint32_t dims, const double* lo, const double* inv_range,
                        uint64_t* keys, uint32_t* vals, cudaStream_t s,
                        uint32_t bits = 3);
void launch_inverse(const uint32_t* J, uint64_t N, uint32_t* posJ, cudaStream_t s);
// tensor-core kernel shape: KB 128-byte k-blocks per operand row (row_halfs = 64*KB),
// G groups of 128 queries per CTA, STAGES candidate tiles in flight
struct TcShape {
    int KB, G, STAGES;
    int TN = 128; // candidates per tile (64: wide operands, KB >= 3)
};
size_t tc_smem_bytes(const TcShape& sh, uint32_t L, uint32_t n_bins, bool hist);
void launch_hist_tc(const TcJoinArgs& a, const TcShape& sh, uint64_t nitems, uint64_t N,
                    cudaStream_t s);
void launch_prep_tc(const double* X64, const uint32_t* A, uint64_t N, uint32_t n, const double* g,
                    double inv_S, uint32_t row_halfs, __half* Bh, cudaStream_t s,
                    uint32_t write_halfs = 0);
void launch_join_tc(const TcJoinArgs& a, const TcShape& sh, uint64_t nitems, uint64_t N,
                    cudaStream_t s);
void launch_scale_f32(const float* in, uint64_t n, float scale, float* out, cudaStream_t s);
int pick_np(uint32_t n);  // padded dimension count used by the templated kernels
size_t join_smem_bytes(int np, uint32_t L, uint32_t qb);
void launch_join(const JoinArgs& a, uint64_t nitems, uint32_t qb, cudaStream_t s);
void launch_finalize(const FinalArgs& a, cudaStream_t s, uint32_t max_blocks = 0);
size_t hist_smem_bytes(int np, uint32_t n_bins);
void launch_histogram(const HistArgs& a, uint64_t n_slabs, cudaStream_t s);

void launch_check_finite(const double* X, uint64_t count, unsigned long long* first_bad,
                         cudaStream_t s);
void launch_col_sums(const double* X, uint64_t N, uint32_t n, const double* mean,
                     double* partial, uint32_t nblk, cudaStream_t s);
void launch_permute_cols(const double* X0, double* X, uint64_t N, uint32_t n,
                         const uint32_t* order, cudaStream_t s);
void launch_to_float_soa(const double* X, uint64_t N, uint32_t n, const double* g, float* Xf,
                         uint64_t Npad, unsigned long long* rmax_bits, cudaStream_t s);
void launch_pair_sq(const double* X, uint32_t n, const uint64_t* ij, uint64_t npairs,
                    double limit, double* out, cudaStream_t s);
void launch_minmax(const double* X, uint64_t N, uint32_t n, uint32_t m,
                   unsigned long long* mn, unsigned long long* mx, cudaStream_t s);
void launch_cell_keys(const double* X, uint64_t N, uint32_t n, uint32_t m, const double* mins,
                      double w, const uint64_t* cpd, const uint64_t* strides, uint64_t* keys,
                      uint32_t* vals, cudaStream_t s, uint32_t base = 0);
void launch_iota(uint32_t* v, uint64_t N, cudaStream_t s);
void launch_head_flags(const uint64_t* keys, uint64_t N, uint32_t* flags, cudaStream_t s);
void launch_grid_tables(const uint64_t* skeys, const uint32_t* A, const uint32_t* runidx,
                        uint64_t N, uint64_t* B, uint2* G, uint32_t* slot, uint32_t* posOf,
                        cudaStream_t s);
void launch_gather_x64(const double* X, const double* g, const uint32_t* A, uint64_t N, uint32_t n,
                       uint64_t Npad, float* Xs, cudaStream_t s);
void launch_map_u32(const uint32_t* idx, const uint32_t* table, uint64_t n, uint32_t* out,
                    cudaStream_t s);
void launch_adj_count(const uint64_t* B, uint64_t ncells, const uint32_t* cells, uint64_t nc,
                      uint32_t m, const uint64_t* cpd, const uint64_t* strides,
                      uint32_t* counts, cudaStream_t s, const uint32_t* spans = nullptr,
                      const uint2* G = nullptr, unsigned long long* csize = nullptr);
void launch_adj_fill(const uint64_t* B, const uint2* G, uint64_t ncells, const uint32_t* cells,
                     uint64_t nc, uint32_t m, const uint64_t* cpd, const uint64_t* strides,
                     const uint32_t* offs, uint2* adj, unsigned long long* csize,
                     cudaStream_t s, const uint32_t* spans = nullptr,
                     const uint16_t* order = nullptr);
void launch_items(const uint32_t* ufirst, const uint32_t* ucnt, const uint32_t* item_off,
                  const uint32_t* adj_off, uint64_t nuc, const unsigned long long* csize,
                  uint4* items, unsigned long long* work, uint32_t chunk, cudaStream_t s);
void launch_cell_pop(const uint32_t* pids, uint64_t nq, const uint32_t* slot, const uint2* G,
                     uint32_t* pop, cudaStream_t s);
void launch_fill_f32(float* p, uint64_t n, float v, cudaStream_t s);
void launch_range_count(const double* X64, uint32_t n, const uint32_t* A, const uint32_t* qpos,
                        const uint4* items, uint64_t nitems, const uint2* adj, double eps2,
                        unsigned long long* in_eps, cudaStream_t s);
void launch_row_item(const uint4* items, uint64_t nitems, uint32_t* row_item, cudaStream_t s);
void launch_gather_u8(const uint32_t* idx, const uint8_t* table, uint64_t n, uint8_t* out,
                      cudaStream_t s);
void launch_gather_f64(const uint32_t* idx, const double* table, uint64_t n, double* out,
                       cudaStream_t s);
void launch_gather_f32(const uint32_t* idx, const float* table, uint64_t n, float* out,
                       cudaStream_t s);
void launch_slow_exact(const double* X64, uint32_t n, const uint32_t* A, const uint32_t* qpos,
                       const uint32_t* qrow, const uint32_t* rows, uint64_t nrows,
                       const uint4* items, const uint32_t* row_item, const uint2* adj,
                       uint32_t K, double eps2, double cover2, uint32_t* out_ids,
                       double* out_dist, double* out_kth, uint8_t* out_status, double* out_sq,
                       uint32_t* out_count, cudaStream_t s);
void launch_scatter_f32(const uint32_t* idx, const float* vals, uint64_t n, float* out,
                        cudaStream_t s);
void launch_block_boxes(const double* X64, const uint32_t* J, uint64_t N, uint32_t n, float* box,
                        cudaStream_t s);
void launch_item_boxes(const uint4* items, uint64_t nitems, const uint32_t* qpos, const uint32_t* J,
                       const double* X64, uint32_t n, float* qbox, cudaStream_t s);
void launch_filter_ranges(uint4* items, uint64_t nitems, const float* qbox, uint32_t n,
                          const uint2* adj, const float* box, uint64_t nblk, float r2,
                          uint32_t* out_cnt, const uint32_t* out_off, uint2* out_adj,
                          unsigned long long* screened, bool fill, cudaStream_t s,
                          float* out_key = nullptr, unsigned long long* count_total = nullptr,
                          const float* gbox = nullptr, float* item_r2 = nullptr,
                          uint32_t r_m = 0, float r_2w = 0.f, const float* dbox = nullptr,
                          const float* item_rad2 = nullptr);
void launch_fill_u32(uint32_t* p, uint64_t n, uint32_t v, cudaStream_t s);
void launch_merge_parts(const uint4* splits, uint64_t nsplits, uint32_t K, const uint32_t* t_ids,
                        const double* t_sq, const uint32_t* t_count, const uint32_t* qrow,
                        double eps2, double cover2, uint32_t* out_ids, double* out_dist,
                        double* out_kth, uint8_t* out_status, cudaStream_t s);

void launch_split_flags(const uint32_t* pids, uint64_t nq, const uint32_t* slot, const uint2* G,
                        double n_thresh, uint8_t* dense, unsigned long long* n_sparse,
                        cudaStream_t s);
void launch_rows_by(const double* X64, const uint32_t* A, uint64_t N, uint32_t n, double* out,
                    cudaStream_t s);
// per work item: tensor-core screen bound delta(R) = (A R^2 + B R + C)(1 + 1e-6), rounded up,
// from the item's squared data radius r2 (absolute units; scaled by inv_s2 = 1/S^2), and an
// eligibility flag: 2 delta <= lim (the precision rule) and at least min_q queries
void launch_item_delta(const uint4* items, const float* r2, uint64_t nitems, double inv_s2,
                       double A, double B, double C, double lim, uint32_t min_q, float* delta,
                       uint8_t* tc_ok, cudaStream_t s);
void launch_item_max_cut(const uint4* items, uint64_t nitems, const uint32_t* qrow, uint64_t nq,
                         const uint32_t* vsrc, const float* cut_by_row, float* out, cudaStream_t s);
void launch_row_walk(const uint32_t* ufirst, const uint32_t* ucnt, uint64_t nuc,
                     const unsigned long long* csize, unsigned long long* rowwalk, cudaStream_t s);
void launch_walk_sum(const unsigned long long* rowwalk, const uint32_t* qrow, uint64_t n,
                     const uint8_t* dense, unsigned long long* out, cudaStream_t s);
void launch_id_cell_keys(const double* X, const uint32_t* ids, uint64_t cnt, uint32_t n, uint32_t m,
                         const double* mins, double w, const uint64_t* cpd, const uint64_t* strides,
                         uint64_t* keys, cudaStream_t s);
void launch_range_len(const uint2* r, uint64_t n, uint32_t* out, cudaStream_t s);  // out = y - x
void launch_miss_flags(const uint32_t* rows, uint64_t n, const uint8_t* st, uint8_t* flags,
                       cudaStream_t s);
void launch_uncert_flags(const uint32_t* rows, uint64_t n, const uint8_t* st, uint8_t* flags,
                         cudaStream_t s);
void launch_classify(const uint32_t* rows, uint64_t n, const uint8_t* st, const uint8_t* dense,
                     uint8_t* prov, uint8_t* need, cudaStream_t s);
void launch_dense_cand(const uint4* items, const unsigned long long* work, uint64_t nitems,
                       const uint32_t* qrow, const uint8_t* dense, unsigned long long* out,
                       cudaStream_t s);
void launch_find_ovf(const uint32_t* cnt, uint64_t n, uint32_t* rows, unsigned long long* count,
                     cudaStream_t s);
void launch_gather_rows(const uint32_t* rows, uint64_t n, uint32_t K, const uint32_t* ids,
                        const double* dist, uint32_t* oids, double* odist, cudaStream_t s);
void launch_rows_to_host(const uint32_t* rows, uint64_t n, uint32_t K, const uint32_t* ids,
                         const double* dist, uint32_t* hids, double* hdist, uint32_t max_blocks,
                         cudaStream_t s);
void launch_scatter_rows(const uint32_t* rows, uint64_t n, uint32_t K, const uint32_t* ids,
                         const double* dist, uint32_t* oids, double* odist, cudaStream_t s);

}  // namespace kj
