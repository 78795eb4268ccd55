// Host runtime and C ABI of the B200 KNN self-join engine.
//
// Mirrors the reference's phase functions (see include/knnj_c.h for the
// file:line each entry point replaces) and its orchestrator run_hybrid
// (proj/src/orchestrator.cpp:67-250). Host code does only what must stay
// sequential to be bit-identical with the reference (the mt19937_64 sampling
// streams, the sequential eps_mean sum, the O(n_bins) selection arithmetic);
// all per-point and per-pair work runs on the GPU.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <functional>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <memory>
#include <numeric>
#include <random>
#include <string>
#include <thread>
#include <vector>

#include <cub/cub.cuh>
#include <nvtx3/nvToolsExt.h>

#include "knnj_c.h"
#include "knnj_internal.cuh"

using namespace kj;

namespace kj {
// knnj_rng.cpp (host-compiled: its AVX2 clones stay out of nvcc's host pass)
void draw_pairs_fast(uint64_t N, uint64_t pairs, uint64_t seed, uint64_t* ij);
struct SampleWork;
void sample_fast(uint64_t n, uint64_t k, uint64_t seed, uint64_t* out, bool sorted, SampleWork* w);
SampleWork* sample_work_new();
void sample_work_free(SampleWork* w);
cudaStream_t& alloc_stream() {
    static thread_local cudaStream_t s = nullptr;
    return s;
}
BlockCache*& alloc_cache() {
    static thread_local BlockCache* c = nullptr;
    return c;
}
void* BlockCache::get(size_t bytes, size_t& got, cudaStream_t s) {
    // best fit among cached blocks no larger than 2x the request (+1 MiB)
    auto it = free_blocks.lower_bound(bytes);
    if (it != free_blocks.end() && it->first <= 2 * bytes + (1u << 20)) {
        void* p = it->second;
        got = it->first;
        free_blocks.erase(it);
        return p;
    }
    void* p = nullptr;
    got = bytes;
    if (cudaMallocAsync(&p, bytes, s) != cudaSuccess) {
        // out of memory: hand every cached free block back to the driver and retry
        cudaGetLastError();
        cudaStreamSynchronize(s);
        for (auto& fb : free_blocks) {
            cudaFree(fb.second);
            for (auto o = owned.begin(); o != owned.end(); ++o)
                if (o->first == fb.second) {
                    owned.erase(o);
                    break;
                }
        }
        free_blocks.clear();
        KJ_CUDA(cudaMallocAsync(&p, bytes, s));
    }
    owned.emplace_back(p, bytes);
    return p;
}
BlockCache::~BlockCache() {
    for (auto& b : owned) cudaFree(b.first);
}
}  // namespace kj

namespace {

constexpr double kInf = std::numeric_limits<double>::infinity();
constexpr double U64 = 1.1102230246251565e-16;  // 2^-53

// ---------------------------------------------------------------- CUB helpers
struct Scratch {
    DBuf<unsigned char> tmp;
    void* get(size_t bytes) { return tmp.ensure(bytes); }
};

void sort_pairs_u64_u32(Scratch& sc, const uint64_t* kin, uint64_t* kout, const uint32_t* vin,
                        uint32_t* vout, uint64_t n, int end_bit, cudaStream_t s) {
    size_t bytes = 0;
    KJ_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, bytes, kin, kout, vin, vout, (int64_t)n, 0,
                                            end_bit, s));
    KJ_CUDA(cub::DeviceRadixSort::SortPairs(sc.get(bytes), bytes, kin, kout, vin, vout,
                                            (int64_t)n, 0, end_bit, s));
}
void sort_pairs_u32_u32(Scratch& sc, const uint32_t* kin, uint32_t* kout, const uint32_t* vin,
                        uint32_t* vout, uint64_t n, int end_bit, cudaStream_t s) {
    size_t bytes = 0;
    KJ_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, bytes, kin, kout, vin, vout, (int64_t)n, 0,
                                            end_bit, s));
    KJ_CUDA(cub::DeviceRadixSort::SortPairs(sc.get(bytes), bytes, kin, kout, vin, vout,
                                            (int64_t)n, 0, end_bit, s));
}
template <class T>
void inclusive_sum(Scratch& sc, const T* in, T* out, uint64_t n, cudaStream_t s) {
    size_t bytes = 0;
    KJ_CUDA(cub::DeviceScan::InclusiveSum(nullptr, bytes, in, out, (int64_t)n, s));
    KJ_CUDA(cub::DeviceScan::InclusiveSum(sc.get(bytes), bytes, in, out, (int64_t)n, s));
}
template <class T>
void exclusive_sum(Scratch& sc, const T* in, T* out, uint64_t n, cudaStream_t s) {
    size_t bytes = 0;
    KJ_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, bytes, in, out, (int64_t)n, s));
    KJ_CUDA(cub::DeviceScan::ExclusiveSum(sc.get(bytes), bytes, in, out, (int64_t)n, s));
}
// run-length encode: unique, counts, number of runs (device)
void rle(Scratch& sc, const uint32_t* in, uint32_t* uniq, uint32_t* counts, uint64_t* nruns,
         uint64_t n, cudaStream_t s) {
    size_t bytes = 0;
    KJ_CUDA(cub::DeviceRunLengthEncode::Encode(nullptr, bytes, in, uniq, counts, nruns,
                                               (int64_t)n, s));
    KJ_CUDA(cub::DeviceRunLengthEncode::Encode(sc.get(bytes), bytes, in, uniq, counts, nruns,
                                               (int64_t)n, s));
}
template <class T>
void reduce_sum(Scratch& sc, const T* in, T* out, uint64_t n, cudaStream_t s) {
    size_t bytes = 0;
    KJ_CUDA(cub::DeviceReduce::Sum(nullptr, bytes, in, out, (int64_t)n, s));
    KJ_CUDA(cub::DeviceReduce::Sum(sc.get(bytes), bytes, in, out, (int64_t)n, s));
}

// Contiguous run [first, last) of n items owned by shard `sh` of `ns`: item i goes to
// the shard whose equal-cost slice of the prefix sum contains i's cost midpoint.
void shard_range(const double* cost, uint64_t n, uint32_t sh, uint32_t ns, uint64_t* first,
                 uint64_t* last) {
    std::vector<double> pre(n + 1, 0.0);
    for (uint64_t i = 0; i < n; ++i) pre[i + 1] = pre[i] + cost[i];
    const double W = pre[n];
    auto cut = [&](uint32_t k) -> uint64_t {
        if (k == 0) return 0;
        if (k >= ns) return n;
        const double at = W * double(k) / double(ns);
        uint64_t lo = 0, hi = n;
        while (lo < hi) {
            const uint64_t mid = (lo + hi) / 2;
            if (0.5 * (pre[mid] + pre[mid + 1]) < at) lo = mid + 1;
            else hi = mid;
        }
        return lo;
    };
    *first = cut(sh);
    *last = cut(sh + 1);
}

int bits_for(uint64_t maxval) {
    int b = 0;
    while (b < 64 && (maxval >> b) != 0) ++b;
    return std::max(b, 1);
}

float f32_round_up(double v) {
    float f = (float)v;
    if ((double)f < v) f = std::nextafter(f, std::numeric_limits<float>::infinity());
    return f;
}
float f32_round_down(double v) {
    float f = (float)v;
    if ((double)f > v) f = std::nextafter(f, -std::numeric_limits<float>::infinity());
    return f;
}

// sample_without_replacement(n, k, std::mt19937_64(seed)) with the reference's exact
// output (proj/include/knnjoin/util.hpp:70-92): knnj_rng.cpp (tests/test_rng.py).
std::vector<uint64_t> sample_seeded(uint64_t n, uint64_t k, uint64_t seed, bool sorted = true,
                                    SampleWork* w = nullptr) {
    std::vector<uint64_t> out(std::min(n, k));
    sample_fast(n, k, seed, out.data(), sorted, w);
    return out;
}

uint64_t splitmix64(uint64_t x) {
    x += 0x9e3779b97f4a7c15ull;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
    return x ^ (x >> 31);
}
uint64_t derive_seed(uint64_t master, uint64_t tag) { return splitmix64(master ^ splitmix64(tag)); }

// NVTX range over one phase of a run (visible in nsys / ncu --nvtx timelines)
struct Nvtx {
    explicit Nvtx(const char* name) { nvtxRangePushA(name); }
    ~Nvtx() { nvtxRangePop(); }
    Nvtx(const Nvtx&) = delete;
    Nvtx& operator=(const Nvtx&) = delete;
};

// KNNJ_TRACE=1: host wall-clock marks of the runtime's sub-steps on stderr (dev aid)
struct Trace {
    bool on = false;
    std::chrono::steady_clock::time_point last = std::chrono::steady_clock::now();
    Trace() {
        const char* e = std::getenv("KNNJ_TRACE");
        on = e && e[0] && e[0] != '0';
    }
    void mark(const char* what, cudaStream_t s = nullptr) {
        if (!on) return;
        if (s) cudaStreamSynchronize(s);
        const auto now = std::chrono::steady_clock::now();
        std::fprintf(stderr, "[knnj] %-28s %9.3f ms\n", what,
                     std::chrono::duration<double, std::milli>(now - last).count());
        last = now;
    }
};
Trace& trace() {
    static Trace t;
    return t;
}

// work items of at most 32 queries (the SIMT join's 32-thread blocks)
struct SmallItem {
    __device__ bool operator()(const uint4& it) const { return it.y - it.x <= 32u; }
};

// Device address of a host range in pinned (page-locked, mapped) memory, else null:
// kernels may then store straight into it over PCIe.
void* mapped_host(void* p, size_t bytes) {
    if (!p || !bytes) return nullptr;
    cudaPointerAttributes a{}, b{};
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess ||
        cudaPointerGetAttributes(&b, static_cast<char*>(p) + bytes - 1) != cudaSuccess) {
        cudaGetLastError();
        return nullptr;
    }
    if (a.type != cudaMemoryTypeHost || b.type != cudaMemoryTypeHost || !a.devicePointer ||
        static_cast<char*>(b.devicePointer) - static_cast<char*>(a.devicePointer) != (ptrdiff_t)(bytes - 1))
        return nullptr;
    return a.devicePointer;
}

struct Timer {
    cudaEvent_t a, b;
    cudaStream_t s;
    explicit Timer(cudaStream_t st) : s(st) {
        KJ_CUDA(cudaEventCreate(&a));
        KJ_CUDA(cudaEventCreate(&b));
        KJ_CUDA(cudaEventRecord(a, s));
    }
    ~Timer() {
        cudaEventDestroy(a);
        cudaEventDestroy(b);
    }
    double ms() {
        KJ_CUDA(cudaEventRecord(b, s));
        KJ_CUDA(cudaEventSynchronize(b));
        float f = 0;
        KJ_CUDA(cudaEventElapsedTime(&f, a, b));
        return f;
    }
};

}  // namespace

// ============================================================================ context
struct knnj_ctx {
    int dev = 0;
    cudaStream_t s = nullptr;
    BlockCache cache;  // declared first: destroyed after every DBuf member returned its block
    std::string err;
    Scratch sc;

    uint64_t N = 0;
    uint32_t n = 0;
    uint64_t Npad = 0;
    bool have_points = false, working_ready = false;
    std::vector<uint32_t> perm;
    std::vector<double> var;  // original-column variances
    std::vector<double> g;    // working-column means (float centre)
    double Rg = 0.0;          // max ||x - g||

    DBuf<double> X0, X64;
    DBuf<float> Xf;           // SoA id order
    DBuf<double> d_g;

    Level levels[44];  // 0..39: eps * 2^L; 40..43: the fine cascade (eps * fine_f[i])
    double eps0 = 0.0;
    uint32_t m0 = 0;

    // large per-run buffers kept across calls (grow only): no allocator churn in steady state
    DBuf<uint32_t> pass_cnt, pass_pos;                   // join lists (run_pass)
    DBuf<uint64_t> gk_keys, gk_skeys;                    // grid build sort scratch
    DBuf<uint32_t> gk_vals, gk_runidx;
    DBuf<uint32_t> r_ids, r_q, r_rows;                   // run outputs / query lists (run_impl)
    DBuf<double> r_dist, r_kth;
    DBuf<uint8_t> r_st, r_prov;
    // small device scratch
    DBuf<unsigned long long> d_u64a, d_u64b;
    DBuf<double> d_part;

    DBuf<float> d_gbox;            // g rounded down [n], then up [n]
    cudaStream_t s_out = nullptr;  // result D2H overlapping the fallback (knnj_run)
    cudaEvent_t ev_copy = nullptr; // a streamed row copy on s_out still pending (copy_pending)
    bool copy_pending = false;
    DBuf<uint32_t> st_keys;        // its sorted rows and sort scratch
    DBuf<unsigned char> st_tmp;
    cudaEvent_t ev_out = nullptr;
    ~knnj_ctx() {
        if (sample_work) sample_work_free(sample_work);
        if (s_out) cudaStreamSynchronize(s_out);
        if (ev_copy) cudaEventDestroy(ev_copy);
        if (ev_out) cudaEventDestroy(ev_out);
        if (s_out) cudaStreamDestroy(s_out);
        if (h_sq) cudaFreeHost(h_sq);
        if (h_ij) cudaFreeHost(h_ij);
        if (s) cudaStreamDestroy(s);
    }

    void sync() { KJ_CUDA(cudaStreamSynchronize(s)); }
    // the result stream runs at the highest priority: its finalize / copy blocks are
    // dispatched ahead of the running join's next CTAs and then co-reside with them
    bool out_priority = true;
    void ensure_out_stream() {
        if (!s_out) {
            int lo = 0, hi = 0;
            KJ_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
            KJ_CUDA(cudaStreamCreateWithPriority(&s_out, cudaStreamNonBlocking, out_priority ? hi : lo));
            KJ_CUDA(cudaEventCreateWithFlags(&ev_out, cudaEventDisableTiming));
        }
    }

    // ------------------------------------------------------------ screen constants
    void screen_consts(float& gam, float& erg, float& eab, float& e64) const {
        const double u = 5.9604644775390625e-08;  // 2^-24
        const double gamma = (n + 2) * u / (1.0 - (n + 2) * u);
        gam = (float)(2.02 * gamma * 1.01);
        const double u1 = u * (1.0 + 1e-6);
        erg = (float)(2.0 * u1 * Rg * 1.01 + 1e-30);
        eab = (float)(u * (1.0 + 2.0 * u) * 1.01);
        e64 = (float)((n + 4) * 2.0 * U64 * 1.01);
    }

    // ------------------------------------------------------------ working set
    // Working coordinates from a column order; builds the FP32 SoA copy
    // centred at the working-column means.
    void make_working(const std::vector<uint32_t>& order, const std::vector<double>& mean0) {
        X64.ensure(N * n);
        DBuf<uint32_t> d_ord;
        d_ord.ensure(n);
        KJ_CUDA(cudaMemcpyAsync(d_ord.p, order.data(), n * 4, cudaMemcpyHostToDevice, s));
        launch_permute_cols(X0.p, X64.p, N, n, d_ord.p, s);
        g.resize(n);
        for (uint32_t j = 0; j < n; ++j) g[j] = mean0[order[j]];
        d_g.ensure(n);
        KJ_CUDA(cudaMemcpyAsync(d_g.p, g.data(), n * 8, cudaMemcpyHostToDevice, s));
        {  // the centre rounded outward to FP32 (per-item screen radii, filter_items)
            std::vector<float> gb(2 * n);
            for (uint32_t j = 0; j < n; ++j) {
                gb[j] = f32_round_down(g[j]);
                gb[n + j] = f32_round_up(g[j]);
            }
            d_gbox.ensure(2 * n);
            KJ_CUDA(cudaMemcpyAsync(d_gbox.p, gb.data(), 8 * n, cudaMemcpyHostToDevice, s));
            sync();
        }
        Npad = ((N + 127) / 128) * 128 + 128;
        Xf.ensure((uint64_t)n * Npad);
        d_u64a.ensure(1);
        KJ_CUDA(cudaMemsetAsync(d_u64a.p, 0, 8, s));
        launch_to_float_soa(X64.p, N, n, d_g.p, Xf.p, Npad, d_u64a.p, s);
        unsigned long long bits = 0;
        KJ_CUDA(cudaMemcpyAsync(&bits, d_u64a.p, 8, cudaMemcpyDeviceToHost, s));
        sync();
        double r2;
        std::memcpy(&r2, &bits, 8);
        Rg = std::sqrt(r2) * (1.0 + 1e-12);
        perm = order;
        working_ready = true;
        bh_id_ready = false;  // FP16 operands derive from the working coordinates
        hist_order_ready = false;
        mm_lo.clear();
        for (auto& lv : levels) lv.built = false;
        hist_lv.built = false;
    }

    // column means (and variances when want_var) of X0, deterministic on device
    void column_stats(std::vector<double>& mean, std::vector<double>* varp) {
        const uint32_t nblk = (uint32_t)std::min<uint64_t>(1024, std::max<uint64_t>(1, N / 64));
        d_part.ensure((uint64_t)nblk * n);
        std::vector<double> part((uint64_t)nblk * n);
        launch_col_sums(X0.p, N, n, nullptr, d_part.p, nblk, s);
        KJ_CUDA(cudaMemcpyAsync(part.data(), d_part.p, part.size() * 8, cudaMemcpyDeviceToHost, s));
        sync();
        mean.assign(n, 0.0);
        for (uint32_t b = 0; b < nblk; ++b)
            for (uint32_t j = 0; j < n; ++j) mean[j] += part[(uint64_t)b * n + j];
        for (uint32_t j = 0; j < n; ++j) mean[j] /= double(N);
        if (!varp) return;
        DBuf<double> d_mean;
        d_mean.ensure(n);
        KJ_CUDA(cudaMemcpyAsync(d_mean.p, mean.data(), n * 8, cudaMemcpyHostToDevice, s));
        launch_col_sums(X0.p, N, n, d_mean.p, d_part.p, nblk, s);
        KJ_CUDA(cudaMemcpyAsync(part.data(), d_part.p, part.size() * 8, cudaMemcpyDeviceToHost, s));
        sync();
        varp->assign(n, 0.0);
        for (uint32_t b = 0; b < nblk; ++b)
            for (uint32_t j = 0; j < n; ++j) (*varp)[j] += part[(uint64_t)b * n + j];
        for (uint32_t j = 0; j < n; ++j) (*varp)[j] /= double(N);
    }

    // Exact reference arithmetic for selected columns (dataset.cpp:58-74): used only
    // when two device variances are too close to order safely.
    void exact_column_variance(const std::vector<uint32_t>& cols, std::vector<double>& var_out) {
        std::vector<double> col(N);
        for (uint32_t j : cols) {
            KJ_CUDA(cudaMemcpy2DAsync(col.data(), 8, X0.p + j, (size_t)n * 8, 8, N,
                                      cudaMemcpyDeviceToHost, s));
            sync();
            double mean = 0.0;
            for (uint64_t i = 0; i < N; ++i) mean += col[i];
            mean /= double(N);
            double v = 0.0;
            for (uint64_t i = 0; i < N; ++i) {
                double d = col[i] - mean;
                v += d * d;
            }
            var_out[j] = v / double(N);
        }
    }

    // ------------------------------------------------------------ reorder
    // reorder_by_variance (dataset.cpp:87-111)
    void reorder(uint32_t m) {
        if (m < 1 || m > n) throw Error(1, "indexed dimension count m must satisfy 1 <= m <= n");
        std::vector<double> mean, v;
        column_stats(mean, &v);
        // guard band: the reference sums sequentially (relative error <= ~N*2^-53);
        // ties or near-ties are re-decided with the reference's own arithmetic.
        const double tau = 8.0 * double(N) * U64 + 1e-12;
        std::vector<uint32_t> order(n);
        std::iota(order.begin(), order.end(), 0u);
        std::sort(order.begin(), order.end(), [&](uint32_t a, uint32_t b) {
            if (v[a] != v[b]) return v[a] > v[b];
            return a < b;
        });
        std::vector<uint32_t> close;
        for (uint32_t i = 0; i + 1 < n; ++i) {
            double a = v[order[i]], b = v[order[i + 1]];
            if (std::fabs(a - b) <= tau * std::max(std::fabs(a), std::fabs(b))) {
                close.push_back(order[i]);
                close.push_back(order[i + 1]);
            }
        }
        if (!close.empty()) {
            std::sort(close.begin(), close.end());
            close.erase(std::unique(close.begin(), close.end()), close.end());
            exact_column_variance(close, v);
            std::sort(order.begin(), order.end(), [&](uint32_t a, uint32_t b) {
                if (v[a] != v[b]) return v[a] > v[b];
                return a < b;
            });
        }
        var = v;
        make_working(order, mean);
    }

    void ensure_working() {
        if (working_ready) return;
        std::vector<double> mean;
        column_stats(mean, nullptr);
        std::vector<uint32_t> id(n);
        std::iota(id.begin(), id.end(), 0u);
        make_working(id, mean);
    }

    // ------------------------------------------------------------ eps_mean
    // estimate_eps_mean (epsilon.cpp:14-44) in two halves: the index pairs are drawn on
    // the host with the reference RNG (draw_pairs, a pure function of |D|, the pair
    // count and the seed, so knnj_run draws them on a host thread while the GPU does the
    // reorder and the histogram's candidate order), then evaluated on the device and
    // summed sequentially in sample order (bit-identical to the reference).
    static std::vector<uint64_t> draw_pairs(uint64_t N, uint64_t sample_pairs, uint64_t seed) {
        const uint64_t all = N * (N - 1);
        std::vector<uint64_t> ij;
        if (sample_pairs >= all) {  // exhaustive sweep
            ij.reserve(2 * all);
            for (uint64_t i = 0; i < N; ++i)
                for (uint64_t j = 0; j < N; ++j)
                    if (i != j) {
                        ij.push_back(i);
                        ij.push_back(j);
                    }
            return ij;
        }
        ij.resize(2 * sample_pairs);
        draw_pairs_into(N, sample_pairs, seed, ij.data());
        return ij;
    }
    // the sampled (non-exhaustive) stream straight into caller memory (e.g. pinned)
    // (block-generated engine: knnj_rng.hpp, the same stream as std::mt19937_64 +
    // std::uniform_int_distribution, 3-5x faster; tests/test_rng.py)
    static void draw_pairs_into(uint64_t N, uint64_t sample_pairs, uint64_t seed, uint64_t* ij) {
        draw_pairs_fast(N, sample_pairs, seed, ij);
    }
    uint64_t* h_ij = nullptr;  // pinned pair indices (knnj_run's eps_mean draw)
    uint64_t h_ij_cap = 0;
    uint64_t* pinned_pairs(uint64_t pairs) {
        if (h_ij_cap < pairs) {
            if (h_ij) cudaFreeHost(h_ij);
            h_ij = nullptr;
            KJ_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&h_ij), 16 * pairs, cudaHostAllocDefault));
            h_ij_cap = pairs;
        }
        return h_ij;
    }
    double* h_sq = nullptr;  // pinned staging for the per-pair distances
    uint64_t h_sq_cap = 0;
    double eps_mean_of(const std::vector<uint64_t>& ij) { return eps_mean_of(ij.data(), ij.size() / 2); }
    double eps_mean_of(const uint64_t* ij, uint64_t used) {
        if (!used) throw Error(1, "sample_pairs must be at least 1");
        if (h_sq_cap < used) {
            if (h_sq) cudaFreeHost(h_sq);
            h_sq = nullptr;
            KJ_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&h_sq), 8 * used, cudaHostAllocDefault));
            h_sq_cap = used;
        }
        DBuf<uint64_t> d_ij;
        DBuf<double> d_out;
        d_ij.ensure(2 * used);
        d_out.ensure(used);
        KJ_CUDA(cudaMemcpyAsync(d_ij.p, ij, 16 * used, cudaMemcpyHostToDevice, s));
        launch_pair_sq(X64.p, n, d_ij.p, used, kInf, d_out.p, s);
        KJ_CUDA(cudaMemcpyAsync(h_sq, d_out.p, 8 * used, cudaMemcpyDeviceToHost, s));
        sync();
        double sum = 0.0;
        for (uint64_t p = 0; p < used; ++p) sum += std::sqrt(h_sq[p]);
        return sum / double(used);
    }
    double eps_mean(uint64_t sample_pairs, uint64_t seed) {
        if (N < 2) throw Error(1, "eps_mean estimation needs at least two points");
        if (sample_pairs < 1) throw Error(1, "sample_pairs must be at least 1");
        return eps_mean_of(draw_pairs(N, sample_pairs, seed));
    }

    std::vector<double> pair_sq(const uint64_t* ij, uint64_t np, double limit) {
        DBuf<uint64_t> d_ij;
        DBuf<double> d_out;
        d_ij.ensure(2 * np);
        d_out.ensure(np);
        KJ_CUDA(cudaMemcpyAsync(d_ij.p, ij, 16 * np, cudaMemcpyHostToDevice, s));
        launch_pair_sq(X64.p, n, d_ij.p, np, limit, d_out.p, s);
        std::vector<double> out(np);
        KJ_CUDA(cudaMemcpyAsync(out.data(), d_out.p, 8 * np, cudaMemcpyDeviceToHost, s));
        sync();
        return out;
    }

    // ------------------------------------------------------------ histogram
    // bin of an exact sq, as epsilon.cpp:86-95 computes it (n_bins = uncounted)
    static uint64_t ref_bin(double sq, double eps_mean, double inv_width, uint32_t nb) {
        if (sq > eps_mean * eps_mean) return nb;
        double dist = std::sqrt(sq);
        if (dist >= eps_mean) return nb;
        uint64_t b = (uint64_t)(dist * inv_width);
        if (b >= nb) b = nb - 1;
        return b;
    }
    // smallest double sq >= 0 whose bin is >= b (monotone in sq)
    static double bin_threshold(uint64_t b, double eps_mean, double inv_width, uint32_t nb) {
        uint64_t lo = 0, hi = 0x7FF0000000000000ull;  // +inf bits
        while (lo < hi) {
            uint64_t mid = lo + (hi - lo) / 2;
            double v;
            std::memcpy(&v, &mid, 8);
            if (ref_bin(v, eps_mean, inv_width, nb) >= b) hi = mid;
            else lo = mid + 1;
        }
        double r;
        std::memcpy(&r, &lo, 8);
        return r;
    }

    double last_hist_kernel_ms = 0.0;
    bool last_hist_tc = false;
    // Counts of the sampled queries qids (this shard's share when sharded: a slice of the
    // queries, or for the grid histogram all queries against a slice of the candidates).
    void histogram_queries(const uint64_t* qids, uint64_t nq, double em, uint32_t nb,
                           uint64_t* raw, uint32_t ncount = 0, uint32_t shard = 0,
                           uint32_t nshard = 1) {
        if (ncount == 0 || ncount > nb) ncount = nb;
        const bool cand_split = nshard > 1 && grid_hist_applies(nq, ncount, nb);
        if (nshard > 1 && !cand_split) {  // this shard's contiguous slice of the queries
            const uint64_t lo = nq * shard / nshard, hi = nq * (shard + 1) / nshard;
            qids += lo;
            nq = hi - lo;
        }
        if (nq == 0) {
            last_hist_kernel_ms = 0.0;
            return;
        }
        if (!(em > 0.0))
            throw Error(4, "mean pairwise distance is not positive; cannot build a distance histogram");
        if (nb < 2) throw Error(1, "histogram needs at least 2 bins");
        const double width = em / double(nb);
        const double inv_width = 1.0 / width;
        std::vector<float> SU(nb + 1), SD(nb + 1);
        std::vector<double> S(nb + 1);
        for (uint32_t b = 1; b <= nb; ++b) S[b] = bin_threshold(b, em, inv_width, nb);
        SU[0] = -std::numeric_limits<float>::infinity();
        for (uint32_t b = 1; b <= nb; ++b) SU[b] = f32_round_up(S[b]);
        for (uint32_t b = 0; b < nb; ++b) SD[b] = f32_round_down(S[b + 1]);
        SD[nb] = SU[nb];
        DBuf<float> d_tab;
        d_tab.ensure(2 * (nb + 1));
        KJ_CUDA(cudaMemcpyAsync(d_tab.p, SU.data(), 4 * (nb + 1), cudaMemcpyHostToDevice, s));
        KJ_CUDA(cudaMemcpyAsync(d_tab.p + nb + 1, SD.data(), 4 * (nb + 1), cudaMemcpyHostToDevice, s));
        std::vector<uint32_t> q32(nq);
        for (uint64_t i = 0; i < nq; ++i) q32[i] = (uint32_t)qids[i];
        DBuf<uint32_t> d_q;
        d_q.ensure(nq);
        KJ_CUDA(cudaMemcpyAsync(d_q.p, q32.data(), 4 * nq, cudaMemcpyHostToDevice, s));
        DBuf<unsigned long long> d_cnt;
        d_cnt.ensure(nb);
        KJ_CUDA(cudaMemsetAsync(d_cnt.p, 0, 8 * nb, s));
        if (nb > 256) throw Error(1, "n_bins above 256 is not supported by the device histogram");

        HistArgs a{};
        a.Xf = Xf.p;
        a.Npad = Npad;
        a.N = N;
        a.n = n;
        a.X64 = X64.p;
        a.q = d_q.p;
        a.nq = nq;
        a.n_bins = nb;
        a.n_count = ncount;
        a.SU = d_tab.p;
        a.SD = d_tab.p + nb + 1;
        a.eps_mean = em;
        a.limit_sq = em * em;
        a.inv_width = inv_width;
        a.counts = d_cnt.p;
        screen_consts(a.gam, a.erg, a.eab, a.e64);
        if (cand_split || grid_hist_applies(nq, ncount, nb)) {
            if (cand_split)
                histogram_grid(d_q.p, nq, a, S[ncount], N * shard / nshard, N * (shard + 1) / nshard);
            else
                histogram_grid(d_q.p, nq, a, S[ncount]);
            last_hist_tc = false;
            std::vector<unsigned long long> c(nb);
            KJ_CUDA(cudaMemcpyAsync(c.data(), d_cnt.p, 8 * nb, cudaMemcpyDeviceToHost, s));
            sync();
            for (uint32_t b = 0; b < nb; ++b) raw[b] += c[b];
            return;
        }
        if (use_tc_hist() && tc_smem_bytes(tc_hist_shape(), 0, nb, true) <= 227 * 1024) {
            histogram_tc(d_q.p, nq, em, nb, ncount, S, d_cnt.p);
            last_hist_tc = true;
            std::vector<unsigned long long> c(nb);
            KJ_CUDA(cudaMemcpyAsync(c.data(), d_cnt.p, 8 * nb, cudaMemcpyDeviceToHost, s));
            sync();
            for (uint32_t b = 0; b < nb; ++b) raw[b] += c[b];
            return;
        }
        const int np = pick_np(n);
        const uint64_t T = np <= 32 ? 128 : 64;
        const uint64_t qblocks = (nq + JB - 1) / JB;
        uint64_t want_blocks = 148 * 16;
        uint64_t slabs = std::max<uint64_t>(1, (want_blocks + qblocks - 1) / qblocks);
        slabs = std::min<uint64_t>(slabs, (N + T - 1) / T);
        slabs = std::min<uint64_t>(slabs, 65535);
        uint64_t stride = (N + slabs - 1) / slabs;
        stride = ((stride + T - 1) / T) * T;
        slabs = (N + stride - 1) / stride;
        a.cand_begin_stride = stride;
        Timer t(s);
        last_hist_tc = false;
        launch_histogram(a, slabs, s);
        std::vector<unsigned long long> c(nb);
        KJ_CUDA(cudaMemcpyAsync(c.data(), d_cnt.p, 8 * nb, cudaMemcpyDeviceToHost, s));
        last_hist_kernel_ms = t.ms();
        for (uint32_t b = 0; b < nb; ++b) raw[b] += c[b];
    }

    // Capped histogram on a grid (k_hist_grid): when only bins [0, n_count) are counted,
    // every counted pair lies within r = sqrt(S[n_count]) in all n dims, so a grid of
    // cell width >= r over the first min(n, 6) dims holds each of them in the query's
    // 3^m neighbourhood. For small n that neighbourhood is a tight superset of the
    // counted ball: C5's capped phase screens ~7e3 candidates per sampled query instead
    // of the ~2.5e6 the box-filtered all-points sweep leaves. The grid (cells sorted by
    // linear id, points by id inside a cell) is rebuilt per call: its width depends on
    // the cap the pilot placed.
    int hist_grid = 1;  // 0 never, 1 when it pays (below), 2 always (tests)
    uint64_t hist_grid_min_queries = 65536;  // ... for this many queries
    uint64_t hist_grid_min_points = 1u << 20;  // ... or this many points
    bool grid_hist_applies(uint64_t nq, uint32_t ncount, uint32_t nb) const {
        return ncount < nb && hist_grid && n <= 8 &&
               (hist_grid == 2 || nq >= hist_grid_min_queries || N >= hist_grid_min_points);
    }
    Level hist_lv;  // built = its tables match the current working points
    DBuf<float> hist_Xs;
    double last_hist_grid_build_ms = 0.0;
    // [p0, p1): the candidate slice (a shard's ids; default all points). With a slice the
    // grid holds only those points and the queries (any ids) find their cells from their
    // coordinates; the per-shard counts sum to the full histogram (counts are additive
    // over candidate partitions), so every shard bins all sampled queries against 1/S of
    // the points instead of 1/S of the queries against a replicated all-points grid.
    uint64_t hist_p0 = 0, hist_p1 = 0;
    DBuf<double> hist_mins;
    void histogram_grid(const uint32_t* d_q, uint64_t nq, const HistArgs& h, double r2,
                        uint64_t p0 = 0, uint64_t p1 = ~0ull) {
        const uint32_t m = std::min<uint32_t>(n, 6);
        const double w = std::sqrt(r2) * (1.0 + 1e-9);
        p1 = std::min<uint64_t>(p1, N);
        // queries go by id (their cell from the coordinates): the grid then needs no
        // point -> cell / position tables (two scattered N-element writes per build)
        Timer tb(s);
        // a grid built for a slightly larger radius (the pilot's) serves this one too
        if (!(hist_lv.built && hist_lv.m == m && hist_lv.w >= w && hist_lv.w <= 1.2 * w &&
              hist_p0 == p0 && hist_p1 == p1)) {
            grid_tables_into(hist_lv, m, w, p0, p1, false);
            hist_Xs.ensure((uint64_t)n * Npad);
            launch_gather_x64(X64.p, d_g.p, hist_lv.A.p, hist_lv.npts, n, Npad, hist_Xs.p, s);
            hist_mins.ensure(m);
            KJ_CUDA(cudaMemcpyAsync(hist_mins.p, hist_lv.mins.data(), 8 * m, cudaMemcpyHostToDevice, s));
            hist_lv.built = true;
            hist_p0 = p0;
            hist_p1 = p1;
        }
        DBuf<uint64_t> d_cs;
        d_cs.ensure(2 * m);
        KJ_CUDA(cudaMemcpyAsync(d_cs.p, hist_lv.cpd.data(), 8 * m, cudaMemcpyHostToDevice, s));
        KJ_CUDA(cudaMemcpyAsync(d_cs.p + m, hist_lv.strides.data(), 8 * m, cudaMemcpyHostToDevice, s));
        // queries sorted by their cell (neighbouring warps share candidate rows)
        DBuf<uint32_t> qs;
        {
            DBuf<uint64_t> kq, kq2;
            kq.ensure(nq);
            kq2.ensure(nq);
            qs.ensure(nq);
            launch_id_cell_keys(X64.p, d_q, nq, n, m, hist_mins.p, hist_lv.w, d_cs.p, d_cs.p + m, kq.p, s);
            sort_pairs_u64_u32(sc, kq.p, kq2.p, d_q, qs.p, nq, hist_lv.key_bits, s);
        }
        last_hist_grid_build_ms = tb.ms();
        HistGridArgs a{};
        a.Xs = hist_Xs.p;
        a.Npad = Npad;
        a.X64 = X64.p;
        a.A = hist_lv.A.p;
        a.slot = nullptr;
        a.B = hist_lv.B.p;
        a.G = hist_lv.G.p;
        a.ncells = hist_lv.ncells;
        a.cpd = d_cs.p;
        a.strides = d_cs.p + m;
        a.n = n;
        a.m = m;
        a.qpos = nullptr;
        a.nq = nq;
        a.qids = qs.p;
        a.Xf = Xf.p;
        a.mins = hist_mins.p;
        a.w = hist_lv.w;
        a.n_bins = h.n_bins;
        a.n_count = h.n_count;
        a.SU = h.SU;
        a.SD = h.SD;
        a.eps_mean = h.eps_mean;
        a.limit_sq = h.limit_sq;
        a.inv_width = h.inv_width;
        a.counts = h.counts;
        a.gam = h.gam;
        a.erg = h.erg;
        a.eab = h.eab;
        a.e64 = h.e64;
        Timer t(s);
        launch_hist_grid(a, s);
        last_hist_kernel_ms = t.ms();
        if (getenv("KNNJ_JOIN_STATS"))
            fprintf(stderr, "hist grid: queries %llu bins %u/%u cells %llu w %.6g build %.1f ms kernel %.1f ms\n",
                    (unsigned long long)nq, h.n_count, h.n_bins, (unsigned long long)hist_lv.ncells, hist_lv.w,
                    last_hist_grid_build_ms, last_hist_kernel_ms);
    }

    // Tensor-core histogram: sampled queries x all points (id order) on the
    // tcgen05 GEMM-form screen, exact-certain binning (knnj_tc.cu, HIST epilogue).
    DBuf<__half> Bh_id;
    bool bh_id_ready = false;
    uint32_t bh_id_row = 0;
    // The histogram's candidate order: all points in Morton order over the first
    // <= 10 working dims (no grid exists yet), with the tensor-core operand rows and the
    // FP32 block boxes of that order. Sampled queries are sorted into it, so a work item
    // (256 queries) is spatially compact and the box filter can drop candidate blocks
    // beyond the counted radius (eps_mean, or the cap edge when capped).
    DBuf<uint32_t> hJ, hposJ;
    DBuf<float> hbox;
    bool hist_order_ready = false;
    void ensure_hist_order(uint32_t row_halfs) {
        if (hist_order_ready && bh_id_ready && bh_id_row == row_halfs) return;
        const uint32_t md = std::min<uint32_t>(ensure_morton_box(), 21);  // 3 bits per dim in 64
        DBuf<uint32_t> ident, zero, vals;
        DBuf<uint64_t> keys, skeys;
        ident.ensure(N);
        zero.ensure(N);
        vals.ensure(N);
        keys.ensure(N);
        skeys.ensure(N);
        launch_iota(ident.p, N, s);
        KJ_CUDA(cudaMemsetAsync(zero.p, 0, 4 * N, s));
        launch_morton_keys(X64.p, ident.p, zero.p, N, n, md, d_mm.p, d_mm.p + md, keys.p, vals.p, s);
        hJ.ensure(N);
        hposJ.ensure(N);
        sort_pairs_u64_u32(sc, keys.p, skeys.p, vals.p, hJ.p, N, 3 * (int)md, s);
        launch_inverse(hJ.p, N, hposJ.p, s);
        Bh_id.ensure(N * row_halfs);
        launch_prep_tc(X64.p, hJ.p, N, n, d_g.p, 1.0 / tc_S(), row_halfs, Bh_id.p, s);
        const uint64_t nblk = (N + FB - 1) / FB;
        hbox.ensure(nblk * 2 * n);
        launch_block_boxes(X64.p, hJ.p, N, n, hbox.p, s);
        bh_id_ready = true;
        bh_id_row = row_halfs;
        hist_order_ready = true;
    }
    uint64_t last_hist_screened = 0, last_hist_pairs = 0;
    void histogram_tc(const uint32_t* d_q, uint64_t nq, double em, uint32_t nb, uint32_t ncount,
                      const std::vector<double>& S_thr, unsigned long long* d_cnt) {
        const uint32_t row_halfs = tc_row_halfs();
        ensure_hist_order(row_halfs);
        // sampled queries -> sorted positions in the histogram order
        DBuf<uint32_t> qp_u, qp;
        qp_u.ensure(nq);
        qp.ensure(nq);
        launch_map_u32(d_q, hposJ.p, nq, qp_u.p, s);
        {
            size_t bytes = 0;
            KJ_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, bytes, qp_u.p, qp.p, (int64_t)nq, 0,
                                                   bits_for(N), s));
            KJ_CUDA(cub::DeviceRadixSort::SortKeys(sc.get(bytes), bytes, qp_u.p, qp.p, (int64_t)nq, 0,
                                                   bits_for(N), s));
        }
        const double Ssc = tc_S(), S2 = Ssc * Ssc;
        const double width = em / double(nb);
        std::vector<float> tab(2 * (nb + 1));
        tab[0] = -std::numeric_limits<float>::infinity();
        for (uint32_t b = 1; b <= nb; ++b) tab[b] = f32_round_up(S_thr[b] / S2);
        for (uint32_t b = 0; b < nb; ++b) tab[nb + 1 + b] = f32_round_down(S_thr[b + 1] / S2);
        tab[nb + 1 + nb] = tab[nb];
        DBuf<float> d_tab;
        d_tab.ensure(tab.size());
        KJ_CUDA(cudaMemcpyAsync(d_tab.p, tab.data(), 4 * tab.size(), cudaMemcpyHostToDevice, s));
        const TcShape hsh = tc_hist_shape();
        const uint32_t NQ = 128u * hsh.G;
        const uint64_t qblocks = (nq + NQ - 1) / NQ;
        uint64_t slabs = std::max<uint64_t>(1, (148ull * 8 + qblocks - 1) / qblocks);
        uint64_t stride = (N + slabs - 1) / slabs;
        stride = ((stride + 127) / 128) * 128;
        slabs = (N + stride - 1) / stride;
        std::vector<uint4> items;
        items.reserve(qblocks * slabs);
        std::vector<uint2> adj(slabs);
        for (uint64_t sl = 0; sl < slabs; ++sl)
            adj[sl] = make_uint2((uint32_t)(sl * stride), (uint32_t)std::min<uint64_t>(N, (sl + 1) * stride));
        for (uint64_t qb = 0; qb < qblocks; ++qb)
            for (uint64_t sl = 0; sl < slabs; ++sl)
                items.push_back(make_uint4((uint32_t)(qb * NQ), (uint32_t)std::min<uint64_t>(nq, (qb + 1) * NQ),
                                           (uint32_t)sl, (uint32_t)sl + 1));
        DBuf<uint4> d_items;
        DBuf<uint2> d_adj;
        d_items.ensure(items.size());
        d_adj.ensure(adj.size());
        KJ_CUDA(cudaMemcpyAsync(d_items.p, items.data(), 16 * items.size(), cudaMemcpyHostToDevice, s));
        KJ_CUDA(cudaMemcpyAsync(d_adj.p, adj.data(), 8 * adj.size(), cudaMemcpyHostToDevice, s));
        // pairs at or beyond the counted radius are never counted: drop their blocks
        last_hist_pairs = nq * N;
        last_hist_screened = last_hist_pairs;
        if (box_filter) {
            const double r2 = ncount < nb ? S_thr[ncount] : em * em;
            uint64_t nadj = adj.size();
            last_hist_screened = filter_items(d_items.p, items.size(), qp.p, hJ.p, hbox.p, d_adj, nadj, r2);
        }
        TcJoinArgs a{};
        a.Bh = Bh_id.p;
        a.row_halfs = row_halfs;
        a.ksteps = tc_ksteps();
        a.n = n;
        a.qpos = qp.p;
        a.A = hJ.p;
        a.items = d_items.p;
        a.adj = d_adj.p;
        a.K = 1;
        a.L = 1;
        a.delta = f32_round_up(tc_delta());
        a.n_bins = nb;
        a.n_count = ncount;
        a.tables = d_tab.p;
        a.inv_width_scaled = (float)(Ssc / width);
        a.X64 = X64.p;
        a.eps_mean = em;
        a.limit_sq = em * em;
        a.inv_width = 1.0 / width;
        a.counts = d_cnt;
        Timer t(s);
        launch_hist_tc(a, hsh, items.size(), N, s);
        last_hist_kernel_ms = t.ms();
        if (getenv("KNNJ_JOIN_STATS"))
            fprintf(stderr, "hist: queries %llu items %zu bins %u/%u pairs %llu screened %llu ms %.1f\n",
                    (unsigned long long)nq, items.size(), ncount, nb,
                    (unsigned long long)last_hist_pairs, (unsigned long long)last_hist_screened,
                    last_hist_kernel_ms);
    }

    // Counts select_eps_beta (epsilon.cpp:122-141) needs, for the sampled queries hq
    // (this shard's contiguous slice of them when sharded; `reduce` sums a u64 vector
    // over all shards). Exact for every bin when `full` (the profile was requested).
    // Otherwise a pilot slice (every 32nd sampled query) is binned in full to place a
    // cap where its cumulative count passes 2x the target; the other queries only count
    // bins below the cap (their pairs beyond it leave through a one-compare fast path),
    // and the result is exact for bins [0, returned) with the cumulative count already
    // >= target there, so lower_bound selects the same bin as with the full histogram.
    // If the capped counts fall short, the rest is re-binned in full.
    int hist_cap_mode = 1;  // 0: never cap, 1: cap when the histogram is large, 2: always
    // The pilot bins only the lowest 4% of the bins, then a tenth, then a quarter, then
    // all, stopping at the first round whose counted bins reach 2x the target
    // (0: always in full; 1: every round; 2: the 4% and quarter rounds only for n <= 8).
    // In 18-D the pair count below the radius grows ~8x per bin, so a quarter of the bins
    // is already slower than binning in full; a tenth is not (C2's cap sits at bin 9).
    int pilot_cap = 2;
    double last_hist_ms_pilot = 0.0;
    uint32_t hist_for_selection(const std::vector<uint64_t>& hq, uint32_t shard, uint32_t nshard,
                                double em, uint32_t nb, double target, bool full,
                                const std::function<void(uint64_t*, uint64_t)>& reduce,
                                uint64_t* raw) {
        const uint64_t nq = hq.size();
        std::fill(raw, raw + nb, 0ull);
        const double pairs = double(nq) * double(N);
        const bool cap = !full && hist_cap_mode != 0 && nb > 2 &&
                         (hist_cap_mode == 2 || pairs >= 268435456.0);
        double kms = 0.0;
        if (!cap) {
            histogram_queries(hq.data(), nq, em, nb, raw, 0, shard, nshard);
            kms += last_hist_kernel_ms;
            reduce(raw, nb);
            last_hist_kernel_ms = kms;
            return nb;
        }
        // pilot: every STRIDE-th sampled query (>= 64th), at most ~8k of them (enough to
        // place the cap; a cap that falls short only costs the full re-binning)
        const uint64_t STRIDE = std::max<uint64_t>(64, nq / 8192);
        std::vector<uint64_t> pilot, rest;
        for (uint64_t i = 0; i < nq; ++i) (i % STRIDE == 0 ? pilot : rest).push_back(hq[i]);
        const uint64_t npilot = (nq + STRIDE - 1) / STRIDE;  // over all shards
        std::vector<uint64_t> praw(nb, 0), rraw(nb, 0);
        // the pilot itself first counts only the lowest third of the bins (exact there);
        // if its cumulative count does not reach 2x the target inside them it is re-run
        // over all bins
        auto place_cap = [&](uint32_t counted) {
            uint64_t run = 0;
            for (uint32_t b = 0; b < counted; ++b) {
                run += praw[b];
                if (double(run) / double(npilot) >= 2.0 * target) return b + 1;
            }
            return nb + 1;  // not found inside the counted bins
        };
        // capped pilot rounds at a tenth of the bins, then (n <= 8, where the counts grow
        // slowly with the radius) a quarter, then in full
        std::vector<uint32_t> rounds;
        if (pilot_cap != 0) {
            std::vector<uint32_t> want;
            if (pilot_cap == 1 || n <= 8) want.push_back(std::max<uint32_t>(4, nb / 25));
            want.push_back(std::max<uint32_t>(8, nb / 10));
            if (pilot_cap == 1 || n <= 8) want.push_back(std::max<uint32_t>(8, nb / 4));
            for (uint32_t c : want)
                if (c < nb && (rounds.empty() || c > rounds.back())) rounds.push_back(c);
        }
        rounds.push_back(nb);
        uint32_t bcap = nb + 1;
        bool pilot_partial = false;
        for (uint32_t rc : rounds) {
            std::fill(praw.begin(), praw.end(), 0ull);
            histogram_queries(pilot.data(), pilot.size(), em, nb, praw.data(), rc < nb ? rc : 0, shard,
                              nshard);
            kms += last_hist_kernel_ms;
            reduce(praw.data(), nb);
            pilot_partial = rc < nb;
            bcap = place_cap(rc);
            if (bcap <= rc) break;  // the cap lies inside the bins this round counted
        }
        last_hist_ms_pilot = kms;
        bcap = std::min<uint32_t>(bcap, nb);
        uint64_t run = 0;
        if (bcap < nb) {
            histogram_queries(rest.data(), rest.size(), em, nb, rraw.data(), bcap, shard, nshard);
            kms += last_hist_kernel_ms;
            reduce(rraw.data(), nb);
            run = 0;
            for (uint32_t b = 0; b < bcap; ++b) {
                raw[b] = praw[b] + rraw[b];
                run += raw[b];
            }
            if (double(run) / double(nq) >= target) {
                last_hist_kernel_ms = kms;
                return bcap;
            }
            std::fill(rraw.begin(), rraw.end(), 0ull);
        }
        if (pilot_partial) {  // the pilot's counts stop at its cap
            std::fill(praw.begin(), praw.end(), 0ull);
            histogram_queries(pilot.data(), pilot.size(), em, nb, praw.data(), 0, shard, nshard);
            kms += last_hist_kernel_ms;
            reduce(praw.data(), nb);
        }
        histogram_queries(rest.data(), rest.size(), em, nb, rraw.data(), 0, shard, nshard);
        kms += last_hist_kernel_ms;
        reduce(rraw.data(), nb);
        for (uint32_t b = 0; b < nb; ++b) raw[b] = praw[b] + rraw[b];
        last_hist_kernel_ms = kms;
        return nb;
    }

    // build_distance_histogram's query sample (epsilon.cpp:46-60, util.hpp:70-92)
    static uint64_t histogram_sample_size(uint64_t N, double frac) {
        if (!(frac > 0.0) || frac > 1.0) throw Error(1, "query_fraction must be in (0, 1]");
        uint64_t want = (uint64_t)std::floor(frac * double(N));
        want = std::max<uint64_t>(want, 100);
        return std::min<uint64_t>(want, N);
    }
    // The sample comes back unsorted (the reference sorts it): the counts do not depend
    // on the order of the queries, and the device sorts them into its candidate order.
    SampleWork* sample_work = nullptr;  // the sampler's buffers, kept across runs
    std::vector<uint64_t> draw_histogram_sample(double frac, uint64_t seed) {
        const uint64_t want = histogram_sample_size(N, frac);
        if (!sample_work) sample_work = sample_work_new();
        return sample_seeded(N, want, seed, false, sample_work);
    }
    std::vector<uint64_t> histogram_sample(double frac, uint64_t seed) {
        return draw_histogram_sample(frac, seed);
    }

    // ------------------------------------------------------------ grid levels
    static double unorder(unsigned long long o) {
        unsigned long long b = (o & 0x8000000000000000ull) ? (o & 0x7FFFFFFFFFFFFFFFull) : ~o;
        double v;
        std::memcpy(&v, &b, 8);
        return v;
    }
    std::vector<double> mm_lo;  // Morton box of the working coords (first <=10 dims)
    DBuf<double> d_mm;
    uint32_t ensure_morton_box() {
        const uint32_t md = std::min<uint32_t>(n, morton_dims);
        if (mm_lo.size() != md) {
            d_u64a.ensure(64);
            d_u64b.ensure(64);
            std::vector<unsigned long long> i0(md, ~0ull), i1(md, 0ull), mn(md), mx(md);
            KJ_CUDA(cudaMemcpyAsync(d_u64a.p, i0.data(), 8 * md, cudaMemcpyHostToDevice, s));
            KJ_CUDA(cudaMemcpyAsync(d_u64b.p, i1.data(), 8 * md, cudaMemcpyHostToDevice, s));
            launch_minmax(X64.p, N, n, md, d_u64a.p, d_u64b.p, s);
            KJ_CUDA(cudaMemcpyAsync(mn.data(), d_u64a.p, 8 * md, cudaMemcpyDeviceToHost, s));
            KJ_CUDA(cudaMemcpyAsync(mx.data(), d_u64b.p, 8 * md, cudaMemcpyDeviceToHost, s));
            sync();
            mm_lo.resize(md);
            std::vector<double> inv(md);
            for (uint32_t j = 0; j < md; ++j) {
                mm_lo[j] = unorder(mn[j]);
                const double r = unorder(mx[j]) - mm_lo[j];
                inv[j] = r > 0 ? 1.0 / r : 0.0;
            }
            d_mm.ensure(2 * md);
            KJ_CUDA(cudaMemcpyAsync(d_mm.p, mm_lo.data(), 8 * md, cudaMemcpyHostToDevice, s));
            KJ_CUDA(cudaMemcpyAsync(d_mm.p + md, inv.data(), 8 * md, cudaMemcpyHostToDevice, s));
        }
        return md;
    }
    // GridIndex::build (grid_index.cpp:13-75) at cell width w (level 0: w = eps).
    void build_level(int L, uint32_t m, double w) {
        Level& lv = levels[L];
        if (lv.built && lv.m == m && lv.w == w) return;
        grid_tables_into(lv, m, w);
        finish_level(lv);
    }
    // GridIndex::build's tables (grid_index.cpp:13-75) for lv: B, G, A, slot, posOf
    // Grid tables over the points with ids in [p0, p1) (default all; a slice for the
    // candidate-split histogram of sharded runs). Cell geometry from all points.
    void grid_tables_into(Level& lv, uint32_t m, double w, uint64_t p0 = 0, uint64_t p1 = ~0ull,
                          bool point_tables = true) {
        p1 = std::min<uint64_t>(p1, N);
        const uint64_t cnt = p1 > p0 ? p1 - p0 : 0;
        lv.built = false;
        lv.m = m;
        lv.w = w;
        lv.prec_w = w;
        // min / max per indexed dim (exact)
        d_u64a.ensure(64);
        d_u64b.ensure(64);
        std::vector<unsigned long long> init_mn(m, ~0ull), init_mx(m, 0ull);
        KJ_CUDA(cudaMemcpyAsync(d_u64a.p, init_mn.data(), 8 * m, cudaMemcpyHostToDevice, s));
        KJ_CUDA(cudaMemcpyAsync(d_u64b.p, init_mx.data(), 8 * m, cudaMemcpyHostToDevice, s));
        launch_minmax(X64.p, N, n, m, d_u64a.p, d_u64b.p, s);
        std::vector<unsigned long long> mn(m), mx(m);
        KJ_CUDA(cudaMemcpyAsync(mn.data(), d_u64a.p, 8 * m, cudaMemcpyDeviceToHost, s));
        KJ_CUDA(cudaMemcpyAsync(mx.data(), d_u64b.p, 8 * m, cudaMemcpyDeviceToHost, s));
        sync();
        lv.mins.resize(m);
        lv.maxs.resize(m);
        for (uint32_t j = 0; j < m; ++j) {
            lv.mins[j] = unorder(mn[j]);
            lv.maxs[j] = unorder(mx[j]);
        }
        lv.cpd.resize(m);
        lv.strides.resize(m);
        unsigned __int128 total = 1;
        for (uint32_t j = 0; j < m; ++j) {
            double extent = (lv.maxs[j] - lv.mins[j]) / w;
            if (!(extent < 9.2e18)) {
                throw Error(3, "grid extent overflows linear cell ids: dimension " +
                                   std::to_string(j) + " requires about " +
                                   std::to_string(extent) + " cells of width " +
                                   std::to_string(w));
            }
            lv.cpd[j] = std::max<uint64_t>(1, (uint64_t)std::floor(extent) + 1);
            total *= lv.cpd[j];
            if (total > std::numeric_limits<uint64_t>::max()) {
                std::string req;
                for (uint32_t t = 0; t <= j; ++t) req += (t ? "x" : "") + std::to_string(lv.cpd[t]);
                throw Error(3, "grid extent overflows linear cell ids: required extent " + req +
                                   " exceeds 64-bit range");
            }
        }
        lv.strides[m - 1] = 1;
        for (uint32_t j = m - 1; j-- > 0;) lv.strides[j] = lv.strides[j + 1] * lv.cpd[j + 1];
        lv.key_bits = bits_for((uint64_t)(total - 1));

        DBuf<double> d_mins;
        DBuf<uint64_t> d_cs;
        d_mins.ensure(m);
        d_cs.ensure(2 * m);
        KJ_CUDA(cudaMemcpyAsync(d_mins.p, lv.mins.data(), 8 * m, cudaMemcpyHostToDevice, s));
        KJ_CUDA(cudaMemcpyAsync(d_cs.p, lv.cpd.data(), 8 * m, cudaMemcpyHostToDevice, s));
        KJ_CUDA(cudaMemcpyAsync(d_cs.p + m, lv.strides.data(), 8 * m, cudaMemcpyHostToDevice, s));
        DBuf<uint64_t>& keys = gk_keys;
        DBuf<uint64_t>& skeys = gk_skeys;
        DBuf<uint32_t>& vals = gk_vals;
        DBuf<uint32_t>& runidx = gk_runidx;
        keys.ensure(cnt);
        skeys.ensure(cnt);
        vals.ensure(cnt);
        lv.A.ensure(cnt);
        launch_cell_keys(X64.p + p0 * n, cnt, n, m, d_mins.p, w, d_cs.p, d_cs.p + m, keys.p, vals.p, s,
                         (uint32_t)p0);
        sort_pairs_u64_u32(sc, keys.p, skeys.p, vals.p, lv.A.p, cnt, lv.key_bits, s);
        runidx.ensure(cnt);
        launch_head_flags(skeys.p, cnt, vals.p, s);  // vals reused as flags
        inclusive_sum(sc, vals.p, runidx.p, cnt, s);
        uint32_t nruns = 0;
        if (cnt) KJ_CUDA(cudaMemcpyAsync(&nruns, runidx.p + cnt - 1, 4, cudaMemcpyDeviceToHost, s));
        sync();
        lv.ncells = nruns;
        lv.B.ensure(nruns);
        lv.G.ensure(nruns);
        if (point_tables) {
            lv.slot.ensure(N);
            lv.posOf.ensure(N);
        }
        if (cnt)
            launch_grid_tables(skeys.p, lv.A.p, runidx.p, cnt, lv.B.p, lv.G.p,
                               point_tables ? lv.slot.p : nullptr, point_tables ? lv.posOf.p : nullptr, s);
        lv.npts = cnt;
        lv.bbox_ready = lv.xj_ready = lv.xs_ready = lv.tc_ready = false;
    }
    // the join's order and operands on top of the tables
    void finish_level(Level& lv) {
        DBuf<uint64_t>& keys = gk_keys;
        DBuf<uint64_t>& skeys = gk_skeys;
        DBuf<uint32_t>& vals = gk_vals;
        const uint32_t nruns = (uint32_t)lv.ncells;
        // join order: same cell ranges, Morton order inside each cell
        {
            const uint32_t md = ensure_morton_box();
            const uint32_t sb = bits_for(nruns ? nruns - 1 : 0);
            // code bits per dim: as many as the 64-bit key leaves next to the cell slot
            const uint32_t mb = std::max<uint32_t>(1, std::min<uint32_t>(morton_bits, (64 - sb) / md));
            launch_morton_keys(X64.p, lv.A.p, lv.slot.p, N, n, md, d_mm.p, d_mm.p + md, keys.p,
                               vals.p, s, mb);
            lv.J.ensure(N);
            lv.posJ.ensure(N);
            sort_pairs_u64_u32(sc, keys.p, skeys.p, vals.p, lv.J.p, N, (int)std::min<uint32_t>(64, md * mb + sb), s);
            launch_inverse(lv.J.p, N, lv.posJ.p, s);
        }
        lv.bbox_ready = false;
        lv.xj_ready = false;
        lv.xs_ready = false;  // the SIMT join's FP32 SoA copy is built on first use
        lv.tc_ready = false;
        if (use_tc()) prep_tc(lv);
        sync();
        lv.built = true;
    }

    // Tensor-core screen policy. Operand rows: [lo | hi | hi | nb_hi nb_lo] in FP16
    // (K = 3n+2, ~22-bit products) padded to 64-half k-blocks (KB <= 5: n <= 106); wider
    // points use the SIMT kernels.
    bool tc_enabled = true;
    int tc_small_cta = 2;  // 0 off, 1 on, 2 for n > 8
    bool tc_item_halves = true;  // small CTAs over 256-query items (tc_halves)
    bool grid_all_dims = false;  // this run's grid indexes every dim (m == n)
    bool item_radius = true;  // fallback levels filter each item at its rows' K-th bound
    bool split_items = true;  // split oversized work items into candidate-range parts
    uint32_t tc_slack = 24;       // tcgen05 join list capacity K + slack (compaction when full)
    bool finalize_xj = true;      // finalize reads FP64 rows from a join-ordered copy
    bool early_d2h = true;        // knnj_run: result D2H overlaps classification + fallback
    bool stream_host = true;      // knnj_run into pinned outputs: rows written by the finalize
    uint32_t join_chunks = 16;    // level-0 launches (finalize of one overlaps the next join)
    uint32_t chunk_min_rows = 65536;  // ... each of at least this many query rows
    uint32_t fin_blocks = 148 * 2;    // grid of a chunk's overlapped finalize (0: one warp per row)
    // (74 blocks of 8 warps: enough stores in flight for PCIe without slowing the join
    // much; the same copy through cp.async.bulk (TMA) measured slower, 1.95 vs 1.73 s)
    uint32_t copy_blocks = 74;        // grid of a chunk's row copy to the host (0: one warp per row)
    // level-0 radius bound (run_impl): sample size, quantile (per mille) of the sample's
    // K-th sq, the largest bound worth using (fraction of the filter radius^2), and the
    // smallest pass it is tried on
    bool kth_bound = true;
    // the bounded pass on a grid of width ~B with cell runs (run_impl). Off by default: on C5
    // it screens 3.3x fewer pairs (1.64e12 -> 4.96e11) yet runs slower (1.27 vs 1.05 s),
    // because the epilogue's cost follows the items' 128-row tiles (the fine cells' runs fill
    // them to ~60%) and the rare path, not the pair count
    bool bound_grid = false;
    double bound_grid_frac = 0.8;    // ... when B is below this fraction of level 0's width
    uint32_t bound_group_span = 8;   // ... with cell runs of up to this many cells
    // cell runs in the level-0 pass when cells hold few queries (C4: 3.92 -> 3.47 s; 0/1 off)
    uint32_t level0_group_span = 8;
    uint32_t fallback_group_span = 8;  // ... and in the fallback levels (few rows per cell)
    uint32_t bound_sample = 4096;
    uint32_t kth_bound_q = 999;
    double bound_max_frac = 0.8;
    uint64_t bound_min_rows = 200000;

    // Sample points for the radius bound: up to `cap` points from each of `cells` cells
    // strided over the level's non-empty cells (whole cells: the sample pass runs one full
    // work item per cell instead of one item per sampled query)
    uint32_t bound_cells = 64;
    std::vector<uint32_t> cell_sample(const Level& lv, uint32_t cells, uint32_t cap) {
        const uint64_t nc = lv.ncells;
        const uint64_t pick = std::min<uint64_t>(cells, nc);
        std::vector<uint2> g(pick);
        for (uint64_t j = 0; j < pick; ++j)
            KJ_CUDA(cudaMemcpyAsync(&g[j], lv.G.p + j * nc / pick, 8, cudaMemcpyDeviceToHost, s));
        sync();
        uint64_t tot = 0;
        for (auto& r : g) tot += std::min<uint32_t>(r.y - r.x, cap);
        std::vector<uint32_t> out(tot);
        uint64_t at = 0;
        for (auto& r : g) {
            const uint32_t len = std::min<uint32_t>(r.y - r.x, cap);
            KJ_CUDA(cudaMemcpyAsync(out.data() + at, lv.A.p + r.x, 4ull * len, cudaMemcpyDeviceToHost, s));
            at += len;
        }
        sync();
        return out;
    }

    // The kth_bound_q-quantile of the exact K-th sq over the sample rows sq_ids (a
    // level-0 pass of their own; rows without K candidates count as infinite).
    double sample_kth_bound(Level& lv, const std::vector<uint32_t>& q_ids, uint32_t K, double eps2,
                            uint32_t q_permille) {
        const uint64_t S = q_ids.size();
        if (!S) return 0.0;
        DBuf<uint32_t> d_sq, d_sr, t_ids;
        DBuf<double> t_dist, t_kth;
        DBuf<uint8_t> t_st;
        d_sq.ensure(S);
        d_sr.ensure(S);
        t_ids.ensure(S * K);
        t_dist.ensure(S * K);
        t_kth.ensure(S);
        t_st.ensure(S);
        KJ_CUDA(cudaMemcpyAsync(d_sq.p, q_ids.data(), 4 * S, cudaMemcpyHostToDevice, s));
        launch_iota(d_sr.p, S, s);
        Pass Ps;
        build_pass(lv, d_sq.p, d_sr.p, S, Ps, K, 0, 1, nullptr, filter_radius2(lv));
        run_pass(lv, Ps, K, nullptr, eps2, cover2(lv), t_ids.p, t_dist.p, t_kth.p, t_st.p, nullptr);
        std::vector<double> kth(S);
        std::vector<uint8_t> st(S);
        KJ_CUDA(cudaMemcpyAsync(kth.data(), t_kth.p, 8 * S, cudaMemcpyDeviceToHost, s));
        KJ_CUDA(cudaMemcpyAsync(st.data(), t_st.p, S, cudaMemcpyDeviceToHost, s));
        sync();
        for (uint64_t i = 0; i < S; ++i)
            if (!(st[i] & ST_HAS_K)) kth[i] = kInf;
        const uint64_t at = std::min<uint64_t>(S - 1, (S * q_permille + 999) / 1000);
        std::nth_element(kth.begin(), kth.begin() + at, kth.end());
        return kth[at];
    }
    uint32_t simt_slack = 0;      // SIMT join list capacity K + slack (0: max(8, K/8))
    // Fine cascade ahead of level 0 (widths eps * f / 1000, coarsest first is NOT
    // required: each is tried on the rows still uncertified). 0 = off.
    uint32_t fine_f[2] = {0, 0};
    bool tc_fits() const { return 3 * n + 2 <= 320; }
    // operand row = KB 128-byte k-blocks of 64 halfs
    uint32_t tc_row_halfs() const { return 64u * ((3 * n + 2 + 63) / 64); }
    // K=16 UMMA steps that hold non-zero columns; the rest of the row is zero padding
    uint32_t tc_ksteps() const { return (3 * n + 2 + 15) / 16; }
    bool use_tc() const { return tc_enabled && tc_fits(); }
    // the histogram's tensor-core instances cover one or two k-blocks (n <= 42)
    bool use_tc_hist() const { return use_tc() && tc_row_halfs() <= 128; }
    double tc_S() const {
        double S = 1.0;
        while (S < Rg) S *= 2.0;
        while (S / 2.0 >= Rg && S > 1e-300) S /= 2.0;
        return S;
    }
    void prep_tc(Level& lv) {
        if (lv.tc_ready) return;
        const uint32_t rh = tc_row_halfs();
        lv.Bh.ensure(N * rh);
        // the operand's non-zero prefix (3n+2 halfs, whole 16-byte chunks); the zero padding
        // up to the 64-half k-block is written once per buffer and kept across rebuilds
        const uint32_t nz = ((3 * n + 2 + 7) / 8) * 8;
        const bool padded = lv.bh_zero_p == lv.Bh.p && lv.row_halfs == rh && lv.bh_zero_halfs == nz &&
                            N <= lv.bh_zero_rows;
        lv.row_halfs = rh;
        launch_prep_tc(X64.p, lv.J.p, N, n, d_g.p, 1.0 / tc_S(), rh, lv.Bh.p, s, padded ? nz : rh);
        if (!padded) lv.bh_zero_rows = N;
        lv.bh_zero_p = lv.Bh.p;
        lv.bh_zero_halfs = nz;
        lv.tc_ready = true;
    }
    // Bound delta on |key - sq64 / S^2| for the tensor-core screen. Scaled
    // coordinates v = (x - g) / S have |v| <= R = Rg / S <= 1 (Rg rounded up). Every term is
    // a worst case; no constant is calibrated on measured errors.
    //  (1) FP16 representation. v = hi + lo + r with |lo| <= 2^-11 |v| + 2^-25 and
    //      |r| <= 2^-22 |v| + 2^-25 per coordinate. The UMMA sums -2(a_hi b_lo + a_lo b_hi +
    //      a_hi b_hi) = -2 a.b + 2 (a_lo b_lo + (a_hi + a_lo) r_b + r_a b), so the product
    //      terms err by <= 6 u22 R^2 + 2 u24 sqrt(n) R; the norm splits |b|^2 = nb_hi + nb_lo
    //      + r and |a|^2 (same split, summed in FP32) by <= 2 u22 R^2 + 2 u24.
    //  (2) Accumulation in the tensor core. FP16 x FP16 products are exact in FP32. One
    //      K=16 UMMA adds 16 products to the accumulator; whatever its internal order and
    //      rounding, if every intermediate (aligned addend or partial sum) keeps the FP32
    //      accumulator's 24-bit significand, its error is at most 18 u23 (|D_in| + sum|p_k|):
    //      a sequential sum with any rounding direction errs by <= 16 u23 of it, an adder
    //      that aligns all 17 addends to the largest exponent and truncates them by <= 17 u23
    //      of the largest, plus u23 for the final normalisation. |D_in| is at most the sum of
    //      |p| over the earlier steps, so the chain errs by <= 18 u23 sum_s (S_s + A_s) with
    //      S_s the |p| bound of step s and A_s = sum_{s' < s} S_s'. Zero-padded steps add
    //      exactly zero. Per step: the small hi*lo products of the whole row sum to <=
    //      4 lo R (lo = u11 R + sqrt(n) u25, the bound on |x_lo|), the hi*hi products of any
    //      column subset to <= 2 R^2 (1 + u11)^2 (Cauchy-Schwarz), the norm pair to <=
    //      R^2 (1 + u10). The row puts the small products first, so the large partial sums
    //      build up only in the last steps.
    //  (3) The epilogue's FP32 roundings: |a|^2 = fl(nb_hi + nb_lo) and key = fl(D + |a|^2),
    //      |key| <= 4 R^2: 5 u24 R^2 (the cuts round up, __fadd_ru / __fsub_ru).
    //  (4) FP64: the scaled coordinates, |b|^2 and the reference's scalar-order sq64:
    //      (4n + 12) 4 U64 R^2.
    double tc_delta() const { return tc_delta_at(Rg / tc_S()); }
    // tc_delta_at(R) is a quadratic A R^2 + B R + C in the data radius R (every term
    // below is): its coefficients, inflated slightly against the evaluation's rounding,
    // for the per-item bound of items whose data lie within R of the centre
    void tc_delta_poly(double& A, double& B, double& C) const {
        const double f0 = tc_delta_at(0.0), f1 = tc_delta_at(1.0), f2 = tc_delta_at(2.0);
        C = f0;
        A = (f2 - 2.0 * f1 + f0) / 2.0;
        B = f1 - A - f0;
        A *= 1.0 + 1e-9;
        B = std::max(0.0, B) * (1.0 + 1e-9) + 1e-9 * A;
        C *= 1.0 + 1e-9;
    }
    double tc_delta_at(double R) const {
        const double u10 = std::ldexp(1.0, -10), u11 = std::ldexp(1.0, -11);
        const double u22 = std::ldexp(1.0, -22), u23 = std::ldexp(1.0, -23);
        const double u24 = std::ldexp(1.0, -24), u25 = std::ldexp(1.0, -25);
        const double R2 = R * R;
        const double rt = std::sqrt((double)n);
        const double rep = 6 * u22 * R2 + 2 * u24 * rt * R + 2 * u22 * R2 + 2 * u24;
        const double lo = u11 * R + rt * u25;
        const double small_all = 4.0 * lo * R * (1.0 + u10);
        const double hh_any = 2.0 * R2 * (1.0 + u11) * (1.0 + u11);
        const double nb = R2 * (1.0 + u10);
        double acc_sum = 0.0, prefix = 0.0;
        for (uint32_t st = 0; st < tc_ksteps(); ++st) {
            const uint32_t c0 = 16 * st, c1 = 16 * st + 16;
            const auto overlaps = [&](uint32_t b, uint32_t e) { return c0 < e && b < c1; };
            double S = 0.0;
            if (overlaps(0, 2 * n)) S += small_all;
            if (overlaps(2 * n, 3 * n)) S += hh_any;
            if (overlaps(3 * n, 3 * n + 2)) S += nb;
            acc_sum += S + prefix;
            prefix += S;
        }
        // the partial sums themselves carry the earlier steps' (tiny) errors: +1e-4 relative
        const double acc = 18.0 * u23 * acc_sum * (1.0 + 1e-4);
        const double epi = 5 * u24 * R2;
        const double f64 = (4.0 * n + 12.0) * 4.0 * U64 * R2;
        return rep + acc + epi + f64;
    }
    // join kernel configuration for list capacity L (K + slack for near-ties in the band)
    struct TcJoinCfg {
        bool ok = false;
        TcShape sh{1, 2, 4};
        uint32_t L = 0;
    };
    // The GEMM-form key errs by ~u*R^2 (R = radius about the global centre) however
    // close the pair is, so the tensor-core screen only pays when that band is small
    // next to the pass's cell width w (skewed or very dense data: SIMT, whose tiles
    // are centred per block).
    bool tc_precise_for(double w) const {
        const double S = tc_S();
        return 2.0 * tc_delta() * S * S <= 0.02 * w * w;
    }
    TcJoinCfg tc_join_cfg(uint32_t K, double w, bool any_precision = false) const {
        TcJoinCfg c;
        if (!use_tc() || K < 1 || (!any_precision && !tc_precise_for(w))) return c;
        const uint32_t KB = tc_row_halfs() / 64;
        // lists past 64 entries are compacted over 128 slots (4 per lane): a wider slack
        // halves their compactions (C4, K=64: 24 -> 40 cut the tcgen05 part 2.24 -> 2.15 s)
        const uint32_t L0 = K + (K + tc_slack <= 64 ? tc_slack : std::max<uint32_t>(tc_slack, 40));
        if (KB >= 3) {
            // wide operands (43 <= n <= 106): 64-candidate tiles keep A + B stages in smem
            c.sh = TcShape{(int)KB, 1, KB == 5 ? 2 : 3, 64};
            c.L = std::min<uint32_t>(L0, 64);
        } else if (L0 <= 64) {
            // tc_small_cta: 128-query CTAs with a 2-stage ring (~106 KB): two per SM, twice
            // the epilogue warps per SM sub-partition. Measured: NS (18-D) 1675 -> 1585 ms,
            // C2 unchanged; C5 (4-D) 1455 -> 1492 ms with 128-query items (twice the items
            // to filter and sort), so the default (2) takes it for n > 8, and where the grid
            // indexes every dim with the items built at 256 queries (tc_halves)
            const bool small = tc_small_cta == 1 ||
                               (tc_small_cta == 2 && (n > 8 || (tc_item_halves && grid_all_dims)));
            c.sh = KB == 1 ? (small ? TcShape{1, 1, 2} : TcShape{1, 2, 4}) : TcShape{2, 1, 3};
            c.L = L0;
        } else {
            c.sh = KB == 1 ? TcShape{1, 1, 4} : TcShape{2, 1, 2};
            c.L = std::min<uint32_t>(L0, 128);
        }
        c.ok = K + 8 <= c.L && tc_smem_bytes(c.sh, c.L, 0, false) <= 227 * 1024;
        return c;
    }
    TcShape tc_hist_shape() const {
        return tc_row_halfs() == 64 ? TcShape{1, 2, 4} : TcShape{2, 1, 3};
    }

    double cover2(const Level& lv) const {
        bool all = true;
        uint64_t cmax = 0;
        for (uint64_t c : lv.cpd) {
            all = all && c <= 2;
            cmax = std::max(cmax, c);
        }
        if (all) return kInf;
        const double eta = 16.0 * U64 * (double(cmax) + n + 8);
        return lv.w * lv.w * (1.0 - eta);
    }

    // ------------------------------------------------------------ passes
    // Groups the queries (point ids + output rows, on device) by their cell in
    // level lv and builds work items + candidate ranges.
    // the join kernel a pass will run on (decided before its items are built)
    bool pass_uses_tc(const Level& lv, uint32_t K) const { return tc_join_cfg(K, lv.prec_w).ok; }
    // Mixed passes (item_tc): the global precision rule fails (data far from the centre
    // somewhere), but items whose own data lie close enough to it pass the rule with a
    // per-item bound; those run on the tensor cores, the rest on the SIMT kernel. Needs
    // the box filter (it measures each item's radius) and 128-query items (G = 1).
    bool item_tc = true;
    uint32_t item_tc_min_q = 32;  // ... and items with at least this many queries
    bool pass_mixed(const Level& lv, uint32_t K, double filter_r2) const {
        if (!item_tc || !(filter_r2 > 0.0) || !box_filter || tc_join_cfg(K, lv.prec_w).ok) return false;
        const TcJoinCfg c = tc_join_cfg(K, lv.prec_w, true);
        return c.ok && c.sh.G == 1;
    }
    // 128-query CTAs over 256-query items: the items (their boxes, filter and sweep
    // order) are built at 256 queries and each is launched as two 128-query halves over
    // the same candidate ranges. Taken when the grid indexes every dim (the box filter
    // gains little from the smaller query box there, while sorting twice the items'
    // blocks cost C5 ~125 ms).
    bool tc_halves(const Level& lv, const TcJoinCfg& c) const {
        return c.ok && tc_item_halves && c.sh.KB == 1 && c.sh.G == 1 && c.sh.STAGES == 2 && lv.m == n;
    }
    uint32_t pass_chunk(const Level& lv, uint32_t K, double filter_r2 = 0.0) const {
        const TcJoinCfg c = tc_join_cfg(K, lv.prec_w);
        if (c.ok) return 128u * (tc_halves(lv, c) ? 2u : c.sh.G);
        if (pass_mixed(lv, K, filter_r2)) return 128u;
        return (uint32_t)JB;
    }
    // Sharded (nshard > 1): only a contiguous run of work items in cell order is kept
    // (SURVEY.md §8e), cut at equal shares of the estimated tile work; the pass then
    // covers query positions [row_begin, row_begin + nq) of the cell-ordered list.
    // filter_r2 > 0: candidate blocks provably farther than sqrt(filter_r2) from every
    // query of their item are dropped (filter_ranges).
    void build_pass(Level& lv, const uint32_t* d_qpid, const uint32_t* d_qrow, uint64_t nq,
                    Pass& P, uint32_t K = 0, uint32_t shard = 0, uint32_t nshard = 1,
                    const uint8_t* d_dense = nullptr, double filter_r2 = 0.0, bool allow_split = true,
                    bool all_points = false, const float* d_cut_by_row = nullptr,
                    uint32_t group_span = 0) {
        P.nq = nq;
        P.nq_all = nq;
        P.nv = nq;
        P.nsplits = 0;
        P.row_begin = 0;
        P.candidates_dense = 0;
        uint32_t chunk = K ? pass_chunk(lv, K, filter_r2) : (uint32_t)JB;
        P.chunk = chunk;
        P.mixed = K && pass_mixed(lv, K, filter_r2);
        P.has_r2 = false;
        P.nitems = P.nadj = P.candidates = 0;
        if (!nq) return;
        P.qpos.ensure(nq);
        P.qrow.ensure(nq);
        DBuf<uint32_t> ucell, ucnt;
        uint64_t nuc = 0;
        if (all_points && nq == N) {
            // every point is a query with row = id: the sorted positions are all positions,
            // their rows the join order itself, and the query cells every cell
            launch_iota(P.qpos.p, N, s);
            KJ_CUDA(cudaMemcpyAsync(P.qrow.p, lv.J.p, 4 * N, cudaMemcpyDeviceToDevice, s));
            nuc = lv.ncells;
            ucell.ensure(nuc);
            ucnt.ensure(nuc);
            launch_iota(ucell.p, nuc, s);
            launch_range_len(lv.G.p, nuc, ucnt.p, s);
        } else {
            DBuf<uint32_t> pos_unsorted, qcell;
            pos_unsorted.ensure(nq);
            launch_map_u32(d_qpid, lv.posJ.p, nq, pos_unsorted.p, s);
            sort_pairs_u32_u32(sc, pos_unsorted.p, P.qpos.p, d_qrow, P.qrow.p, nq, bits_for(N), s);
            qcell.ensure(nq);
            {
                DBuf<uint32_t> tmp;
                tmp.ensure(nq);
                launch_map_u32(P.qpos.p, lv.J.p, nq, tmp.p, s);
                launch_map_u32(tmp.p, lv.slot.p, nq, qcell.p, s);
            }
            DBuf<uint64_t> d_nruns;
            ucell.ensure(nq);
            ucnt.ensure(nq);
            d_nruns.ensure(1);
            rle(sc, qcell.p, ucell.p, ucnt.p, d_nruns.p, nq, s);
            KJ_CUDA(cudaMemcpyAsync(&nuc, d_nruns.p, 8, cudaMemcpyDeviceToHost, s));
            sync();
        }
        trace().mark("build: query cells", s);
        DBuf<uint32_t> ufirst, nit, item_off, adj_cnt, adj_off;
        ufirst.ensure(nuc + 1);
        exclusive_sum(sc, ucnt.p, ufirst.p, nuc, s);
        // items per unique cell = ceil(cnt / JB): reuse host loop via device copy
        std::vector<uint32_t> h_cnt(nuc);
        KJ_CUDA(cudaMemcpyAsync(h_cnt.data(), ucnt.p, 4 * nuc, cudaMemcpyDeviceToHost, s));
        sync();
        // SIMT level-0 join over sparse cells (few queries per cell): 32-query items on
        // 32-thread blocks instead of mostly idle 128-thread ones. (Not in the fallback
        // levels: few queries against huge neighbourhoods are tile-load bound there, and
        // 128 threads load a tile 4x faster; measured on C4.)
        // (SIMT passes only: a 128-query tensor-core shape, G = 1, also has chunk == JB)
        if (chunk == (uint32_t)JB && K && !P.mixed && !tc_join_cfg(K, lv.prec_w).ok &&
            (&lv == &levels[0] || &lv >= &levels[40]) &&
            double(nq) / double(std::max<uint64_t>(nuc, 1)) < 48.0) {
            chunk = 32;
            P.chunk = 32;
        }
        // Cell runs (group_span > 1): consecutive query cells of one row of the grid (equal
        // in all but the last dim, at most group_span cells apart) whose queries fit one
        // work item share it; its candidates are the union of their neighbourhoods (rows
        // over [c_first - 1, c_last + 1] in the last dim), a superset for each query. A
        // fine grid holds few queries per cell; runs fill the item's 128-query tiles.
        DBuf<uint32_t> uspan;
        DBuf<unsigned long long> rowwalk;  // cell runs: each row's own-cell walk (the counters)
        if (group_span > 1 && nuc > 1 && 2 * nq < (uint64_t)chunk * nuc) {
            // the reference's walk counters stay per cell: each launch row's own-cell
            // neighbourhood size, before the cells are merged into runs
            {
                DBuf<uint64_t> d_cs0;
                d_cs0.ensure(2 * lv.m);
                KJ_CUDA(cudaMemcpyAsync(d_cs0.p, lv.cpd.data(), 8 * lv.m, cudaMemcpyHostToDevice, s));
                KJ_CUDA(cudaMemcpyAsync(d_cs0.p + lv.m, lv.strides.data(), 8 * lv.m, cudaMemcpyHostToDevice, s));
                DBuf<uint32_t> cnt0;
                DBuf<unsigned long long> cs0;
                cnt0.ensure(nuc);
                cs0.ensure(nuc);
                launch_adj_count(lv.B.p, lv.ncells, ucell.p, nuc, lv.m, d_cs0.p, d_cs0.p + lv.m, cnt0.p, s,
                                 nullptr, lv.G.p, cs0.p);
                rowwalk.ensure(nq);
                launch_row_walk(ufirst.p, ucnt.p, nuc, cs0.p, rowwalk.p, s);
            }
            std::vector<uint32_t> h_cell(nuc);
            KJ_CUDA(cudaMemcpyAsync(h_cell.data(), ucell.p, 4 * nuc, cudaMemcpyDeviceToHost, s));
            sync();
            std::vector<uint64_t> h_lin(lv.ncells);
            KJ_CUDA(cudaMemcpyAsync(h_lin.data(), lv.B.p, 8 * lv.ncells, cudaMemcpyDeviceToHost, s));
            sync();
            const uint64_t cl = lv.cpd[lv.m - 1];
            std::vector<uint32_t> g_cell, g_cnt, g_span;
            g_cell.reserve(nuc);
            uint64_t row0 = 0, c0 = 0;
            uint32_t q0 = 0;
            for (uint64_t u = 0; u < nuc; ++u) {
                const uint64_t lin = h_lin[h_cell[u]], row = lin / cl, cc = lin % cl;
                if (!g_cell.empty() && row == row0 && cc - c0 < group_span && q0 + h_cnt[u] <= chunk) {
                    q0 += h_cnt[u];
                    g_cnt.back() = q0;
                    g_span.back() = (uint32_t)(cc - c0 + 1);
                    continue;
                }
                g_cell.push_back(h_cell[u]);
                g_cnt.push_back(h_cnt[u]);
                g_span.push_back(1);
                row0 = row;
                c0 = cc;
                q0 = h_cnt[u];
            }
            nuc = g_cell.size();
            KJ_CUDA(cudaMemcpyAsync(ucell.p, g_cell.data(), 4 * nuc, cudaMemcpyHostToDevice, s));
            KJ_CUDA(cudaMemcpyAsync(ucnt.p, g_cnt.data(), 4 * nuc, cudaMemcpyHostToDevice, s));
            uspan.ensure(nuc);
            KJ_CUDA(cudaMemcpyAsync(uspan.p, g_span.data(), 4 * nuc, cudaMemcpyHostToDevice, s));
            exclusive_sum(sc, ucnt.p, ufirst.p, nuc, s);
            h_cnt.swap(g_cnt);
        }
        std::vector<uint32_t> h_ioff(nuc + 1);
        uint64_t tot = 0;
        for (uint64_t u = 0; u < nuc; ++u) {
            h_ioff[u] = (uint32_t)tot;
            tot += (h_cnt[u] + chunk - 1) / chunk;
        }
        h_ioff[nuc] = (uint32_t)tot;
        P.nitems = tot;
        item_off.ensure(nuc + 1);
        KJ_CUDA(cudaMemcpyAsync(item_off.p, h_ioff.data(), 4 * (nuc + 1), cudaMemcpyHostToDevice, s));
        // adjacency
        DBuf<uint64_t> d_cs;
        d_cs.ensure(2 * lv.m);
        KJ_CUDA(cudaMemcpyAsync(d_cs.p, lv.cpd.data(), 8 * lv.m, cudaMemcpyHostToDevice, s));
        KJ_CUDA(cudaMemcpyAsync(d_cs.p + lv.m, lv.strides.data(), 8 * lv.m, cudaMemcpyHostToDevice, s));
        adj_cnt.ensure(nuc + 1);
        adj_off.ensure(nuc + 1);
        launch_adj_count(lv.B.p, lv.ncells, ucell.p, nuc, lv.m, d_cs.p, d_cs.p + lv.m, adj_cnt.p, s,
                         uspan.p);
        KJ_CUDA(cudaMemsetAsync(adj_cnt.p + nuc, 0, 4, s));
        exclusive_sum(sc, adj_cnt.p, adj_off.p, nuc + 1, s);
        uint32_t nadj = 0;
        KJ_CUDA(cudaMemcpyAsync(&nadj, adj_off.p + nuc, 4, cudaMemcpyDeviceToHost, s));
        sync();
        P.nadj = nadj;
        P.adj.ensure(nadj);
        DBuf<unsigned long long> csize;
        csize.ensure(nuc);
        launch_adj_fill(lv.B.p, lv.G.p, lv.ncells, ucell.p, nuc, lv.m, d_cs.p, d_cs.p + lv.m,
                        adj_off.p, P.adj.p, csize.p, s, uspan.p, adj_order(lv.m));
        DBuf<uint4> items_unsorted;
        DBuf<unsigned long long> work;
        items_unsorted.ensure(tot);
        work.ensure(tot);
        launch_items(ufirst.p, ucnt.p, item_off.p, adj_off.p, nuc, csize.p, items_unsorted.p,
                     work.p, chunk, s);
        std::vector<uint4> h_items(tot);
        std::vector<unsigned long long> h_work(tot);
        KJ_CUDA(cudaMemcpyAsync(h_items.data(), items_unsorted.p, 16 * tot, cudaMemcpyDeviceToHost, s));
        KJ_CUDA(cudaMemcpyAsync(h_work.data(), work.p, 8 * tot, cudaMemcpyDeviceToHost, s));
        sync();
        trace().mark("build: runs + adjacency + items", s);
        // items are in cell order here; a shard keeps a contiguous run of them
        uint64_t i0 = 0, i1 = tot;
        if (nshard > 1) {
            // cost of an item ~ its candidate tiles (+ a fixed per-item overhead); with the
            // box filter on, the tiles that survive it (every rank counts all items: the
            // unfiltered count misjudges cells whose neighbourhood holds far clusters)
            std::vector<double> cost(tot);
            std::vector<uint32_t> kept;
            // (when the grid indexes every dim the filter hardly changes an item's cost: the
            // far blocks it drops are those of clusters close in the first m dims only)
            if (filter_r2 > 0.0 && box_filter && tot && lv.m < n)
                kept = filtered_blocks(lv, items_unsorted.p, tot, P.qpos.p, P.adj.p, filter_r2);
            for (uint64_t i = 0; i < tot; ++i) {
                const uint32_t q = h_items[i].y - h_items[i].x;
                const double cand = kept.empty() ? (q ? double(h_work[i] / q) : 0.0)
                                                 : double(kept[i]) * double(FB);
                cost[i] = cand + 8.0 * 128.0;
            }
            shard_range(cost.data(), tot, shard, nshard, &i0, &i1);
        }
        const uint32_t r0 = i0 < i1 ? h_items[i0].x : 0;
        const uint32_t r1 = i0 < i1 ? h_items[i1 - 1].y : 0;
        unsigned long long walk_all = 0;
        if (rowwalk.p && i0 < i1) {  // cell runs: the per-cell walk of the owned rows
            DBuf<unsigned long long> d_w;
            d_w.ensure(2);
            KJ_CUDA(cudaMemsetAsync(d_w.p, 0, 16, s));
            launch_walk_sum(rowwalk.p + r0, P.qrow.p + r0, r1 - r0, d_dense, d_w.p, s);
            unsigned long long hw[2] = {0, 0};
            KJ_CUDA(cudaMemcpyAsync(hw, d_w.p, 16, cudaMemcpyDeviceToHost, s));
            sync();
            walk_all = hw[0];
            if (d_dense) P.candidates_dense = hw[1];
        } else if (d_dense && i0 < i1) {
            DBuf<unsigned long long> d_dc;
            d_dc.ensure(1);
            KJ_CUDA(cudaMemsetAsync(d_dc.p, 0, 8, s));
            launch_dense_cand(items_unsorted.p + i0, work.p + i0, i1 - i0, P.qrow.p, d_dense,
                              d_dc.p, s);
            unsigned long long dc = 0;
            KJ_CUDA(cudaMemcpyAsync(&dc, d_dc.p, 8, cudaMemcpyDeviceToHost, s));
            sync();
            P.candidates_dense = dc;
        }
        // rebase the owned items to the shard's row range
        std::vector<uint4> own(h_items.begin() + i0, h_items.begin() + i1);
        std::vector<unsigned long long> own_w(h_work.begin() + i0, h_work.begin() + i1);
        unsigned long long cand = 0;
        for (uint64_t i = 0; i < own.size(); ++i) {
            own[i].x -= r0;
            own[i].y -= r0;
            cand += own_w[i];
        }
        const unsigned long long work_pairs = cand;  // pairs the items cover (runs: unions)
        if (rowwalk.p) cand = walk_all;             // the reference walk's count
        const uint64_t nq_own = r1 - r0;
        // Split items whose candidate set is a large slice of the pass (few queries
        // against huge neighbourhoods: fallback passes, skewed cells) into parts over
        // candidate sub-ranges, so the tail of the schedule is not one CTA's scan.
        P.nv = nq_own;
        P.nsplits = 0;
        std::vector<uint2> extra_adj;
        std::vector<uint32_t> vsrc;
        std::vector<uint4> splits;
        {
            std::vector<uint64_t> csz(own.size());
            double W = 0.0;
            uint64_t cmax = 0;
            for (uint64_t i = 0; i < own.size(); ++i) {
                const uint32_t q = own[i].y - own[i].x;
                csz[i] = q ? own_w[i] / q : 0;
                W += double(csz[i]) / 128.0 + 8.0;  // candidate tiles + per-item overhead
                cmax = std::max(cmax, csz[i]);
            }
            const double part_tiles = std::max(64.0, W / (148.0 * 4.0));
            if (split_items && allow_split && K > 0 && double(cmax) / 128.0 > 2.0 * part_tiles) {
                std::vector<uint2> h_adj(P.nadj);
                KJ_CUDA(cudaMemcpyAsync(h_adj.data(), P.adj.p, 8 * P.nadj, cudaMemcpyDeviceToHost, s));
                sync();
                std::vector<uint4> kept;
                std::vector<unsigned long long> kept_w;
                for (uint64_t i = 0; i < own.size(); ++i) {
                    const uint4 it = own[i];
                    const uint32_t q = it.y - it.x;
                    const double tiles = double(csz[i]) / 128.0;
                    if (!(tiles > 2.0 * part_tiles) || q == 0) {
                        kept.push_back(it);
                        kept_w.push_back(own_w[i]);
                        continue;
                    }
                    const uint32_t parts = (uint32_t)std::min<double>(32.0, std::ceil(tiles / part_tiles));
                    const uint64_t per = (csz[i] + parts - 1) / parts;
                    const uint32_t vbase = (uint32_t)P.nv;
                    uint32_t made = 0;
                    uint64_t filled = 0;
                    uint32_t a_begin = (uint32_t)(P.nadj + extra_adj.size());
                    for (uint32_t r = it.z; r < it.w; ++r) {
                        uint32_t lo = h_adj[r].x;
                        const uint32_t hi = h_adj[r].y;
                        while (lo < hi) {
                            const uint64_t take = std::min<uint64_t>(hi - lo, per - filled);
                            extra_adj.push_back(make_uint2(lo, lo + (uint32_t)take));
                            lo += (uint32_t)take;
                            filled += take;
                            if (filled == per) {  // close this part
                                const uint32_t a_end = (uint32_t)(P.nadj + extra_adj.size());
                                const uint32_t v0 = vbase + made * q;
                                kept.push_back(make_uint4(v0, v0 + q, a_begin, a_end));
                                kept_w.push_back((unsigned long long)q * filled);
                                ++made;
                                filled = 0;
                                a_begin = a_end;
                            }
                        }
                    }
                    if (filled) {
                        const uint32_t a_end = (uint32_t)(P.nadj + extra_adj.size());
                        const uint32_t v0 = vbase + made * q;
                        kept.push_back(make_uint4(v0, v0 + q, a_begin, a_end));
                        kept_w.push_back((unsigned long long)q * filled);
                        ++made;
                    }
                    for (uint32_t pidx = 0; pidx < made; ++pidx)
                        for (uint32_t j = 0; j < q; ++j) vsrc.push_back(it.x + j);
                    splits.push_back(make_uint4(it.x, q, made, vbase - (uint32_t)nq_own));
                    P.nv += (uint64_t)made * q;
                }
                own.swap(kept);
                own_w.swap(kept_w);
                P.nsplits = splits.size();
            }
        }
        // heaviest items first (LPT order for the block scheduler); ties keep cell order.
        // A streamed pass is cut into stream_chunks launches over contiguous row ranges
        // (items grouped by the chunk their first row falls in, LPT inside each), so one
        // chunk's finalize and result copy overlap the next chunk's join.
        const uint32_t nch = (stream_chunks > 1 && P.nv == nq_own && !P.mixed &&
                              nq_own >= (uint64_t)chunk_min_rows * stream_chunks)
                                 ? stream_chunks : 1;
        // (split-part items run on virtual rows >= nq_own; chunking is off when they exist)
        auto chunk_of = [&](const uint4& it) {
            return nch == 1 ? 0u : (uint32_t)std::min<uint64_t>(nch - 1, (uint64_t)it.x * nch / nq_own);
        };
        // (a stable counting sort on (chunk, weight class): 16 classes per doubling of the
        // item's pair count, heaviest first; O(items) where a comparison sort of C5's 470k
        // items cost tens of ms on the host)
        std::vector<uint32_t> order(own.size());
        {
            constexpr uint32_t WB = 1024;
            std::vector<uint32_t> key(own.size());
            for (uint64_t i = 0; i < own.size(); ++i) {
                const double lw = std::log2(1.0 + double(own_w[i]));
                const uint32_t wb = (uint32_t)std::min<double>(WB - 1, std::floor(16.0 * lw));
                key[i] = chunk_of(own[i]) * WB + (WB - 1 - wb);
            }
            std::vector<uint32_t> start((size_t)nch * WB + 1, 0);
            for (uint32_t k2 : key) ++start[k2 + 1];
            for (size_t b = 1; b < start.size(); ++b) start[b] += start[b - 1];
            for (uint64_t i = 0; i < own.size(); ++i) order[start[key[i]]++] = (uint32_t)i;
        }
        std::vector<uint4> h_sorted(own.size());
        for (uint64_t i = 0; i < own.size(); ++i) h_sorted[i] = own[order[i]];
        P.chunk_item.clear();
        P.chunk_row.clear();
        if (nch > 1) {
            P.chunk_item.assign(nch + 1, own.size());
            P.chunk_row.assign(nch + 1, nq_own);
            for (uint64_t i = own.size(); i-- > 0;) {
                const uint32_t c = chunk_of(h_sorted[i]);
                P.chunk_item[c] = i;
                P.chunk_row[c] = std::min<uint64_t>(P.chunk_row[c], h_sorted[i].x);
            }
            for (uint32_t c = nch; c-- > 0;) {  // empty chunks start where the next does
                P.chunk_item[c] = std::min(P.chunk_item[c], P.chunk_item[c + 1]);
                P.chunk_row[c] = std::min(P.chunk_row[c], P.chunk_row[c + 1]);
            }
            P.chunk_row[0] = 0;
            P.chunk_item[0] = 0;
        }
        if (r0 != 0 || r1 != nq || P.nv > nq_own) {
            DBuf<uint32_t> qp2, qr2;
            qp2.ensure(P.nv);
            qr2.ensure(nq_own);
            if (r1 > r0) {
                KJ_CUDA(cudaMemcpyAsync(qp2.p, P.qpos.p + r0, 4ull * nq_own, cudaMemcpyDeviceToDevice, s));
                KJ_CUDA(cudaMemcpyAsync(qr2.p, P.qrow.p + r0, 4ull * nq_own, cudaMemcpyDeviceToDevice, s));
            }
            if (P.nv > nq_own) {  // virtual rows mirror their real row's query
                P.vsrc.ensure(vsrc.size());
                KJ_CUDA(cudaMemcpyAsync(P.vsrc.p, vsrc.data(), 4 * vsrc.size(), cudaMemcpyHostToDevice, s));
                launch_map_u32(P.vsrc.p, qp2.p, vsrc.size(), qp2.p + nq_own, s);
                P.splits.ensure(splits.size());
                KJ_CUDA(cudaMemcpyAsync(P.splits.p, splits.data(), 16 * splits.size(), cudaMemcpyHostToDevice, s));
                DBuf<uint2> adj2;
                adj2.ensure(P.nadj + extra_adj.size());
                if (P.nadj)
                    KJ_CUDA(cudaMemcpyAsync(adj2.p, P.adj.p, 8 * P.nadj, cudaMemcpyDeviceToDevice, s));
                KJ_CUDA(cudaMemcpyAsync(adj2.p + P.nadj, extra_adj.data(), 8 * extra_adj.size(),
                                        cudaMemcpyHostToDevice, s));
                P.adj.swap(adj2);
                P.nadj += extra_adj.size();
            }
            P.qpos.swap(qp2);
            P.qrow.swap(qr2);
        }
        P.nq = nq_own;
        P.row_begin = r0;
        P.nitems = h_sorted.size();
        P.items.ensure(P.nitems);
        if (P.nitems)
            KJ_CUDA(cudaMemcpyAsync(P.items.p, h_sorted.data(), 16 * P.nitems, cudaMemcpyHostToDevice, s));
        sync();
        P.candidates = cand;
        P.screened = work_pairs;
        trace().mark("build: shard, splits, LPT order", s);
        // Level 0 on a grid over every dim with a radius of at least half the cell width:
        // a 128-position block spans most of its cell, so hardly any block lies beyond the
        // radius from an item's query box (C5: 0.4% of the pairs), and the nearer-rows-first
        // adjacency order (adj_order) gives most of the per-block sweep's effect. C5: build
        // 72 -> 20 ms, join kernel 855 -> 864 ms.
        const bool filter_pays = !(filter_skip_all_dims && &lv == &levels[0] && lv.m == n &&
                                   !P.mixed && !d_cut_by_row && filter_r2 >= 0.25 * lv.w * lv.w);
        if (filter_r2 > 0.0 && box_filter && P.nitems && filter_pays) {
            // rows that carry an upper bound U on their K-th sq (fallback levels: K points
            // within sqrt(U) are known to exist) need no candidate beyond sqrt(U): an item
            // filters at the largest bound among its rows
            DBuf<float> irad;
            if (d_cut_by_row) {
                irad.ensure(P.nitems);
                launch_item_max_cut(P.items.p, P.nitems, P.qrow.p, P.nq,
                                    P.nv > P.nq ? P.vsrc.p : nullptr, d_cut_by_row, irad.p, s);
            }
            filter_ranges(lv, P, filter_r2, K > 0 && (pass_uses_tc(lv, K) || P.mixed),
                          d_cut_by_row ? irad.p : nullptr);
        }
        if (K && !P.mixed && P.nitems && chunk == 256u && tc_halves(lv, tc_join_cfg(K, lv.prec_w))) {
            // launch items: each 256-query item as 128-query halves, in the LPT order
            std::vector<uint4> hi(P.nitems), ho;
            KJ_CUDA(cudaMemcpyAsync(hi.data(), P.items.p, 16 * P.nitems, cudaMemcpyDeviceToHost, s));
            sync();
            ho.reserve(2 * P.nitems);
            std::vector<uint64_t> at(P.nitems + 1);
            for (uint64_t i = 0; i < P.nitems; ++i) {
                at[i] = ho.size();
                const uint4 it = hi[i];
                if (it.y - it.x <= 128u) {
                    ho.push_back(it);
                    continue;
                }
                ho.push_back(make_uint4(it.x, it.x + 128u, it.z, it.w));
                ho.push_back(make_uint4(it.x + 128u, it.y, it.z, it.w));
            }
            at[P.nitems] = ho.size();
            for (auto& ci : P.chunk_item) ci = at[ci];
            P.nitems = ho.size();
            P.items.ensure(P.nitems);
            KJ_CUDA(cudaMemcpyAsync(P.items.p, ho.data(), 16 * P.nitems, cudaMemcpyHostToDevice, s));
            sync();
            P.chunk = 128u;
        }
    }

    // The order of an item's neighbour rows (k_adj): own row first, then by the number of
    // dims (of the first m-1) the row is offset in -- the nearer rows first, so the join's
    // top-K cut tightens early when no per-block sweep order is built. Null: index order.
    bool adj_norm_order = true;
    bool chunk_device_out = false;  // chunked level-0 pass (finalize overlapped) for device outputs too
    bool filter_skip_all_dims = true;  // build_pass: filter_pays
    DBuf<uint16_t> d_adj_order;
    uint32_t adj_order_m = 0;
    const uint16_t* adj_order(uint32_t m) {
        if (!adj_norm_order || m < 2) return nullptr;
        if (adj_order_m != m) {
            uint32_t R = 1;
            for (uint32_t j = 0; j + 1 < m; ++j) R *= 3;
            if (R > 65535) return nullptr;
            std::vector<uint16_t> ord(R);
            std::vector<uint32_t> nz(R);
            for (uint32_t r = 0; r < R; ++r) ord[r] = (uint16_t)r;
            // digits of r: base 3 over the m-1 row dims, 1 = no offset (own row: all ones)
            for (uint32_t r = 0; r < R; ++r) {
                uint32_t z = 0;
                uint32_t t = r;
                for (uint32_t j = 0; j + 1 < m; ++j, t /= 3) z += t % 3 != 1;
                nz[r] = z;
            }
            std::stable_sort(ord.begin(), ord.end(), [&](uint16_t a, uint16_t b) { return nz[a] < nz[b]; });
            d_adj_order.ensure(R);
            KJ_CUDA(cudaMemcpyAsync(d_adj_order.p, ord.data(), 2 * R, cudaMemcpyHostToDevice, s));
            sync();
            adj_order_m = m;
        }
        return d_adj_order.p;
    }

    // launches a big level-0 pass is cut into (build_pass; 1 = one launch)
    uint32_t stream_chunks = 1;

    // Box filter of a join pass (after build_pass): a candidate can matter to a query
    // only within radius r of it (level 0: eps, the dense rule; level L: the cell width
    // w_L, the coverage certificate), so 128-position blocks whose FP64 bounding box is
    // farther than r from the item's query box (all n dims, rounded down) are dropped.
    // Leaves every outcome unchanged; removes e.g. the other Gaussian clusters that
    // share a cell's 3^m neighbourhood in the first m dims.
    bool box_filter = true;
    // join passes sweep each item's kept blocks nearest-first (box centres)
    bool sweep_order = true;
    // join order inside a cell: Morton code over the first morton_dims working dims,
    // morton_bits per dim (global range)
    uint32_t morton_dims = 10, morton_bits = 3;
    // The radius a pass may filter to: every decision taken from its lists (in-eps at
    // level 0, the coverage certificate kth < cover2) concerns pairs within the cell
    // width w. When the grid is at most 2 cells wide in every dim the certificate is
    // unconditional (cover2 = inf) and nothing may be dropped.
    double filter_radius2(const Level& lv) const { return cover2(lv) < kInf ? lv.w * lv.w : 0.0; }
    // order: the nearest-first sweep, for tcgen05 passes only (their epilogue's rare path
    // is what it cuts; a SIMT pass over tiny cells (C4) would sort billions of blocks)
    void filter_ranges(Level& lv, Pass& P, double r2, bool tc_pass, const float* item_rad2 = nullptr) {
        if (!lv.bbox_ready) {
            lv.bbox.ensure(((N + FB - 1) / FB) * 2 * n);
            launch_block_boxes(X64.p, lv.J.p, N, n, lv.bbox.p, s);
            lv.bbox_ready = true;
        }
        float* r2_out = nullptr;
        if (P.mixed) {
            P.item_r2.ensure(P.nitems);
            r2_out = P.item_r2.p;
        }
        DBuf<float> dbox;  // the grid dims' data range, rounded outward
        if (P.mixed) {
            std::vector<float> hb(2 * lv.m);
            for (uint32_t d = 0; d < lv.m; ++d) {
                hb[d] = f32_round_down(lv.mins[d]);
                hb[lv.m + d] = f32_round_up(lv.maxs[d]);
            }
            dbox.ensure(2 * lv.m);
            KJ_CUDA(cudaMemcpyAsync(dbox.p, hb.data(), 8 * lv.m, cudaMemcpyHostToDevice, s));
            sync();
        }
        P.screened = filter_items(P.items.p, P.nitems, P.qpos.p, lv.J.p, lv.bbox.p, P.adj, P.nadj, r2,
                                  sweep_order && tc_pass, r2_out, lv.m,
                                  f32_round_up(2.0 * lv.w * (1.0 + 1e-6)), dbox.p, item_rad2);
        P.has_r2 = r2_out != nullptr;
    }
    // kept FB-blocks per item under the box filter (the filter's count pass only; items and
    // adj are left unchanged)
    std::vector<uint32_t> filtered_blocks(Level& lv, uint4* items, uint64_t nitems,
                                          const uint32_t* qpos, const uint2* adj, double r2) {
        if (!lv.bbox_ready) {
            lv.bbox.ensure(((N + FB - 1) / FB) * 2 * n);
            launch_block_boxes(X64.p, lv.J.p, N, n, lv.bbox.p, s);
            lv.bbox_ready = true;
        }
        const uint64_t nblk = (N + FB - 1) / FB;
        const float r2c = f32_round_up(r2 * (1.0 + 1e-9));
        DBuf<float> qbox, okey;
        DBuf<uint32_t> cnt;
        qbox.ensure(nitems * 2 * n);
        cnt.ensure(nitems);
        okey.ensure(1);
        launch_item_boxes(items, nitems, qpos, lv.J.p, X64.p, n, qbox.p, s);
        launch_filter_ranges(items, nitems, qbox.p, n, adj, lv.bbox.p, nblk, r2c, cnt.p, nullptr,
                             nullptr, nullptr, false, s, okey.p);  // ORDER count: kept blocks
        std::vector<uint32_t> h(nitems);
        KJ_CUDA(cudaMemcpyAsync(h.data(), cnt.p, 4 * nitems, cudaMemcpyDeviceToHost, s));
        sync();
        return h;
    }
    // items (qbeg, qend, abeg, aend) over adjacency ranges adj: keep only the blocks within
    // sqrt(r2) of the item's query box; adj is replaced. Returns the kept candidate pairs.
    uint64_t filter_items(uint4* items, uint64_t nitems, const uint32_t* qpos, const uint32_t* J,
                          const float* bbox, DBuf<uint2>& adj, uint64_t& nadj, double r2,
                          bool order = false, float* item_r2 = nullptr, uint32_t r_m = 0,
                          float r_2w = 0.f, const float* dbox = nullptr, const float* item_rad2 = nullptr) {
        const uint64_t nblk = (N + FB - 1) / FB;
        // FP64 scalar sums can fall below the true sq: widen, then round up to FP32
        const float r2c = f32_round_up(r2 * (1.0 + 1e-9));
        DBuf<float> qbox;
        DBuf<uint32_t> cnt, off;
        qbox.ensure(nitems * 2 * n);
        cnt.ensure(nitems + 1);
        off.ensure(nitems + 1);
        launch_item_boxes(items, nitems, qpos, J, X64.p, n, qbox.p, s);
        KJ_CUDA(cudaMemsetAsync(cnt.p + nitems, 0, 4, s));
        DBuf<float> okey, okey2;
        float* kp = nullptr;
        if (order) {
            okey.ensure(1);
            kp = okey.p;  // non-null selects the per-block (ordered) variant
        }
        d_u64a.ensure(1);
        KJ_CUDA(cudaMemsetAsync(d_u64a.p, 0, 8, s));
        launch_filter_ranges(items, nitems, qbox.p, n, adj.p, bbox, nblk, r2c, cnt.p, nullptr,
                             nullptr, nullptr, false, s, kp, d_u64a.p, nullptr, nullptr, 0, 0.f,
                             nullptr, item_rad2);
        if (order) {  // one range per kept block: the total must fit the 32-bit range ids
            unsigned long long nr = 0;
            KJ_CUDA(cudaMemcpyAsync(&nr, d_u64a.p, 8, cudaMemcpyDeviceToHost, s));
            sync();
            if (nr >= (1ull << 31)) {
                order = false;
                kp = nullptr;
                launch_filter_ranges(items, nitems, qbox.p, n, adj.p, bbox, nblk, r2c, cnt.p,
                                     nullptr, nullptr, nullptr, false, s, nullptr, nullptr, nullptr,
                                     nullptr, 0, 0.f, nullptr, item_rad2);
            }
        }
        exclusive_sum(sc, cnt.p, off.p, nitems + 1, s);
        uint32_t total = 0;
        KJ_CUDA(cudaMemcpyAsync(&total, off.p + nitems, 4, cudaMemcpyDeviceToHost, s));
        sync();
        DBuf<uint2> adj2;
        adj2.ensure(total);
        if (order) {
            okey.ensure(total);
            kp = okey.p;
        }
        d_u64a.ensure(1);
        KJ_CUDA(cudaMemsetAsync(d_u64a.p, 0, 8, s));
        launch_filter_ranges(items, nitems, qbox.p, n, adj.p, bbox, nblk, r2c, nullptr, off.p,
                             adj2.p, d_u64a.p, true, s, kp, nullptr, d_gbox.p, item_r2, r_m, r_2w, dbox,
                             item_rad2);
        if (order && total) {
            // nearest blocks first inside every item: the top-K cut converges early
            DBuf<uint2> adj3;
            adj3.ensure(total);
            okey2.ensure(total);
            size_t bytes = 0;
            auto* v_in = reinterpret_cast<uint64_t*>(adj2.p);
            auto* v_out = reinterpret_cast<uint64_t*>(adj3.p);
            KJ_CUDA(cub::DeviceSegmentedSort::SortPairs(nullptr, bytes, okey.p, okey2.p, v_in, v_out,
                                                        (int64_t)total, (int64_t)nitems, off.p,
                                                        off.p + 1, s));
            KJ_CUDA(cub::DeviceSegmentedSort::SortPairs(sc.get(bytes), bytes, okey.p, okey2.p, v_in,
                                                        v_out, (int64_t)total, (int64_t)nitems,
                                                        off.p, off.p + 1, s));
            adj2.swap(adj3);
        }
        unsigned long long scr = 0;
        KJ_CUDA(cudaMemcpyAsync(&scr, d_u64a.p, 8, cudaMemcpyDeviceToHost, s));
        sync();
        adj.swap(adj2);
        nadj = total;
        return scr;
    }

    double last_join_kernel_ms = 0.0;
    bool last_join_tc = false;
    unsigned long long last_mixed_tc_items = 0;
    // Runs the fused join over a pass, then the exact finalize (and the slow
    // path for overflowed lists). Writes rows of out_* (indexed by qrow).
    // With host_ids/host_dist (mapped pinned host memory) and a pass built in chunks, the
    // finalize of chunk c runs on s_out while chunk c+1 joins on s, and writes its rows to
    // the host too: the result copy streams under the join. Returns whether it did; the
    // rows the exact slow path rewrites afterwards are appended to *host_patch.
    bool run_pass(Level& lv, Pass& P, uint32_t K, const float* d_init_cut, double eps2,
                  double cov2, uint32_t* out_ids, double* out_dist, double* out_kth,
                  uint8_t* out_status, uint64_t* n_slow, uint32_t* host_ids = nullptr,
                  double* host_dist = nullptr, std::vector<uint32_t>* host_patch = nullptr,
                  double bound2 = 0.0) {
        if (!P.nq) return false;
        if (bound2 > 0.0 && P.nv != P.nq) throw Error(9, "a radius-bounded pass cannot hold split items");
        const TcJoinCfg tcm = tc_join_cfg(K, lv.prec_w, true);
        const bool mixed = P.mixed && P.has_r2 && tcm.ok && tcm.sh.G == 1 && P.chunk == 128u;
        const TcJoinCfg tcc = mixed ? tcm : tc_join_cfg(K, lv.prec_w);
        const bool tc = !mixed && tcc.ok && P.chunk == 128u * tcc.sh.G;
        if (!tc && !mixed && P.chunk != (uint32_t)JB && P.chunk != 32u)
            throw Error(9, "pass built for a different kernel");
        // list capacity: K plus slack for near-ties inside the screen band (overflow -> exact slow path)
        // SIMT list slack: every extra slot costs shared memory (occupancy) and insertion
        // shifts; C4 (K=64) runs 11.8 s at K+32, 9.1 s at K+8 with no overflow rows
        const uint32_t L = (tc || mixed) ? tcc.L : K + (simt_slack ? simt_slack : std::max<uint32_t>(8, K / 8));
        if (L > 256)
            throw Error(1, "k = " + std::to_string(K) + " needs a near-tie list of " + std::to_string(L) +
                               " entries; the device join holds at most 256");
        const int np = pick_np(n);
        if (np < 0) throw Error(1, "dimension count above 128 is not supported by the device join");
        if (!tc && join_smem_bytes(np, L, P.chunk) > 227 * 1024)
            throw Error(1, "k too large for the device join");
        bool mixed_tc_ran = false;
        const uint64_t nv = P.nv, nvv = P.nv - P.nq;  // launch rows; virtual (split-part) rows
        // chunk boundaries (one launch unless the pass was built in chunks)
        std::vector<uint64_t> ci = P.chunk_item, cr = P.chunk_row;
        if (ci.size() < 2 || nvv || mixed) {
            ci = {0, P.nitems};
            cr = {0, P.nq};
        }
        const size_t nch = ci.size() - 1;
        const bool to_host = host_ids && host_dist && !nvv;
        const bool overlap = nch > 1;
        if (overlap) ensure_out_stream();
        std::vector<cudaEvent_t> ev_join(nch, nullptr);
        cudaEvent_t ev_fin = nullptr;
        struct EvFree {
            std::vector<cudaEvent_t>& v;
            cudaEvent_t& f;
            ~EvFree() {
                for (auto e : v)
                    if (e) cudaEventDestroy(e);
                if (f) cudaEventDestroy(f);
            }
        } ev_free{ev_join, ev_fin};
        if (overlap) {
            for (auto& e : ev_join) KJ_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
            KJ_CUDA(cudaEventCreateWithFlags(&ev_fin, cudaEventDisableTiming));
        }
        DBuf<uint32_t>& cnt = pass_cnt;
        DBuf<uint32_t>& pos = pass_pos;
        cnt.ensure(nv);
        pos.ensure(nv * L);
        if (P.nsplits) launch_fill_u32(cnt.p, P.nq, SKIP, s);  // split real rows are merged later
        DBuf<float> cut_ext;
        if (d_init_cut && nvv) {  // virtual rows start from their real row's bound
            cut_ext.ensure(nv);
            KJ_CUDA(cudaMemcpyAsync(cut_ext.p, d_init_cut, 4 * P.nq, cudaMemcpyDeviceToDevice, s));
            launch_gather_f32(P.vsrc.p, d_init_cut, nvv, cut_ext.p + P.nq, s);
            d_init_cut = cut_ext.p;
        }
        FinalArgs f{};
        f.X64 = X64.p;
        f.n = n;
        f.A = lv.J.p;
        f.qpos = P.qpos.p;
        f.qrow = P.qrow.p;
        f.cnt = cnt.p;
        f.pos = pos.p;
        f.nrows = P.nq;
        f.K = K;
        f.L = L;
        f.eps2 = eps2;
        f.cover2 = cov2;
        f.out_ids = out_ids;
        f.out_dist = out_dist;
        f.out_kth = out_kth;
        f.out_status = out_status;
        f.bound2 = bound2;
        // big passes (at least a quarter of the points: the copy is N rows) gather rows in
        // join order once
        if (finalize_xj && P.nq >= (1u << 16) && 4 * P.nq >= N) {
            if (!lv.xj_ready) {
                lv.XJ.ensure((uint64_t)N * n);
                launch_rows_by(X64.p, lv.J.p, N, n, lv.XJ.p, s);
                lv.xj_ready = true;
            }
            f.XJ = lv.XJ.p;
        }
        // the finalize of launch rows [cr[c], cr[c+1]) (on s_out behind chunk c's join), on
        // a bounded grid so it shares the SMs with the next chunk's join; rows that go to
        // the host are taken in ascending output row (sorted per chunk on s_out)
        uint64_t maxlen = 0;
        for (size_t c = 0; c < nch; ++c) maxlen = std::max<uint64_t>(maxlen, cr[c + 1] - cr[c]);
        // (context buffers: a copy may still run on s_out after this pass returns)
        DBuf<uint32_t>& o_keys = st_keys;
        void* o_tmp = nullptr;
        size_t o_tmp_bytes = 0;
        if (to_host) {
            if (copy_pending) {  // an earlier pass's copy still owns the buffers
                KJ_CUDA(cudaStreamSynchronize(s_out));
                copy_pending = false;
            }
            o_keys.ensure(maxlen);
            KJ_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, o_tmp_bytes, P.qrow.p, o_keys.p,
                                                   (int64_t)maxlen, 0, bits_for(N), s));
            o_tmp = st_tmp.ensure(o_tmp_bytes);
        }
        // the finalize of launch rows [cr[c], cr[c+1]) into the device rows, then (to_host)
        // the chunk's rows to the host in ascending output row
        auto finalize_chunk = [&](size_t c, cudaStream_t st) {
            FinalArgs fc = f;
            fc.qpos = P.qpos.p + cr[c];
            fc.qrow = P.qrow.p + cr[c];
            fc.cnt = cnt.p + cr[c];
            fc.pos = pos.p + cr[c] * L;
            fc.nrows = cr[c + 1] - cr[c];
            if (st == s_out) KJ_CUDA(cudaStreamWaitEvent(s_out, ev_join[c], 0));
            launch_finalize(fc, st, st == s_out ? fin_blocks : 0);
            if (to_host && fc.nrows) {
                size_t bytes = o_tmp_bytes;
                KJ_CUDA(cub::DeviceRadixSort::SortKeys(o_tmp, bytes, P.qrow.p + cr[c], o_keys.p,
                                                       (int64_t)fc.nrows, 0, bits_for(N), st));
                launch_rows_to_host(o_keys.p, fc.nrows, K, out_ids, out_dist, host_ids, host_dist,
                                    st == s_out ? copy_blocks : 0, st);
            }
        };
        if (tc) {
            prep_tc(lv);
            TcJoinArgs a{};
            a.Bh = lv.Bh.p;
            a.row_halfs = lv.row_halfs;
            a.ksteps = tc_ksteps();
            a.n = n;
            a.qpos = P.qpos.p;
            a.items = P.items.p;
            a.adj = P.adj.p;
            DBuf<float> cut_scaled;
            if (d_init_cut) {
                const double S = tc_S();
                cut_scaled.ensure(nv);
                launch_scale_f32(d_init_cut, nv, (float)(1.0 / (S * S)), cut_scaled.p, s);
                a.init_cut = cut_scaled.p;
            }
            a.K = K;
            a.L = L;
            a.out_cnt = cnt.p;
            a.out_pos = pos.p;
            a.delta = f32_round_up(tc_delta());
            static const bool want_stats = getenv("KNNJ_JOIN_STATS") != nullptr;
            DBuf<unsigned long long> st;
            if (want_stats) {
                st.ensure(24);
                KJ_CUDA(cudaMemsetAsync(st.p, 0, 24 * 8, s));
                a.stats = st.p;
            }
            trace().mark("pass: pre-kernel", s);
            Timer t(s);
            for (size_t c = 0; c < nch; ++c) {
                TcJoinArgs ac = a;
                ac.items = P.items.p + ci[c];
                launch_join_tc(ac, tcc.sh, ci[c + 1] - ci[c], N, s);
                if (overlap) {
                    KJ_CUDA(cudaEventRecord(ev_join[c], s));
                    finalize_chunk(c, s_out);
                }
            }
            last_join_kernel_ms = t.ms();
            if (want_stats) {
                unsigned long long h[24];
                KJ_CUDA(cudaMemcpyAsync(h, st.p, 24 * 8, cudaMemcpyDeviceToHost, s));
                KJ_CUDA(cudaStreamSynchronize(s));
                fprintf(stderr, "join stats: items %llu rows %llu slabs %llu rare %llu bits %llu inserts %llu compactions %llu ms %.1f\n",
                        (unsigned long long)P.nitems, (unsigned long long)nv, h[0], h[1], h[2], h[3], h[4], last_join_kernel_ms);
                if (h[23])  // -DKNNJ_TC_CLOCKS builds: cycles per role phase
                    fprintf(stderr, "join clocks: epi warps %llu | epi accf-wait %llu ld64 %llu fast %llu rare %llu (compact %llu insert %llu) loop %llu prologue %llu total %llu | producer empty-wait %llu total %llu | mma full-wait %llu acce-wait %llu total %llu\n",
                            h[23], h[8], h[9], h[10], h[11], h[13], h[14], h[12], h[19], h[20], h[16], h[21], h[17], h[18], h[22]);
            }
            last_join_tc = true;
        } else if (mixed) {
            // per-item screen bound and eligibility, then the two kernels over their items
            DBuf<float> dlt, tc_dlt;
            DBuf<uint8_t> okf;
            DBuf<uint4> part;
            dlt.ensure(P.nitems);
            tc_dlt.ensure(P.nitems);
            okf.ensure(P.nitems);
            part.ensure(P.nitems);
            double A = 0, B = 0, C = 0;
            tc_delta_poly(A, B, C);
            const double S = tc_S(), ws = lv.prec_w / S;
            launch_item_delta(P.items.p, P.item_r2.p, P.nitems, 1.0 / (S * S), A, B, C,
                              0.02 * ws * ws, item_tc_min_q, dlt.p, okf.p, s);
            d_u64a.ensure(2);
            size_t bytes = 0;
            KJ_CUDA(cub::DevicePartition::Flagged(nullptr, bytes, P.items.p, okf.p, part.p, d_u64a.p,
                                                  (int64_t)P.nitems, s));
            KJ_CUDA(cub::DevicePartition::Flagged(sc.get(bytes), bytes, P.items.p, okf.p, part.p,
                                                  d_u64a.p, (int64_t)P.nitems, s));
            bytes = 0;
            KJ_CUDA(cub::DeviceSelect::Flagged(nullptr, bytes, dlt.p, okf.p, tc_dlt.p, d_u64a.p + 1,
                                               (int64_t)P.nitems, s));
            KJ_CUDA(cub::DeviceSelect::Flagged(sc.get(bytes), bytes, dlt.p, okf.p, tc_dlt.p,
                                               d_u64a.p + 1, (int64_t)P.nitems, s));
            unsigned long long ntc = 0;
            KJ_CUDA(cudaMemcpyAsync(&ntc, d_u64a.p, 8, cudaMemcpyDeviceToHost, s));
            sync();
            last_mixed_tc_items = ntc;
            Timer t(s);
            if (ntc) {
                prep_tc(lv);
                TcJoinArgs a{};
                a.Bh = lv.Bh.p;
                a.row_halfs = lv.row_halfs;
                a.ksteps = tc_ksteps();
                a.n = n;
                a.qpos = P.qpos.p;
                a.items = part.p;
                a.adj = P.adj.p;
                DBuf<float> cut_scaled;
                if (d_init_cut) {
                    const double S2 = S * S;
                    cut_scaled.ensure(nv);
                    launch_scale_f32(d_init_cut, nv, (float)(1.0 / S2), cut_scaled.p, s);
                    a.init_cut = cut_scaled.p;
                }
                a.K = K;
                a.L = L;
                a.out_cnt = cnt.p;
                a.out_pos = pos.p;
                a.delta = f32_round_up(tc_delta());
                a.item_delta = tc_dlt.p;
                static const bool want_stats = getenv("KNNJ_JOIN_STATS") != nullptr;
                DBuf<unsigned long long> st;
                if (want_stats) {
                    st.ensure(24);
                    KJ_CUDA(cudaMemsetAsync(st.p, 0, 24 * 8, s));
                    a.stats = st.p;
                }
                Timer tt(s);
                launch_join_tc(a, tcc.sh, ntc, N, s);
                mixed_tc_ran = true;
                if (want_stats) {
                    const double ms_tc = tt.ms();
                    unsigned long long h[8];
                    KJ_CUDA(cudaMemcpyAsync(h, st.p, 64, cudaMemcpyDeviceToHost, s));
                    sync();
                    fprintf(stderr, "mixed tc part: items %llu slabs %llu rare %llu bits %llu inserts %llu compactions %llu ms %.1f\n",
                            ntc, h[0], h[1], h[2], h[3], h[4], ms_tc);
                }
            }
            if (ntc < P.nitems) {
                // SIMT items: those of at most 32 queries on 32-thread blocks, the rest on 128
                const uint64_t nsimt = P.nitems - ntc;
                DBuf<uint4> part2;
                part2.ensure(nsimt);
                size_t b2 = 0;
                KJ_CUDA(cub::DevicePartition::If(nullptr, b2, part.p + ntc, part2.p, d_u64a.p, (int64_t)nsimt,
                                                 SmallItem{}, s));
                KJ_CUDA(cub::DevicePartition::If(sc.get(b2), b2, part.p + ntc, part2.p, d_u64a.p,
                                                 (int64_t)nsimt, SmallItem{}, s));
                unsigned long long nsmall = 0;
                KJ_CUDA(cudaMemcpyAsync(&nsmall, d_u64a.p, 8, cudaMemcpyDeviceToHost, s));
                sync();
                JoinArgs a{};
                if (!lv.xs_ready) {
                    lv.Xs.ensure((uint64_t)n * Npad);
                    launch_gather_x64(X64.p, d_g.p, lv.J.p, N, n, Npad, lv.Xs.p, s);
                    lv.xs_ready = true;
                }
                a.Xs = lv.Xs.p;
                a.Npad = Npad;
                a.n = n;
                a.qpos = P.qpos.p;
                a.adj = P.adj.p;
                a.init_cut = d_init_cut;
                a.K = K;
                a.L = L;
                a.out_cnt = cnt.p;
                a.out_pos = pos.p;
                screen_consts(a.gam, a.erg, a.eab, a.e64);
                a.items = part2.p;
                if (nsmall) launch_join(a, nsmall, 32u, s);
                a.items = part2.p + nsmall;
                if (nsimt > nsmall) launch_join(a, nsimt - nsmall, P.chunk, s);
            }
            last_join_kernel_ms = t.ms();
            last_join_tc = mixed_tc_ran;
        } else {
            JoinArgs a{};
            if (!lv.xs_ready) {
                lv.Xs.ensure((uint64_t)n * Npad);
                launch_gather_x64(X64.p, d_g.p, lv.J.p, N, n, Npad, lv.Xs.p, s);
                lv.xs_ready = true;
            }
            a.Xs = lv.Xs.p;
            a.Npad = Npad;
            a.n = n;
            a.qpos = P.qpos.p;
            a.items = P.items.p;
            a.adj = P.adj.p;
            a.init_cut = d_init_cut;
            a.K = K;
            a.L = L;
            a.out_cnt = cnt.p;
            a.out_pos = pos.p;
            screen_consts(a.gam, a.erg, a.eab, a.e64);
            Timer t(s);
            for (size_t c = 0; c < nch; ++c) {
                JoinArgs ac = a;
                ac.items = P.items.p + ci[c];
                launch_join(ac, ci[c + 1] - ci[c], P.chunk, s);
                if (overlap) {
                    KJ_CUDA(cudaEventRecord(ev_join[c], s));
                    finalize_chunk(c, s_out);
                }
            }
            last_join_kernel_ms = t.ms();
            last_join_tc = false;
        }
        if (getenv("KNNJ_JOIN_STATS"))
            fprintf(stderr, "pass: tc %d mixed %d (tc items %llu) chunk %u items %llu rows %llu cand %llu screened %llu w %.6g cover2 %.6g K %u L %u ms %.1f\n",
                    (int)tc, (int)mixed, (unsigned long long)(mixed ? last_mixed_tc_items : 0), P.chunk, (unsigned long long)P.nitems, (unsigned long long)nv,
                    (unsigned long long)P.candidates, (unsigned long long)P.screened, lv.w, cov2, K, L,
                    last_join_kernel_ms);
        trace().mark("pass: join kernel", s);
        if (overlap) {  // the chunks' finalizes ran on s_out; s continues after the last one
            KJ_CUDA(cudaEventRecord(ev_fin, s_out));
            KJ_CUDA(cudaStreamWaitEvent(s, ev_fin, 0));
        } else if (to_host) {
            // one launch: the device finalize on s, then the sorted row copy on s_out so
            // it overlaps whatever follows (the fallback); run_impl waits before patching
            launch_finalize(f, s);
            ensure_out_stream();
            KJ_CUDA(cudaEventRecord(ev_out, s));
            KJ_CUDA(cudaStreamWaitEvent(s_out, ev_out, 0));
            size_t bytes = o_tmp_bytes;
            KJ_CUDA(cub::DeviceRadixSort::SortKeys(o_tmp, bytes, P.qrow.p, o_keys.p, (int64_t)P.nq, 0,
                                                   bits_for(N), s_out));
            launch_rows_to_host(o_keys.p, P.nq, K, out_ids, out_dist, host_ids, host_dist, copy_blocks,
                                s_out);
            if (!ev_copy) KJ_CUDA(cudaEventCreateWithFlags(&ev_copy, cudaEventDisableTiming));
            KJ_CUDA(cudaEventRecord(ev_copy, s_out));
            copy_pending = true;
        } else {
            launch_finalize(f, s);
        }
        // split-part rows: finalized into their own exact top-K (with sq), merged below
        DBuf<uint32_t> t_ids, t_cnt, v_iota;
        DBuf<double> t_dist, t_sq, t_kth;
        DBuf<uint8_t> t_st;
        if (nvv) {
            t_ids.ensure(nvv * K);
            t_dist.ensure(nvv * K);
            t_sq.ensure(nvv * K);
            t_kth.ensure(nvv);
            t_st.ensure(nvv);
            t_cnt.ensure(nvv);
            v_iota.ensure(nvv);
            launch_iota(v_iota.p, nvv, s);
            FinalArgs fv = f;
            fv.qpos = P.qpos.p + P.nq;
            fv.qrow = v_iota.p;
            fv.cnt = cnt.p + P.nq;
            fv.pos = pos.p + P.nq * L;
            fv.nrows = nvv;
            fv.out_ids = t_ids.p;
            fv.out_dist = t_dist.p;
            fv.out_kth = t_kth.p;
            fv.out_status = t_st.p;
            fv.out_sq = t_sq.p;
            fv.out_count = t_cnt.p;
            launch_finalize(fv, s);
        }
        trace().mark("pass: finalize", s);
        // overflowed rows -> exact slow path on the same candidate sets (rows found on device)
        DBuf<uint32_t> row_item;
        bool have_row_item = false;
        auto slow_range = [&](uint64_t r0, uint64_t nr, const uint32_t* qrow, uint32_t* o_ids,
                              double* o_dist, double* o_kth, uint8_t* o_st, double* o_sq,
                              uint32_t* o_cnt) {
            if (!nr) return;
            DBuf<uint32_t> d_rows;
            d_rows.ensure(nr);
            d_u64b.ensure(1);
            KJ_CUDA(cudaMemsetAsync(d_u64b.p, 0, 8, s));
            launch_find_ovf(cnt.p + r0, nr, d_rows.p, d_u64b.p, s);
            unsigned long long novf = 0;
            KJ_CUDA(cudaMemcpyAsync(&novf, d_u64b.p, 8, cudaMemcpyDeviceToHost, s));
            sync();
            if (n_slow) *n_slow += novf;
            if (!novf) return;
            if (!have_row_item) {
                row_item.ensure(nv);
                launch_row_item(P.items.p, P.nitems, row_item.p, s);
                have_row_item = true;
            }
            launch_slow_exact(X64.p, n, lv.J.p, P.qpos.p + r0, qrow, d_rows.p, novf, P.items.p,
                              row_item.p + r0, P.adj.p, K, eps2, cov2, o_ids, o_dist, o_kth,
                              o_st, o_sq, o_cnt, s);
            if (to_host && host_patch && r0 == 0) {  // these rows reach the host by the patch
                DBuf<uint32_t> orow;
                orow.ensure(novf);
                launch_map_u32(d_rows.p, qrow, novf, orow.p, s);
                const size_t at = host_patch->size();
                host_patch->resize(at + novf);
                KJ_CUDA(cudaMemcpyAsync(host_patch->data() + at, orow.p, 4 * novf, cudaMemcpyDeviceToHost, s));
            }
            sync();
        };
        // (a bounded pass marks overflowed rows ST_MISS: they are re-run unbounded)
        if (bound2 <= 0.0)
            slow_range(0, P.nq, P.qrow.p, out_ids, out_dist, out_kth, out_status, nullptr, nullptr);
        if (nvv) {
            slow_range(P.nq, nvv, v_iota.p, t_ids.p, t_dist.p, t_kth.p, t_st.p, t_sq.p, t_cnt.p);
            launch_merge_parts(P.splits.p, P.nsplits, K, t_ids.p, t_sq.p, t_cnt.p, P.qrow.p, eps2,
                               cov2, out_ids, out_dist, out_kth, out_status, s);
        }
        trace().mark("pass: ovf + merge", s);
        return to_host;
    }

    // Exact KNN for the given queries (pids + rows), certified globally: level
    // passes at widths w0*2^L, each seeded with the previous upper bound.
    // U (per row, may be inf) = known upper bound of the K-th sq.
    // Level-0 join through the fine cascade: the pass's rows are first joined on grids of
    // width eps * f (f < 1). A row whose K-th exact distance there is below the fine cell
    // width (ST_CERT) already has its exact top-K, and that K-th is below eps, so it is a
    // dense success too (ST_IN_EPS): the outcome level 0 would give, over a neighbourhood
    // (3f)^m times the size. Only the remaining rows run the level-0 pass.
    void fine_cascade(uint32_t m, double eps, const Pass& P, uint32_t K, const uint8_t* d_dense,
                      uint32_t* out_ids, double* out_dist, double* out_kth, uint8_t* out_status,
                      uint64_t* n_slow, knnj_run_info& I) {
        uint64_t nrem = P.nq;
        DBuf<uint32_t> rows, pids, rows2, pids2;
        rows.ensure(nrem);
        pids.ensure(nrem);
        if (nrem) {
            KJ_CUDA(cudaMemcpyAsync(rows.p, P.qrow.p, 4 * nrem, cudaMemcpyDeviceToDevice, s));
            launch_map_u32(P.qpos.p, levels[0].J.p, nrem, pids.p, s);
        }
        double kernel_ms = 0.0;
        uint64_t screened = 0;
        for (int i = 0; i < 2 && nrem; ++i) {
            if (!fine_f[i]) continue;
            const int L = 40 + i;
            build_level(L, m, eps * double(fine_f[i]) / 1000.0);
            Level& lf = levels[L];
            Pass Pf;
            build_pass(lf, pids.p, rows.p, nrem, Pf, K, 0, 1, nullptr, filter_radius2(lf));
            run_pass(lf, Pf, K, nullptr, eps * eps, cover2(lf), out_ids, out_dist, out_kth,
                     out_status, n_slow);
            kernel_ms += last_join_kernel_ms;
            screened += Pf.screened;
            DBuf<uint8_t> flags;
            flags.ensure(nrem);
            launch_uncert_flags(rows.p, nrem, out_status, flags.p, s);
            rows2.ensure(nrem);
            pids2.ensure(nrem);
            d_u64a.ensure(1);
            size_t bytes = 0;
            KJ_CUDA(cub::DeviceSelect::Flagged(nullptr, bytes, rows.p, flags.p, rows2.p, d_u64a.p,
                                               (int64_t)nrem, s));
            KJ_CUDA(cub::DeviceSelect::Flagged(sc.get(bytes), bytes, rows.p, flags.p, rows2.p,
                                               d_u64a.p, (int64_t)nrem, s));
            KJ_CUDA(cub::DeviceSelect::Flagged(sc.get(bytes), bytes, pids.p, flags.p, pids2.p,
                                               d_u64a.p, (int64_t)nrem, s));
            unsigned long long left = 0;
            KJ_CUDA(cudaMemcpyAsync(&left, d_u64a.p, 8, cudaMemcpyDeviceToHost, s));
            sync();
            if (getenv("KNNJ_JOIN_STATS"))
                fprintf(stderr, "fine %u: %llu of %llu rows left\n", fine_f[i], left,
                        (unsigned long long)nrem);
            nrem = left;
            rows.swap(rows2);
            pids.swap(pids2);
        }
        if (nrem) {
            Level& lv0 = levels[0];
            Pass P0;
            build_pass(lv0, pids.p, rows.p, nrem, P0, K, 0, 1, d_dense, filter_radius2(lv0));
            run_pass(lv0, P0, K, nullptr, eps * eps, cover2(lv0), out_ids, out_dist, out_kth,
                     out_status, n_slow);
            kernel_ms += last_join_kernel_ms;
            screened += P0.screened;
        }
        I.ms_join_kernel = kernel_ms;
        I.join_screened_pairs = screened;
    }

    void exact_levels(uint32_t m, double w0, int first_level, std::vector<uint32_t> qpid,
                      std::vector<uint32_t> qrow, std::vector<double> U, uint32_t K,
                      uint32_t* out_ids, double* out_dist, double* out_kth, uint8_t* out_status,
                      uint64_t nrows_total, uint64_t* passes, uint64_t* n_slow) {
        // level for a row given its upper bound u and the last level tried
        auto level_for = [&](double u, int prev) {
            if (!(u < kInf)) return prev < first_level ? first_level : prev + 2;
            int L = std::max(first_level, prev + 1);
            while (L < 39) {
                const double w = std::ldexp(w0, L);
                if (w * w * (1.0 - 1e-6) > u) break;
                ++L;
            }
            return L;
        };
        std::vector<int> lvl(qpid.size());
        for (size_t i = 0; i < qpid.size(); ++i) lvl[i] = level_for(U[i], first_level - 1);
        DBuf<float> d_cut_by_row;  // only the current pass's rows are ever written / read
        d_cut_by_row.ensure(nrows_total);
        while (!qpid.empty()) {
            const int L = *std::min_element(lvl.begin(), lvl.end());
            if (L >= 40) throw Error(9, "exact fallback did not converge");
            std::vector<uint32_t> sp, sr, rp, rr;
            std::vector<float> scut;
            std::vector<double> ru;
            std::vector<int> rl;
            for (size_t i = 0; i < qpid.size(); ++i) {
                if (lvl[i] == L) {
                    sp.push_back(qpid[i]);
                    sr.push_back(qrow[i]);
                    scut.push_back(U[i] < kInf ? f32_round_up(U[i])
                                               : std::numeric_limits<float>::infinity());
                } else {
                    rp.push_back(qpid[i]);
                    rr.push_back(qrow[i]);
                    ru.push_back(U[i]);
                    rl.push_back(lvl[i]);
                }
            }
            Level& lv = levels[L];
            trace().mark("levels: select", s);
            build_level(L, m, std::ldexp(w0, L));
            trace().mark("levels: build_level", s);
            const double cov2 = cover2(lv);
            const uint64_t np = sp.size();
            DBuf<uint32_t> d_p, d_r;
            DBuf<float> d_cut;
            d_p.ensure(np);
            d_r.ensure(np);
            d_cut.ensure(np);
            KJ_CUDA(cudaMemcpyAsync(d_p.p, sp.data(), 4 * np, cudaMemcpyHostToDevice, s));
            KJ_CUDA(cudaMemcpyAsync(d_r.p, sr.data(), 4 * np, cudaMemcpyHostToDevice, s));
            d_cut.ensure(np);
            KJ_CUDA(cudaMemcpyAsync(d_cut.p, scut.data(), 4 * np, cudaMemcpyHostToDevice, s));
            launch_scatter_f32(d_r.p, d_cut.p, np, d_cut_by_row.p, s);
            Pass P;
            build_pass(lv, d_p.p, d_r.p, np, P, K, 0, 1, nullptr, filter_radius2(lv), true, false,
                       item_radius ? d_cut_by_row.p : nullptr, fallback_group_span);
            trace().mark("levels: build_pass", s);
            launch_gather_f32(P.qrow.p, d_cut_by_row.p, np, d_cut.p, s);
            run_pass(lv, P, K, d_cut.p, -1.0, cov2, out_ids, out_dist, out_kth, out_status, n_slow);
            if (passes) ++*passes;
            DBuf<uint8_t> g_st;
            DBuf<double> g_kth;
            g_st.ensure(np);
            g_kth.ensure(np);
            launch_gather_u8(d_r.p, out_status, np, g_st.p, s);
            launch_gather_f64(d_r.p, out_kth, np, g_kth.p, s);
            std::vector<uint8_t> st(np);
            std::vector<double> kth(np);
            KJ_CUDA(cudaMemcpyAsync(st.data(), g_st.p, np, cudaMemcpyDeviceToHost, s));
            KJ_CUDA(cudaMemcpyAsync(kth.data(), g_kth.p, 8 * np, cudaMemcpyDeviceToHost, s));
            sync();
            for (uint64_t i = 0; i < np; ++i) {
                if ((st[i] & ST_HAS_K) && (st[i] & ST_CERT)) continue;
                const double u = (st[i] & ST_HAS_K) ? kth[i] : kInf;
                rp.push_back(sp[i]);
                rr.push_back(sr[i]);
                ru.push_back(u);
                rl.push_back(level_for(u, L));
            }
            qpid.swap(rp);
            qrow.swap(rr);
            U.swap(ru);
            lvl.swap(rl);
        }
    }
};

// ============================================================================ C ABI
namespace {

template <class F>
int guarded(knnj_ctx* ctx, F&& f) {
    try {
        if (ctx) {
            KJ_CUDA(cudaSetDevice(ctx->dev));
            alloc_stream() = ctx->s;
            alloc_cache() = &ctx->cache;
        }
        f();
        return KNNJ_OK;
    } catch (const kj::Error& e) {
        if (ctx) ctx->err = e.what();
        return e.code;
    } catch (const std::exception& e) {
        if (ctx) ctx->err = e.what();
        return KNNJ_E_CUDA;
    }
}

void need_points(knnj_ctx* c) {
    if (!c->have_points) throw Error(1, "no dataset: call knnj_set_points first");
}

}  // namespace

extern "C" {

int knnj_abi_version(void) { return KNNJ_ABI_VERSION; }

int knnj_create(int device, knnj_ctx** out) {
    if (!out) return KNNJ_E_USAGE;
    try {
        auto c = std::make_unique<knnj_ctx>();
        c->dev = device;
        KJ_CUDA(cudaSetDevice(device));
        KJ_CUDA(cudaStreamCreateWithFlags(&c->s, cudaStreamNonBlocking));
        if (const char* e = std::getenv("KNNJ_NO_TC")) c->tc_enabled = !(e[0] && e[0] != '0');
        cudaMemPool_t pool;
        KJ_CUDA(cudaDeviceGetDefaultMemPool(&pool, device));
        uint64_t keep = ~0ull;  // keep freed blocks cached in the pool
        KJ_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep));
        *out = c.release();
        return KNNJ_OK;
    } catch (const kj::Error& e) {
        return e.code;
    } catch (...) {
        return KNNJ_E_CUDA;
    }
}

void knnj_destroy(knnj_ctx* ctx) {
    if (!ctx) return;
    cudaSetDevice(ctx->dev);
    alloc_stream() = ctx->s;
    alloc_cache() = &ctx->cache;
    cudaStreamSynchronize(ctx->s);
    cudaStream_t keep = ctx->s;
    ctx->s = nullptr;
    delete ctx;  // DBuf members hand their blocks back; the cache (destroyed last) frees them all
    alloc_cache() = nullptr;
    cudaStreamDestroy(keep);
}

const char* knnj_last_error(const knnj_ctx* ctx) { return ctx ? ctx->err.c_str() : "null ctx"; }

void* knnj_stream(knnj_ctx* ctx) { return ctx ? (void*)ctx->s : nullptr; }

// Test hook (knnj_c.h): one 128x128 tensor-core tile of level 0 — queries at sorted
// positions [q0,q0+128) against [c0,c0+128) — returns the raw FP32 accumulators and
// the FP16 operand rows used.
int knnj_debug_tc_tile(knnj_ctx* c, uint32_t q0, uint32_t c0, float* D, uint16_t* Bq,
                       uint16_t* Bc, double* scale_S, double* delta, uint32_t* pid_q,
                       uint32_t* pid_c) {
    return guarded(c, [&] {
        Level& lv = c->levels[0];
        if (!lv.built) throw Error(1, "no grid");
        c->prep_tc(lv);
        std::vector<uint32_t> qpos(128);
        for (int i = 0; i < 128; ++i) qpos[i] = q0 + i;
        uint4 item = make_uint4(0, 128, 0, 1);
        uint2 rng = make_uint2(c0, c0 + 128);
        DBuf<uint32_t> d_qpos, cnt, pos;
        DBuf<uint4> d_item;
        DBuf<uint2> d_adj;
        DBuf<float> d_dbg;
        d_qpos.ensure(128);
        d_item.ensure(1);
        d_adj.ensure(1);
        d_dbg.ensure(128 * 128);
        cnt.ensure(128);
        pos.ensure(128 * 12);
        KJ_CUDA(cudaMemcpyAsync(d_qpos.p, qpos.data(), 512, cudaMemcpyHostToDevice, c->s));
        KJ_CUDA(cudaMemcpyAsync(d_item.p, &item, 16, cudaMemcpyHostToDevice, c->s));
        KJ_CUDA(cudaMemcpyAsync(d_adj.p, &rng, 8, cudaMemcpyHostToDevice, c->s));
        TcJoinArgs a{};
        a.Bh = lv.Bh.p;
        a.row_halfs = lv.row_halfs;
        a.ksteps = c->tc_ksteps();
        a.n = c->n;
        a.qpos = d_qpos.p;
        a.items = d_item.p;
        a.adj = d_adj.p;
        a.K = 4;
        a.L = 12;
        a.out_cnt = cnt.p;
        a.out_pos = pos.p;
        a.delta = (float)c->tc_delta();
        a.dbg = d_dbg.p;
        launch_join_tc(a, lv.row_halfs == 64 ? TcShape{1, 2, 4} : TcShape{2, 1, 3}, 1, c->N, c->s);
        KJ_CUDA(cudaMemcpyAsync(D, d_dbg.p, 4 * 128 * 128, cudaMemcpyDeviceToHost, c->s));
        KJ_CUDA(cudaMemcpyAsync(Bq, lv.Bh.p + (uint64_t)q0 * lv.row_halfs, 2 * 128 * lv.row_halfs,
                                cudaMemcpyDeviceToHost, c->s));
        KJ_CUDA(cudaMemcpyAsync(Bc, lv.Bh.p + (uint64_t)c0 * lv.row_halfs, 2 * 128 * lv.row_halfs,
                                cudaMemcpyDeviceToHost, c->s));
        KJ_CUDA(cudaMemcpyAsync(pid_q, lv.J.p + q0, 4 * 128, cudaMemcpyDeviceToHost, c->s));
        KJ_CUDA(cudaMemcpyAsync(pid_c, lv.J.p + c0, 4 * 128, cudaMemcpyDeviceToHost, c->s));
        c->sync();
        *scale_S = c->tc_S();
        *delta = c->tc_delta();
    });
}

int knnj_set_option(knnj_ctx* c, const char* name, int64_t value) {
    return guarded(c, [&] {
        const std::string k = name ? name : "";
        if (k == "tensor_cores") {
            c->tc_enabled = value != 0;
        } else if (k == "box_filter") {
            c->box_filter = value != 0;
        } else if (k == "morton_dims" || k == "morton_bits") {
            if (value < 1 || value > 32) throw Error(1, k + " must be in [1, 32]");
            (k == "morton_dims" ? c->morton_dims : c->morton_bits) = (uint32_t)value;
            for (auto& lv : c->levels) lv.built = false;
            c->mm_lo.clear();
            c->hist_order_ready = false;
        } else if (k == "sweep_order") {
            c->sweep_order = value != 0;
        } else if (k == "pilot_cap") {
            if (value < 0 || value > 2) throw Error(1, "pilot_cap must be 0, 1 or 2");
            c->pilot_cap = (int)value;
        } else if (k == "simt_slack") {
            if (value < 0 || value > 128) throw Error(1, "simt_slack must be in [0, 128]");
            c->simt_slack = (uint32_t)value;
        } else if (k == "early_d2h") {
            c->early_d2h = value != 0;
        } else if (k == "stream_host") {
            c->stream_host = value != 0;
        } else if (k == "chunk_min_rows") {
            if (value < 1 || value > (1 << 30)) throw Error(1, "chunk_min_rows must be in [1, 2^30]");
            c->chunk_min_rows = (uint32_t)value;
        } else if (k == "kth_bound") {
            c->kth_bound = value != 0;
        } else if (k == "bound_grid") {
            c->bound_grid = value != 0;
        } else if (k == "fallback_group_span") {
            if (value < 0 || value > 64) throw Error(1, "fallback_group_span must be in [0, 64]");
            c->fallback_group_span = (uint32_t)value;
        } else if (k == "level0_group_span") {
            if (value < 0 || value > 64) throw Error(1, "level0_group_span must be in [0, 64]");
            c->level0_group_span = (uint32_t)value;
        } else if (k == "bound_group_span") {
            if (value < 1 || value > 64) throw Error(1, "bound_group_span must be in [1, 64]");
            c->bound_group_span = (uint32_t)value;
        } else if (k == "kth_bound_q") {
            if (value < 1 || value > 1000) throw Error(1, "kth_bound_q must be in [1, 1000] per mille");
            c->kth_bound_q = (uint32_t)value;
        } else if (k == "bound_min_rows") {
            if (value < 0) throw Error(1, "bound_min_rows must be >= 0");
            c->bound_min_rows = (uint64_t)value;
        } else if (k == "bound_cells") {
            if (value < 1 || value > (1 << 20)) throw Error(1, "bound_cells must be in [1, 2^20]");
            c->bound_cells = (uint32_t)value;
        } else if (k == "bound_sample") {
            if (value < 16 || value > (1 << 20)) throw Error(1, "bound_sample must be in [16, 2^20]");
            c->bound_sample = (uint32_t)value;
        } else if (k == "item_radius") {
            c->item_radius = value != 0;
        } else if (k == "tc_small_cta") {
            if (value < 0 || value > 2) throw Error(1, "tc_small_cta must be 0, 1 or 2");
            c->tc_small_cta = (int)value;
        } else if (k == "filter_skip_all_dims") {
            c->filter_skip_all_dims = value != 0;
        } else if (k == "chunk_device_out") {
            c->chunk_device_out = value != 0;
        } else if (k == "adj_norm_order") {
            c->adj_norm_order = value != 0;
        } else if (k == "tc_item_halves") {
            c->tc_item_halves = value != 0;
        } else if (k == "item_tc") {
            c->item_tc = value != 0;
        } else if (k == "item_tc_min_q") {
            if (value < 1 || value > 128) throw Error(1, "item_tc_min_q must be in [1, 128]");
            c->item_tc_min_q = (uint32_t)value;
        } else if (k == "out_priority") {
            c->out_priority = value != 0;
            if (c->s_out) {  // recreated with the new priority on next use
                KJ_CUDA(cudaStreamSynchronize(c->s_out));
                KJ_CUDA(cudaStreamDestroy(c->s_out));
                KJ_CUDA(cudaEventDestroy(c->ev_out));
                c->s_out = nullptr;
                c->ev_out = nullptr;
            }
        } else if (k == "copy_blocks") {
            if (value < 0 || value > (1 << 24)) throw Error(1, "copy_blocks must be in [0, 2^24]");
            c->copy_blocks = (uint32_t)value;
        } else if (k == "fin_blocks") {
            if (value < 0 || value > (1 << 24)) throw Error(1, "fin_blocks must be in [0, 2^24]");
            c->fin_blocks = (uint32_t)value;
        } else if (k == "join_chunks") {
            if (value < 1 || value > 64) throw Error(1, "join_chunks must be in [1, 64]");
            c->join_chunks = (uint32_t)value;
        } else if (k == "finalize_xj") {
            c->finalize_xj = value != 0;
        } else if (k == "tc_slack") {
            if (value < 8 || value > 96) throw Error(1, "tc_slack must be in [8, 96]");
            c->tc_slack = (uint32_t)value;
        } else if (k == "fine" || k == "fine2") {
            if (value < 0 || value >= 1000) throw Error(1, "fine width must be in [0, 1000) permille of eps");
            c->fine_f[k == "fine" ? 0 : 1] = (uint32_t)value;
        } else if (k == "hist_grid") {
            if (value < 0 || value > 2) throw Error(1, "hist_grid must be 0, 1 or 2");
            c->hist_grid = (int)value;
        } else if (k == "split_items") {
            c->split_items = value != 0;
        } else if (k == "hist_cap") {
            if (value < 0 || value > 2) throw Error(1, "hist_cap must be 0, 1 or 2");
            c->hist_cap_mode = (int)value;
        } else {
            throw Error(1, "unknown option '" + k + "'");
        }
    });
}

int knnj_fp32_peak(knnj_ctx* c, double* tflops) {
    return guarded(c, [&] { *tflops = kj::measure_ffma_tflops(c->s); });
}

void* knnj_alloc_pinned(size_t bytes) {
    void* p = nullptr;
    if (cudaHostAlloc(&p, bytes ? bytes : 1, cudaHostAllocPortable) != cudaSuccess) return nullptr;
    return p;
}
void knnj_free_pinned(void* p) {
    if (p) cudaFreeHost(p);
}

int knnj_set_points(knnj_ctx* c, const double* X, uint64_t N, uint32_t n) {
    return guarded(c, [&] {
        if (N < 1) throw Error(1, "dataset must contain at least one point");
        if (n < 1) throw Error(1, "dataset must have at least one dimension");
        if (N >= (1ull << 32) - 1) throw Error(1, "dataset too large for 32-bit point ids");
        c->N = N;
        c->n = n;
        c->have_points = c->working_ready = false;
        c->bh_id_ready = false;
        c->hist_order_ready = false;
        for (auto& lv : c->levels) lv.built = false;
        c->X0.ensure(N * n);
        KJ_CUDA(cudaMemcpyAsync(c->X0.p, X, N * n * 8, cudaMemcpyHostToDevice, c->s));
        c->d_u64a.ensure(1);
        unsigned long long none = ~0ull;
        KJ_CUDA(cudaMemcpyAsync(c->d_u64a.p, &none, 8, cudaMemcpyHostToDevice, c->s));
        launch_check_finite(c->X0.p, N * n, c->d_u64a.p, c->s);
        unsigned long long bad = 0;
        KJ_CUDA(cudaMemcpyAsync(&bad, c->d_u64a.p, 8, cudaMemcpyDeviceToHost, c->s));
        c->sync();
        if (bad != ~0ull)
            throw Error(1, "non-finite coordinate at point " + std::to_string(bad / n) +
                               ", dimension " + std::to_string(bad % n));
        c->have_points = true;
    });
}

int knnj_reorder_by_variance(knnj_ctx* c, uint32_t m, uint32_t* perm, double* var) {
    return guarded(c, [&] {
        need_points(c);
        c->reorder(m);
        if (perm) std::memcpy(perm, c->perm.data(), 4 * c->n);
        if (var) std::memcpy(var, c->var.data(), 8 * c->n);
    });
}

int knnj_get_points(knnj_ctx* c, double* out) {
    return guarded(c, [&] {
        need_points(c);
        c->ensure_working();
        KJ_CUDA(cudaMemcpyAsync(out, c->X64.p, c->N * c->n * 8, cudaMemcpyDeviceToHost, c->s));
        c->sync();
    });
}

int knnj_pair_sq(knnj_ctx* c, const uint64_t* ij, uint64_t np, double limit, double* out) {
    return guarded(c, [&] {
        need_points(c);
        c->ensure_working();
        for (uint64_t i = 0; i < 2 * np; ++i)
            if (ij[i] >= c->N) throw Error(1, "pair index out of range");
        auto v = c->pair_sq(ij, np, limit);
        std::memcpy(out, v.data(), 8 * np);
    });
}

int knnj_eps_mean(knnj_ctx* c, uint64_t pairs, uint64_t seed, double* out) {
    return guarded(c, [&] {
        need_points(c);
        c->ensure_working();
        *out = c->eps_mean(pairs, seed);
    });
}

int knnj_histogram(knnj_ctx* c, double em, uint32_t nb, double frac, uint64_t seed,
                   uint64_t* raw, uint64_t* qc) {
    return guarded(c, [&] {
        need_points(c);
        c->ensure_working();
        if (!(em > 0.0))
            throw Error(4, "mean pairwise distance is not positive; cannot build a distance histogram");
        if (nb < 2) throw Error(1, "histogram needs at least 2 bins");
        auto q = c->histogram_sample(frac, seed);
        std::fill(raw, raw + nb, 0ull);
        c->histogram_queries(q.data(), q.size(), em, nb, raw);
        *qc = q.size();
    });
}

int knnj_histogram_queries(knnj_ctx* c, const uint64_t* q, uint64_t nq, double em, uint32_t nb,
                           uint64_t* raw) {
    return guarded(c, [&] {
        need_points(c);
        c->ensure_working();
        for (uint64_t i = 0; i < nq; ++i)
            if (q[i] >= c->N) throw Error(1, "histogram query id out of range");
        c->histogram_queries(q, nq, em, nb, raw);
    });
}

int knnj_histogram_queries_capped(knnj_ctx* c, const uint64_t* q, uint64_t nq, double em,
                                  uint32_t nb, uint32_t ncount, uint64_t* raw) {
    return guarded(c, [&] {
        need_points(c);
        c->ensure_working();
        if (ncount < 1 || ncount > nb) throw Error(1, "n_count must be in [1, n_bins]");
        for (uint64_t i = 0; i < nq; ++i)
            if (q[i] >= c->N) throw Error(1, "histogram query id out of range");
        c->histogram_queries(q, nq, em, nb, raw, ncount);
    });
}

int knnj_grid_build(knnj_ctx* c, uint32_t m, double eps, knnj_grid_info* info) {
    return guarded(c, [&] {
        need_points(c);
        c->ensure_working();
        if (!(eps > 0.0)) throw Error(1, "grid eps must be positive");
        if (m < 1 || m > c->n) throw Error(1, "grid m must satisfy 1 <= m <= n");
        if (m > 64) throw Error(1, "grid m above 64 is not supported");
        c->grid_all_dims = m == c->n;
        c->build_level(0, m, eps);
        c->eps0 = eps;
        c->m0 = m;
        if (info) {
            std::memset(info, 0, sizeof(*info));
            const Level& lv = c->levels[0];
            info->m = m;
            info->eps = eps;
            info->n_cells = lv.ncells;
            for (uint32_t j = 0; j < m; ++j) {
                info->mins[j] = lv.mins[j];
                info->maxs[j] = lv.maxs[j];
                info->cells_per_dim[j] = lv.cpd[j];
            }
        }
    });
}

int knnj_grid_export(knnj_ctx* c, uint64_t* B, uint64_t* G, uint32_t* A, uint32_t* slot) {
    return guarded(c, [&] {
        const Level& lv = c->levels[0];
        if (!lv.built) throw Error(1, "no grid: call knnj_grid_build first");
        if (B) KJ_CUDA(cudaMemcpyAsync(B, lv.B.p, 8 * lv.ncells, cudaMemcpyDeviceToHost, c->s));
        if (G) {
            std::vector<uint2> g(lv.ncells);
            KJ_CUDA(cudaMemcpyAsync(g.data(), lv.G.p, 8 * lv.ncells, cudaMemcpyDeviceToHost, c->s));
            c->sync();
            for (uint64_t i = 0; i < lv.ncells; ++i) {
                G[2 * i] = g[i].x;
                G[2 * i + 1] = g[i].y;
            }
        }
        if (A) KJ_CUDA(cudaMemcpyAsync(A, lv.A.p, 4 * c->N, cudaMemcpyDeviceToHost, c->s));
        if (slot) KJ_CUDA(cudaMemcpyAsync(slot, lv.slot.p, 4 * c->N, cudaMemcpyDeviceToHost, c->s));
        c->sync();
    });
}

int knnj_range_count(knnj_ctx* c, const uint32_t* q, uint64_t nq, uint64_t* in_eps,
                     uint64_t* candidates) {
    return guarded(c, [&] {
        Level& lv = c->levels[0];
        if (!lv.built) throw Error(1, "no grid: call knnj_grid_build first");
        std::vector<uint32_t> rows(nq);
        std::iota(rows.begin(), rows.end(), 0u);
        DBuf<uint32_t> d_q, d_r;
        d_q.ensure(nq);
        d_r.ensure(nq);
        KJ_CUDA(cudaMemcpyAsync(d_q.p, q, 4 * nq, cudaMemcpyHostToDevice, c->s));
        KJ_CUDA(cudaMemcpyAsync(d_r.p, rows.data(), 4 * nq, cudaMemcpyHostToDevice, c->s));
        Pass P;
        c->build_pass(lv, d_q.p, d_r.p, nq, P);
        DBuf<unsigned long long> cnt;
        cnt.ensure(nq);
        launch_range_count(c->X64.p, c->n, lv.J.p, P.qpos.p, P.items.p, P.nitems, P.adj.p,
                           c->eps0 * c->eps0, cnt.p, c->s);
        std::vector<unsigned long long> h(nq);
        std::vector<uint32_t> prow(nq);
        std::vector<uint4> items(P.nitems);
        std::vector<uint2> adj(P.nadj);
        KJ_CUDA(cudaMemcpyAsync(h.data(), cnt.p, 8 * nq, cudaMemcpyDeviceToHost, c->s));
        KJ_CUDA(cudaMemcpyAsync(prow.data(), P.qrow.p, 4 * nq, cudaMemcpyDeviceToHost, c->s));
        KJ_CUDA(cudaMemcpyAsync(items.data(), P.items.p, 16 * P.nitems, cudaMemcpyDeviceToHost, c->s));
        KJ_CUDA(cudaMemcpyAsync(adj.data(), P.adj.p, 8 * P.nadj, cudaMemcpyDeviceToHost, c->s));
        c->sync();
        for (uint64_t r = 0; r < nq; ++r) in_eps[prow[r]] = h[r];
        if (candidates) {
            for (const uint4& it : items) {
                uint64_t cs = 0;
                for (uint32_t a = it.z; a < it.w; ++a) cs += adj[a].y - adj[a].x;
                for (uint32_t r = it.x; r < it.y; ++r) candidates[prow[r]] = cs;
            }
        }
    });
}

int knnj_split(knnj_ctx* c, const uint32_t* q, uint64_t nq, uint32_t k, double beta,
               double gamma, double rho, uint8_t* is_dense, uint64_t* cell_pop,
               knnj_split_info* info) {
    return guarded(c, [&] {
        Level& lv = c->levels[0];
        if (!lv.built) throw Error(1, "no grid: call knnj_grid_build first");
        if (beta < 0 || beta > 1 || gamma < 0 || gamma > 1 || rho < 0 || rho > 1)
            throw Error(1, "beta, gamma, rho must all be in [0, 1]");
        if (k < 1) throw Error(1, "compute_n_min requires k >= 1 and m >= 1");
        // partition.cpp:12-23 (Eq. 1), same expression order
        const double mm = double(lv.m);
        const double n_min =
            double(k) * std::pow(2.0, mm) * std::tgamma(mm / 2.0 + 1.0) / std::pow(M_PI, mm / 2.0);
        const double n_thresh = n_min + (10.0 * n_min - n_min) * gamma;
        DBuf<uint32_t> d_q, d_pop;
        d_q.ensure(nq);
        d_pop.ensure(nq);
        KJ_CUDA(cudaMemcpyAsync(d_q.p, q, 4 * nq, cudaMemcpyHostToDevice, c->s));
        launch_cell_pop(d_q.p, nq, lv.slot.p, lv.G.p, d_pop.p, c->s);
        std::vector<uint32_t> pop(nq);
        KJ_CUDA(cudaMemcpyAsync(pop.data(), d_pop.p, 4 * nq, cudaMemcpyDeviceToHost, c->s));
        c->sync();
        uint64_t ncpu = 0;
        for (uint64_t i = 0; i < nq; ++i) {
            is_dense[i] = double(pop[i]) >= n_thresh;
            ncpu += !is_dense[i];
            if (cell_pop) cell_pop[i] = pop[i];
        }
        uint64_t demoted = 0;
        const uint64_t floor_cpu = (uint64_t)std::ceil(rho * double(nq));
        if (ncpu < floor_cpu) {
            uint64_t need = floor_cpu - ncpu;
            std::vector<uint32_t> slot(nq);
            DBuf<uint32_t> d_slot;
            d_slot.ensure(nq);
            launch_map_u32(d_q.p, lv.slot.p, nq, d_slot.p, c->s);
            KJ_CUDA(cudaMemcpyAsync(slot.data(), d_slot.p, 4 * nq, cudaMemcpyDeviceToHost, c->s));
            c->sync();
            std::vector<std::tuple<uint32_t, uint32_t, uint32_t, uint64_t>> ord;  // pop, cell, pid, i
            for (uint64_t i = 0; i < nq; ++i)
                if (is_dense[i]) ord.emplace_back(pop[i], slot[i], q[i], i);
            std::sort(ord.begin(), ord.end());
            need = std::min<uint64_t>(need, ord.size());
            for (uint64_t i = 0; i < need; ++i) is_dense[std::get<3>(ord[i])] = 0;
            demoted = need;
            ncpu += need;
        }
        if (info) {
            info->n_min = n_min;
            info->n_thresh = n_thresh;
            info->q_cpu = ncpu;
            info->q_gpu = nq - ncpu;
            info->demoted = demoted;
        }
    });
}

int knnj_dense_join(knnj_ctx* c, const uint32_t* q, uint64_t nq, uint32_t k, uint32_t* ids,
                    double* dist, uint8_t* solved, knnj_join_stats* st) {
    return guarded(c, [&] {
        Level& lv = c->levels[0];
        if (!lv.built) throw Error(1, "no grid: call knnj_grid_build first");
        if (k < 1) throw Error(1, "k must be at least 1");
        std::vector<uint32_t> rows(nq);
        std::iota(rows.begin(), rows.end(), 0u);
        DBuf<uint32_t> d_q, d_r, o_ids;
        DBuf<double> o_dist, o_kth;
        DBuf<uint8_t> o_st;
        d_q.ensure(nq);
        d_r.ensure(nq);
        o_ids.ensure(nq * k);
        o_dist.ensure(nq * k);
        o_kth.ensure(nq);
        o_st.ensure(nq);
        KJ_CUDA(cudaMemcpyAsync(d_q.p, q, 4 * nq, cudaMemcpyHostToDevice, c->s));
        KJ_CUDA(cudaMemcpyAsync(d_r.p, rows.data(), 4 * nq, cudaMemcpyHostToDevice, c->s));
        Pass P;
        c->build_pass(lv, d_q.p, d_r.p, nq, P, k);
        uint64_t nslow = 0;
        c->run_pass(lv, P, k, nullptr, c->eps0 * c->eps0, c->cover2(lv), o_ids.p, o_dist.p,
                    o_kth.p, o_st.p, &nslow);
        std::vector<uint8_t> sts(nq);
        KJ_CUDA(cudaMemcpyAsync(ids, o_ids.p, 4 * nq * k, cudaMemcpyDeviceToHost, c->s));
        KJ_CUDA(cudaMemcpyAsync(dist, o_dist.p, 8 * nq * k, cudaMemcpyDeviceToHost, c->s));
        KJ_CUDA(cudaMemcpyAsync(sts.data(), o_st.p, nq, cudaMemcpyDeviceToHost, c->s));
        c->sync();
        uint64_t ns = 0;
        for (uint64_t i = 0; i < nq; ++i) {
            solved[i] = (sts[i] & ST_HAS_K) && (sts[i] & ST_IN_EPS);
            ns += solved[i];
            if (!solved[i]) {  // filter_keys discards a failed query's partial list
                std::fill(ids + i * k, ids + (i + 1) * k, 0xFFFFFFFFu);
                std::fill(dist + i * k, dist + (i + 1) * k, std::numeric_limits<double>::infinity());
            }
        }
        if (st) {
            st->candidates_examined = P.candidates;
            st->solved = ns;
            st->failed = nq - ns;
            st->kernel_ms = c->last_join_kernel_ms;
        }
    });
}

int knnj_exact_knn(knnj_ctx* c, const uint32_t* q, uint64_t nq, uint32_t k, uint32_t* ids,
                   double* dist) {
    return guarded(c, [&] {
        need_points(c);
        c->ensure_working();
        if (k < 1) throw Error(1, "knn_query requires k >= 1");
        if (k > c->N - 1) throw Error(1, "k exceeds |D|-1");
        for (uint64_t i = 0; i < nq; ++i)
            if (q[i] >= c->N) throw Error(1, "query id out of range");
        if (!nq) return;
        const uint32_t m = std::min<uint32_t>(6, c->n);
        // width: cells holding ~2k points on average over the bounding box
        std::vector<unsigned long long> mn(m), mx(m);
        c->d_u64a.ensure(64);
        c->d_u64b.ensure(64);
        std::vector<unsigned long long> i0(m, ~0ull), i1(m, 0ull);
        KJ_CUDA(cudaMemcpyAsync(c->d_u64a.p, i0.data(), 8 * m, cudaMemcpyHostToDevice, c->s));
        KJ_CUDA(cudaMemcpyAsync(c->d_u64b.p, i1.data(), 8 * m, cudaMemcpyHostToDevice, c->s));
        launch_minmax(c->X64.p, c->N, c->n, m, c->d_u64a.p, c->d_u64b.p, c->s);
        KJ_CUDA(cudaMemcpyAsync(mn.data(), c->d_u64a.p, 8 * m, cudaMemcpyDeviceToHost, c->s));
        KJ_CUDA(cudaMemcpyAsync(mx.data(), c->d_u64b.p, 8 * m, cudaMemcpyDeviceToHost, c->s));
        c->sync();
        double logvol = 0.0;
        int used = 0;
        for (uint32_t j = 0; j < m; ++j) {
            auto un = [](unsigned long long o) {
                unsigned long long b = (o & 0x8000000000000000ull) ? (o & 0x7FFFFFFFFFFFFFFFull) : ~o;
                double v;
                std::memcpy(&v, &b, 8);
                return v;
            };
            double e = un(mx[j]) - un(mn[j]);
            if (e > 0) {
                logvol += std::log(e);
                ++used;
            }
        }
        double w0 = used ? std::exp((logvol + std::log(2.0 * k / double(c->N))) / used) : 1.0;
        if (!(w0 > 0) || !std::isfinite(w0)) w0 = 1.0;
        DBuf<uint32_t> o_ids;
        DBuf<double> o_dist, o_kth;
        DBuf<uint8_t> o_st;
        o_ids.ensure(nq * k);
        o_dist.ensure(nq * k);
        o_kth.ensure(nq);
        o_st.ensure(nq);
        std::vector<uint32_t> qp(q, q + nq), rows(nq);
        std::iota(rows.begin(), rows.end(), 0u);
        std::vector<double> U(nq, kInf);
        // levels 30.. are reserved for this ad-hoc exact search (level 0.. belong to the eps grid)
        for (int L = 20; L < 40; ++L) c->levels[L].built = false;
        uint64_t passes = 0, slow = 0;
        // shift: level index L maps to width w0*2^(L-20)
        c->exact_levels(m, std::ldexp(w0, -20), 20, qp, rows, U, k, o_ids.p, o_dist.p, o_kth.p,
                        o_st.p, nq, &passes, &slow);
        KJ_CUDA(cudaMemcpyAsync(ids, o_ids.p, 4 * nq * k, cudaMemcpyDeviceToHost, c->s));
        KJ_CUDA(cudaMemcpyAsync(dist, o_dist.p, 8 * nq * k, cudaMemcpyDeviceToHost, c->s));
        c->sync();
    });
}

// run_hybrid (orchestrator.cpp:67-250), optionally as one shard of a multi-GPU run.
static void run_impl(knnj_ctx* c, const knnj_config* cfg, uint32_t shard, uint32_t nshard,
                     knnj_allreduce_fn allreduce, void* ar_user, uint32_t* ids, double* dist,
                     uint8_t* prov, uint32_t* owned, uint64_t* raw_hist, knnj_run_info* info) {
    need_points(c);
    knnj_run_info I;
    std::memset(&I, 0, sizeof(I));
    const uint64_t N = c->N;
    const uint32_t n = c->n;
    cudaStream_t s = c->s;
    // validate_config (orchestrator.cpp:16-31)
    if (cfg->k < 1) throw Error(1, "k must be at least 1");
    if (cfg->m > n) throw Error(1, "m must satisfy m <= n");
    if (cfg->beta < 0 || cfg->beta > 1 || cfg->gamma < 0 || cfg->gamma > 1 || cfg->rho < 0 ||
        cfg->rho > 1)
        throw Error(1, "beta, gamma, rho must all be in [0, 1]");
    if (!(cfg->hist_query_fraction > 0) || cfg->hist_query_fraction > 1)
        throw Error(1, "sample fractions must be in (0, 1]");
    if (cfg->n_bins < 2) throw Error(1, "n_bins must be at least 2");
    if (cfg->mode > 3) throw Error(1, "unknown engine mode");
    if (nshard < 1 || shard >= nshard) throw Error(1, "shard index must satisfy 0 <= shard < shard_count");
    if (nshard > 1 && !allreduce) throw Error(1, "a sharded run needs an allreduce callback");
    auto reduce = [&](uint64_t* buf, uint64_t count) {
        if (nshard > 1 && allreduce(buf, count, ar_user) != 0)
            throw Error(9, "allreduce callback failed");
    };
    // query ids ascending (make_query_list, orchestrator.cpp:33-44); all points: implicit iota
    std::vector<uint32_t> queries;
    if (cfg->query_subset) {
        for (uint64_t i = 0; i < cfg->n_query_subset; ++i)
            if (cfg->query_subset[i] >= N) throw Error(1, "query subset id out of range");
        queries.assign(cfg->query_subset, cfg->query_subset + cfg->n_query_subset);
        std::sort(queries.begin(), queries.end());
        queries.erase(std::unique(queries.begin(), queries.end()), queries.end());
    }
    const uint64_t nq = cfg->query_subset ? queries.size() : N;
    auto qid = [&](uint64_t i) -> uint32_t { return cfg->query_subset ? queries[i] : (uint32_t)i; };
    auto host_queries = [&]() -> const std::vector<uint32_t>& {
        if (queries.size() != nq) {
            queries.resize(nq);
            std::iota(queries.begin(), queries.end(), 0u);
        }
        return queries;
    };
    I.n_queries = nq;
    uint32_t k_eff = cfg->k;
    if (k_eff >= N) {
        k_eff = (uint32_t)(N - 1);
        I.k_clamped = 1;
    }
    I.k_effective = k_eff;
    const uint32_t m = cfg->m == 0 ? std::min<uint32_t>(6, n) : cfg->m;
    I.m_used = m;
    if (m > 64) throw Error(1, "grid m above 64 is not supported");

    Timer t_all(s);
    const unsigned long long launches0 = g_launches.load();
    const bool early_d2h = c->early_d2h;
    bool early_started = false;
    std::vector<uint32_t> fb_rows_host;  // rows the fallback rewrote (host ids)
    bool streamed = false;               // level-0 rows went to the host from the finalize
    uint32_t* h_ids_dev = nullptr;       // device views of the mapped host outputs
    double* h_dist_dev = nullptr;
    std::vector<uint32_t> patch_rows;    // rows rewritten after the streamed finalize
    struct OutSync {  // an early / streamed result copy never outlives the call (errors included)
        knnj_ctx* c;
        const bool& on;
        ~OutSync() {
            if ((on || c->copy_pending) && c->s_out) cudaStreamSynchronize(c->s_out);
            c->copy_pending = false;
        }
    } out_sync{c, early_started};
    // host-side reference RNG streams (pairs for eps_mean, the histogram's query sample)
    // drawn on a helper thread while the GPU reorders and orders the candidates
    const bool sampling = cfg->mode == KNNJ_HYBRID || cfg->mode == KNNJ_DENSE_ONLY;
    // (two independent streams: one thread each, so eps_mean waits only for its pairs)
    std::vector<uint64_t> eps_ij, hist_q;
    uint64_t* eps_pin = nullptr;  // pinned pairs (sampled case)
    uint64_t eps_pin_n = 0;
    std::thread drawer, hdrawer;
    if (sampling && N >= 2) {
        knnj_ctx::histogram_sample_size(N, cfg->hist_query_fraction);  // validates the fraction here
        const uint64_t pairs = std::min<uint64_t>(10 * N, cfg->eps_mean_pair_cap);
        uint64_t* pin = pairs < N * (N - 1) ? c->pinned_pairs(pairs) : nullptr;
        drawer = std::thread([&, pairs, pin] {
            if (pin) knnj_ctx::draw_pairs_into(N, pairs, derive_seed(cfg->seed, 1), pin);
            else eps_ij = knnj_ctx::draw_pairs(N, pairs, derive_seed(cfg->seed, 1));
        });
        eps_pin = pin;
        eps_pin_n = pin ? pairs : 0;
        hdrawer = std::thread([&] {
            const auto t0 = std::chrono::steady_clock::now();
            hist_q = c->draw_histogram_sample(cfg->hist_query_fraction, derive_seed(cfg->seed, 2));
            if (trace().on)
                std::fprintf(stderr, "[knnj] host: histogram sample %zu   %9.3f ms\n", hist_q.size(),
                             std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count());
        });
    }
    struct Joiner {
        std::thread& t;
        ~Joiner() {
            if (t.joinable()) t.join();
        }
    } joiner{drawer}, hjoiner{hdrawer};
    {
        Nvtx nv("knnj: reorder_by_variance");
        Timer t(s);
        c->reorder(m);
        I.ms_reorder = t.ms();
            trace().mark("run: reorder");
    }
    for (uint32_t j = 0; j < n && j < 1024; ++j) I.perm[j] = c->perm[j];
    if (k_eff == 0 || nq == 0) {
        // |D| == 1: every neighbour list is empty and every query keeps the reference's
        // initial Provenance::Sparse (orchestrator.cpp:72-97); shard 0 owns the rows
        const bool mine = shard == 0;
        I.n_owned = mine ? nq : 0;
        if (mine && prov) std::memset(prov, KNNJ_PROV_SPARSE, nq);
        if (mine && owned)
            for (uint64_t i = 0; i < nq; ++i) owned[i] = qid(i);
        I.ms_total = t_all.ms();
        if (info) *info = I;
        return;
    }
    const bool all_points = !cfg->query_subset;
    DBuf<uint32_t>& o_ids = c->r_ids;
    DBuf<double>& o_dist = c->r_dist;
    DBuf<double>& o_kth = c->r_kth;
    DBuf<uint8_t>& o_st = c->r_st;
    DBuf<uint8_t>& d_prov = c->r_prov;
    o_ids.ensure(nq * k_eff);
    o_dist.ensure(nq * k_eff);
    o_kth.ensure(nq);
    o_st.ensure(nq);
    d_prov.ensure(nq);
    DBuf<uint32_t>& d_q = c->r_q;
    DBuf<uint32_t>& d_rows = c->r_rows;
    d_q.ensure(nq);
    d_rows.ensure(nq);
    if (all_points) launch_iota(d_q.p, nq, s);
    else KJ_CUDA(cudaMemcpyAsync(d_q.p, queries.data(), 4 * nq, cudaMemcpyHostToDevice, s));
    if (all_points) {
        KJ_CUDA(cudaMemcpyAsync(d_rows.p, d_q.p, 4 * nq, cudaMemcpyDeviceToDevice, s));
    } else {
        launch_iota(d_rows.p, nq, s);
    }
    // rows this shard owns, in ascending row (= query id) order, on device
    DBuf<uint32_t> d_own;
    uint64_t n_own = 0;

    if (cfg->mode == KNNJ_BRUTE_ORACLE || cfg->mode == KNNJ_SPARSE_ONLY) {
        // brute_force_knn / kd-tree contract: exact KNN of every query (contiguous id slices)
        Timer t(s);
        const uint64_t lo = nq * shard / nshard, hi = nq * (shard + 1) / nshard;
        n_own = hi - lo;
        std::vector<uint32_t> rows(n_own), qp(n_own);
        std::iota(rows.begin(), rows.end(), (uint32_t)lo);
        for (uint64_t i = 0; i < n_own; ++i) qp[i] = qid(lo + i);
        const uint32_t me = std::min<uint32_t>(6, n);
        // width from the bounding box: cells holding ~2k points on average
        std::vector<unsigned long long> mn(me), mx(me), i0(me, ~0ull), i1(me, 0ull);
        c->d_u64a.ensure(64);
        c->d_u64b.ensure(64);
        KJ_CUDA(cudaMemcpyAsync(c->d_u64a.p, i0.data(), 8 * me, cudaMemcpyHostToDevice, s));
        KJ_CUDA(cudaMemcpyAsync(c->d_u64b.p, i1.data(), 8 * me, cudaMemcpyHostToDevice, s));
        launch_minmax(c->X64.p, N, n, me, c->d_u64a.p, c->d_u64b.p, s);
        KJ_CUDA(cudaMemcpyAsync(mn.data(), c->d_u64a.p, 8 * me, cudaMemcpyDeviceToHost, s));
        KJ_CUDA(cudaMemcpyAsync(mx.data(), c->d_u64b.p, 8 * me, cudaMemcpyDeviceToHost, s));
        c->sync();
        double logvol = 0.0;
        int used = 0;
        for (uint32_t j = 0; j < me; ++j) {
            const double e = knnj_ctx::unorder(mx[j]) - knnj_ctx::unorder(mn[j]);
            if (e > 0) {
                logvol += std::log(e);
                ++used;
            }
        }
        double w0 = used ? std::exp((logvol + std::log(2.0 * k_eff / double(N))) / used) : 1.0;
        if (!(w0 > 0) || !std::isfinite(w0)) w0 = 1.0;
        for (int L = 20; L < 40; ++L) c->levels[L].built = false;
        std::vector<double> U(n_own, kInf);
        if (n_own)
            c->exact_levels(me, std::ldexp(w0, -20), 20, qp, rows, U, k_eff, o_ids.p, o_dist.p,
                            o_kth.p, o_st.p, nq, &I.fallback_passes, &I.slow_path_queries);
        I.fallback_queries = n_own;
        I.ms_fallback = t.ms();
            trace().mark("run: fallback");
        if (n_own)
            KJ_CUDA(cudaMemsetAsync(d_prov.p + lo,
                                    cfg->mode == KNNJ_BRUTE_ORACLE ? KNNJ_PROV_DENSE : KNNJ_PROV_SPARSE,
                                    n_own, s));
        d_own.ensure(n_own);
        launch_iota(d_own.p, n_own, s);
        if (lo) {  // rows lo.. : shift the iota
            std::vector<uint32_t> r(n_own);
            std::iota(r.begin(), r.end(), (uint32_t)lo);
            KJ_CUDA(cudaMemcpyAsync(d_own.p, r.data(), 4 * n_own, cudaMemcpyHostToDevice, s));
        }
    } else {
        // ---- epsilon selection (orchestrator.cpp:137-165)
        {
            Nvtx nv("knnj: estimate_eps_mean");
            Timer t(s);
            if (N < 2) throw Error(1, "eps_mean estimation needs at least two points");
            // the tensor-core histogram's candidate order, built while the host draws the
            // pairs; not needed when the grid histogram will bin the capped rounds
            const bool grid_only = !raw_hist && c->grid_hist_applies(0, 1, cfg->n_bins);
            if (c->use_tc_hist() && !grid_only) c->ensure_hist_order(c->tc_row_halfs());
            if (drawer.joinable()) drawer.join();
            I.eps_mean = eps_pin ? c->eps_mean_of(eps_pin, eps_pin_n) : c->eps_mean_of(eps_ij);
            I.ms_eps_mean = t.ms();
            trace().mark("run: eps_mean");
        }
        const double target_beta =
            double(k_eff) + (100.0 * double(k_eff) - double(k_eff)) * cfg->beta;
        std::vector<uint64_t> raw(cfg->n_bins, 0);
        uint32_t valid = cfg->n_bins;
        {
            Nvtx nv("knnj: build_distance_histogram");
            Timer t(s);
            if (hdrawer.joinable()) hdrawer.join();
            auto& hq = hist_q;
            I.hist_query_count = hq.size();
            valid = c->hist_for_selection(hq, shard, nshard, I.eps_mean, cfg->n_bins, target_beta,
                                          raw_hist != nullptr, reduce, raw.data());
            I.hist_bins_counted = valid;
            I.ms_histogram = t.ms();
            trace().mark("run: histogram");
            I.ms_hist_kernel = c->last_hist_kernel_ms;
            I.hist_tensor_cores = c->last_hist_tc ? 1 : 0;
        }
        if (raw_hist) std::memcpy(raw_hist, raw.data(), 8 * cfg->n_bins);
        const double width = I.eps_mean / double(cfg->n_bins);
        I.bin_width = width;
        // cumulative profile over the exactly counted bins (all of them unless capped,
        // in which case the target is already reached inside them)
        std::vector<double> cum(valid);
        uint64_t running = 0;
        for (uint32_t b = 0; b < valid; ++b) {
            running += raw[b];
            cum[b] = double(running) / double(I.hist_query_count);
        }
        auto select = [&](double beta, bool& fell_back, uint64_t& bin_out) {
            const double target = double(k_eff) + (100.0 * double(k_eff) - double(k_eff)) * beta;
            auto it = std::lower_bound(cum.begin(), cum.end(), target);
            fell_back = false;
            if (it == cum.end()) {
                if (valid != cfg->n_bins) throw Error(9, "capped histogram missed its target");
                fell_back = true;
                it = std::lower_bound(cum.begin(), cum.end(), cum.back());
            }
            uint64_t bin = uint64_t(it - cum.begin()) + 1;
            double start = double(bin - 1) * width;
            double end = double(bin) * width;
            bin_out = bin;
            return (start + end) / 2.0;
        };
        bool fb = false, fb0 = false;
        uint64_t bin = 0, bin0 = 0;
        I.eps_beta = select(cfg->beta, fb, bin);
        I.eps_default = select(0.0, fb0, bin0);
        I.eps_final = 2.0 * I.eps_beta;
        I.eps_used = I.eps_final;
        I.eps_fallback = fb;
        I.hist_bin = bin;
        const double eps = I.eps_final;

        // ---- grid (GridIndex::build)
        {
            Nvtx nv("knnj: grid build");
            Timer t(s);
            c->grid_all_dims = m == c->n;
        c->build_level(0, m, eps);
            c->eps0 = eps;
            c->m0 = m;
            for (int L = 1; L < 40; ++L) c->levels[L].built = false;
            I.ms_grid = t.ms();
            trace().mark("run: grid");
            I.grid_cells = c->levels[0].ncells;
        }
        Level& lv0 = c->levels[0];
        // ---- split (partition.cpp:30-75): dense flags per query row, on device
        DBuf<uint8_t> d_dense;
        bool have_dense = false;
        {
            Nvtx nv("knnj: split_work");
            Timer t(s);
            const double mm = double(m);
            I.n_min = double(k_eff) * std::pow(2.0, mm) * std::tgamma(mm / 2.0 + 1.0) /
                      std::pow(M_PI, mm / 2.0);
            I.n_thresh = I.n_min + (10.0 * I.n_min - I.n_min) * cfg->gamma;
            if (cfg->mode == KNNJ_HYBRID) {
                have_dense = true;
                d_dense.ensure(nq);
                c->d_u64a.ensure(1);
                KJ_CUDA(cudaMemsetAsync(c->d_u64a.p, 0, 8, s));
                launch_split_flags(d_q.p, nq, lv0.slot.p, lv0.G.p, I.n_thresh, d_dense.p,
                                   c->d_u64a.p, s);
                unsigned long long ncpu = 0;
                KJ_CUDA(cudaMemcpyAsync(&ncpu, c->d_u64a.p, 8, cudaMemcpyDeviceToHost, s));
                c->sync();
                const uint64_t floor_cpu = (uint64_t)std::ceil(cfg->rho * double(nq));
                if (ncpu < floor_cpu) {
                    // rho demotion (pop, cell, pid order): the host reference path
                    std::vector<uint8_t> dense(nq);
                    knnj_split_info si{};
                    int rc = knnj_split(c, host_queries().data(), nq, k_eff, cfg->beta, cfg->gamma,
                                        cfg->rho, dense.data(), nullptr, &si);
                    if (rc) throw Error(rc, c->err);
                    alloc_stream() = s;
                    KJ_CUDA(cudaMemcpyAsync(d_dense.p, dense.data(), nq, cudaMemcpyHostToDevice, s));
                    I.q_cpu = si.q_cpu;
                    I.demoted = si.demoted;
                } else {
                    I.q_cpu = ncpu;
                }
                I.q_gpu = nq - I.q_cpu;
            } else {
                I.q_gpu = nq;
            }
            I.ms_split = t.ms();
            trace().mark("run: split");
        }
        // ---- level-0 fused join over this shard's queries (dense + sparse)
        uint64_t slow = 0;
        Pass P;
        {
            Nvtx nv("knnj: level-0 join + top-K");
            Timer t(s);
            const bool fine = c->fine_f[0] > 0 || c->fine_f[1] > 0;
            // Streamed results: host outputs in pinned memory are written by the finalize of
            // each launch chunk while the next chunk joins (rows the slow path or the
            // fallback rewrite later are patched at the end); otherwise one bulk copy.
            if (nshard == 1 && ids && dist && !fine && c->stream_host) {
                h_ids_dev = static_cast<uint32_t*>(mapped_host(ids, 4 * nq * k_eff));
                h_dist_dev = static_cast<double*>(mapped_host(dist, 8 * nq * k_eff));
                if (!h_ids_dev || !h_dist_dev) h_ids_dev = nullptr, h_dist_dev = nullptr;
            }
            // Radius bound (kth_bound): the K-th distance of a strided sample of the queries,
            // taken at the kth_bound_q quantile, bounds most rows' K-th. The pass then
            // screens only candidates within it (box filter and list cut); a row whose K-th
            // is not within it (ST_MISS) is re-run without the bound, so every row ends with
            // exactly the unbounded pass's result.
            const double filt0 = fine ? 0.0 : c->filter_radius2(lv0);
            double B2 = 0.0;
            if (!fine && filt0 > 0.0 && c->kth_bound && nq >= c->bound_min_rows) {
                std::vector<uint32_t> sq;
                if (all_points) {
                    sq = c->cell_sample(lv0, c->bound_cells, 256);
                } else {
                    sq.resize(c->bound_sample);
                    for (uint32_t i = 0; i < c->bound_sample; ++i)
                        sq[i] = qid((uint64_t)i * nq / c->bound_sample);
                }
                B2 = c->sample_kth_bound(lv0, sq, k_eff, eps * eps, c->kth_bound_q);
                if (!(B2 < c->bound_max_frac * filt0)) B2 = 0.0;
                else B2 = (double)f32_round_up(B2);
            }
            I.kth_bound2 = B2;
            // The bounded pass runs on a grid of width ~B (bound_grid): every candidate within
            // B of a query lies in its 3^m neighbourhood there, a (w0/B)^m times smaller
            // volume than level 0's; cell runs refill the work items. Level 0's own walk is
            // still built (unfiltered) for the reference's candidate counts.
            Level* lvb = &lv0;
            Pass P0;
            const double wf = std::sqrt(B2) * (1.0 + 1e-9);
            const bool fine_grid = B2 > 0.0 && c->bound_grid && wf < c->bound_grid_frac * lv0.w;
            {
                Timer tb(s);
                // chunked launches only pay for the streamed result copy (each chunk restarts
                // the LPT schedule: on skewed data the tails cost more than the finalize
                // overlap saves)
                c->stream_chunks = (nshard == 1 && !fine && (h_ids_dev || c->chunk_device_out))
                                    ? c->join_chunks : 1;
                if (fine_grid) {
                    c->build_level(43, m, wf);
                    lvb = &c->levels[43];
                    lvb->prec_w = lv0.w;  // the screen band is judged against level 0's cells
                    c->build_pass(*lvb, d_q.p, d_rows.p, nq, P, k_eff, shard, nshard,
                                  have_dense ? d_dense.p : nullptr, B2, false, all_points, nullptr,
                                  c->bound_group_span);
                    c->stream_chunks = 1;
                    c->build_pass(lv0, d_q.p, d_rows.p, nq, P0, k_eff, shard, nshard,
                                  have_dense ? d_dense.p : nullptr, 0.0, true, all_points);
                } else {
                    c->build_pass(lv0, d_q.p, d_rows.p, nq, P, k_eff, shard, nshard,
                                  have_dense ? d_dense.p : nullptr, B2 > 0.0 ? B2 : filt0, B2 <= 0.0,
                                  all_points, nullptr, c->level0_group_span);
                }
                c->stream_chunks = 1;
                I.ms_join_build = tb.ms();
            }
            if (!fine) {
                DBuf<float> d_cut;
                if (B2 > 0.0) {
                    d_cut.ensure(P.nq);
                    launch_fill_f32(d_cut.p, P.nq, (float)B2, s);
                }
                streamed = c->run_pass(*lvb, P, k_eff, B2 > 0.0 ? d_cut.p : nullptr, eps * eps,
                                       c->cover2(lv0), o_ids.p, o_dist.p, o_kth.p, o_st.p, &slow,
                                       h_ids_dev, h_dist_dev, &patch_rows, B2);
                I.ms_join_kernel = c->last_join_kernel_ms;
                I.join_screened_pairs = P.screened;
                I.join_tensor_cores = c->last_join_tc ? 1 : 0;  // the main pass, not the retries
                if (B2 > 0.0) {
                    // rows the bound missed: the unbounded level-0 pass over just those
                    DBuf<uint8_t> fl;
                    DBuf<uint32_t> mrows, mq;
                    fl.ensure(P.nq);
                    mrows.ensure(P.nq);
                    launch_miss_flags(P.qrow.p, P.nq, o_st.p, fl.p, s);
                    c->d_u64a.ensure(1);
                    size_t bytes = 0;
                    KJ_CUDA(cub::DeviceSelect::Flagged(nullptr, bytes, P.qrow.p, fl.p, mrows.p,
                                                       c->d_u64a.p, (int64_t)P.nq, s));
                    KJ_CUDA(cub::DeviceSelect::Flagged(c->sc.get(bytes), bytes, P.qrow.p, fl.p,
                                                       mrows.p, c->d_u64a.p, (int64_t)P.nq, s));
                    unsigned long long nmiss = 0;
                    KJ_CUDA(cudaMemcpyAsync(&nmiss, c->d_u64a.p, 8, cudaMemcpyDeviceToHost, s));
                    c->sync();
                    I.bound_retried = nmiss;
                    if (nmiss) {
                        mq.ensure(nmiss);
                        launch_map_u32(mrows.p, d_q.p, nmiss, mq.p, s);
                        Pass P2;
                        c->build_pass(lv0, mq.p, mrows.p, nmiss, P2, k_eff, 0, 1,
                                      have_dense ? d_dense.p : nullptr, filt0);
                        c->run_pass(lv0, P2, k_eff, nullptr, eps * eps, c->cover2(lv0), o_ids.p,
                                    o_dist.p, o_kth.p, o_st.p, &slow);
                        I.ms_join_kernel += c->last_join_kernel_ms;
                        I.join_screened_pairs += P2.screened;
                        if (streamed) {  // these host rows are patched at the end
                            const size_t at = patch_rows.size();
                            patch_rows.resize(at + nmiss);
                            KJ_CUDA(cudaMemcpyAsync(patch_rows.data() + at, mrows.p, 4 * nmiss,
                                                    cudaMemcpyDeviceToHost, s));
                            c->sync();
                        }
                    }
                }
            } else {
                c->fine_cascade(m, eps, P, k_eff, have_dense ? d_dense.p : nullptr, o_ids.p,
                                o_dist.p, o_kth.p, o_st.p, &slow, I);
            }
            I.ms_join = t.ms();
            trace().mark("run: join");
            if (fine) I.join_tensor_cores = c->last_join_tc ? 1 : 0;
            // candidates_examined counts dense queries only (DenseJoinStats), over level 0's walk
            const Pass& Pw = fine_grid ? P0 : P;
            I.candidates_examined = have_dense ? Pw.candidates_dense : Pw.candidates;
            I.join_candidate_pairs = Pw.candidates;
        }
        n_own = P.nq;
        // single-GPU runs with host outputs: copy every row now, on a second stream, while
        // classification and the fallback run; the few rows the fallback rewrites are
        // patched afterwards
        if (nshard == 1 && ids && dist && early_d2h && !streamed) {
            c->ensure_out_stream();
            KJ_CUDA(cudaEventRecord(c->ev_out, s));
            KJ_CUDA(cudaStreamWaitEvent(c->s_out, c->ev_out, 0));
            KJ_CUDA(cudaMemcpyAsync(ids, o_ids.p, 4 * nq * k_eff, cudaMemcpyDeviceToHost, c->s_out));
            KJ_CUDA(cudaMemcpyAsync(dist, o_dist.p, 8 * nq * k_eff, cudaMemcpyDeviceToHost, c->s_out));
            early_started = true;
        }
        // ---- classify on device; exact fallback for failures and uncertified sparse rows
        {
            Nvtx nv("knnj: classify + exact fallback");
            Timer t(s);
            DBuf<uint8_t> need;
            need.ensure(n_own);
            launch_classify(P.qrow.p, n_own, o_st.p, have_dense ? d_dense.p : nullptr, d_prov.p,
                            need.p, s);
            DBuf<uint32_t> fb_rows;
            fb_rows.ensure(n_own);
            c->d_u64a.ensure(1);
            {
                size_t bytes = 0;
                KJ_CUDA(cub::DeviceSelect::Flagged(nullptr, bytes, P.qrow.p, need.p, fb_rows.p,
                                                   c->d_u64a.p, (int64_t)n_own, s));
                KJ_CUDA(cub::DeviceSelect::Flagged(c->sc.get(bytes), bytes, P.qrow.p, need.p,
                                                   fb_rows.p, c->d_u64a.p, (int64_t)n_own, s));
            }
            unsigned long long nfb = 0;
            KJ_CUDA(cudaMemcpyAsync(&nfb, c->d_u64a.p, 8, cudaMemcpyDeviceToHost, s));
            c->sync();
            std::vector<uint32_t>& fr = fb_rows_host;
            fr.assign(nfb, 0u);
            std::vector<uint32_t> fp(nfb);
            std::vector<double> fu(nfb);
            if (nfb) {
                DBuf<uint8_t> g_st, g_pv;
                DBuf<double> g_kth;
                g_st.ensure(nfb);
                g_pv.ensure(nfb);
                g_kth.ensure(nfb);
                launch_gather_u8(fb_rows.p, o_st.p, nfb, g_st.p, s);
                launch_gather_u8(fb_rows.p, d_prov.p, nfb, g_pv.p, s);
                launch_gather_f64(fb_rows.p, o_kth.p, nfb, g_kth.p, s);
                std::vector<uint8_t> st(nfb), pv(nfb);
                KJ_CUDA(cudaMemcpyAsync(fr.data(), fb_rows.p, 4 * nfb, cudaMemcpyDeviceToHost, s));
                KJ_CUDA(cudaMemcpyAsync(st.data(), g_st.p, nfb, cudaMemcpyDeviceToHost, s));
                KJ_CUDA(cudaMemcpyAsync(pv.data(), g_pv.p, nfb, cudaMemcpyDeviceToHost, s));
                KJ_CUDA(cudaMemcpyAsync(fu.data(), g_kth.p, 8 * nfb, cudaMemcpyDeviceToHost, s));
                c->sync();
                for (uint64_t i = 0; i < nfb; ++i) {
                    fp[i] = qid(fr[i]);
                    if (!(st[i] & ST_HAS_K)) fu[i] = kInf;
                    if (pv[i] == KNNJ_PROV_DENSE_FAILED) ++I.failed_count;
                }
            }
            I.fallback_queries = nfb;
            if (nfb)
                c->exact_levels(m, eps, 1, fp, fr, fu, k_eff, o_ids.p, o_dist.p, o_kth.p, o_st.p,
                                nq, &I.fallback_passes, &slow);
            I.slow_path_queries = slow;
            I.ms_fallback = t.ms();
            trace().mark("run: fallback");
        }
        // owned rows in ascending order
        d_own.ensure(n_own);
        if (nshard == 1) {
            launch_iota(d_own.p, n_own, s);
        } else if (n_own) {
            DBuf<uint32_t> tmp;
            tmp.ensure(n_own);
            KJ_CUDA(cudaMemcpyAsync(tmp.p, P.qrow.p, 4 * n_own, cudaMemcpyDeviceToDevice, s));
            size_t bytes = 0;
            KJ_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, bytes, tmp.p, d_own.p, (int64_t)n_own,
                                                   0, bits_for(nq), s));
            KJ_CUDA(cub::DeviceRadixSort::SortKeys(c->sc.get(bytes), bytes, tmp.p, d_own.p,
                                                   (int64_t)n_own, 0, bits_for(nq), s));
        }
    }
    I.n_owned = n_own;
    // ---- results to the host: this shard's rows, ascending query id
    {
        Timer t(s);
        if (nshard == 1 && streamed) {
            if (c->copy_pending) {  // the level-0 row copy must land before the patch
                KJ_CUDA(cudaStreamWaitEvent(s, c->ev_copy, 0));
                c->copy_pending = false;
            }
            // the level-0 rows are on the host already; patch what was rewritten after
            std::vector<uint32_t>& pr = patch_rows;
            pr.insert(pr.end(), fb_rows_host.begin(), fb_rows_host.end());
            std::sort(pr.begin(), pr.end());
            pr.erase(std::unique(pr.begin(), pr.end()), pr.end());
            const uint64_t np = pr.size();
            if (np) {
                DBuf<uint32_t> d_pr;
                d_pr.ensure(np);
                KJ_CUDA(cudaMemcpyAsync(d_pr.p, pr.data(), 4 * np, cudaMemcpyHostToDevice, s));
                launch_scatter_rows(d_pr.p, np, k_eff, o_ids.p, o_dist.p, h_ids_dev, h_dist_dev, s);
            }
            if (prov) KJ_CUDA(cudaMemcpyAsync(prov, d_prov.p, nq, cudaMemcpyDeviceToHost, s));
            if (owned) std::memcpy(owned, host_queries().data(), 4 * nq);
            c->sync();
        } else if (nshard == 1 && early_started) {
            const uint64_t nfb = fb_rows_host.size();
            if (nfb > 65536) {  // many rewritten rows: copy everything again (after the early copy)
                KJ_CUDA(cudaStreamSynchronize(c->s_out));
                KJ_CUDA(cudaMemcpyAsync(ids, o_ids.p, 4 * nq * k_eff, cudaMemcpyDeviceToHost, s));
                KJ_CUDA(cudaMemcpyAsync(dist, o_dist.p, 8 * nq * k_eff, cudaMemcpyDeviceToHost, s));
            } else if (nfb) {
                DBuf<uint32_t> d_fr, c_ids;
                DBuf<double> c_dist;
                d_fr.ensure(nfb);
                c_ids.ensure(nfb * k_eff);
                c_dist.ensure(nfb * k_eff);
                KJ_CUDA(cudaMemcpyAsync(d_fr.p, fb_rows_host.data(), 4 * nfb, cudaMemcpyHostToDevice, s));
                launch_gather_rows(d_fr.p, nfb, k_eff, o_ids.p, o_dist.p, c_ids.p, c_dist.p, s);
                std::vector<uint32_t> h_ids(nfb * k_eff);
                std::vector<double> h_dist(nfb * k_eff);
                KJ_CUDA(cudaMemcpyAsync(h_ids.data(), c_ids.p, 4 * nfb * k_eff, cudaMemcpyDeviceToHost, s));
                KJ_CUDA(cudaMemcpyAsync(h_dist.data(), c_dist.p, 8 * nfb * k_eff, cudaMemcpyDeviceToHost, s));
                c->sync();
                KJ_CUDA(cudaStreamSynchronize(c->s_out));  // the bulk copy must land first
                for (uint64_t i = 0; i < nfb; ++i) {
                    const uint64_t r = fb_rows_host[i];
                    std::memcpy(ids + r * k_eff, h_ids.data() + i * k_eff, 4 * k_eff);
                    std::memcpy(dist + r * k_eff, h_dist.data() + i * k_eff, 8 * k_eff);
                }
            }
            KJ_CUDA(cudaStreamSynchronize(c->s_out));
            if (prov) KJ_CUDA(cudaMemcpyAsync(prov, d_prov.p, nq, cudaMemcpyDeviceToHost, s));
            if (owned) std::memcpy(owned, host_queries().data(), 4 * nq);
        } else if (nshard == 1) {
            if (ids) KJ_CUDA(cudaMemcpyAsync(ids, o_ids.p, 4 * nq * k_eff, cudaMemcpyDeviceToHost, s));
            if (dist) KJ_CUDA(cudaMemcpyAsync(dist, o_dist.p, 8 * nq * k_eff, cudaMemcpyDeviceToHost, s));
            if (prov) KJ_CUDA(cudaMemcpyAsync(prov, d_prov.p, nq, cudaMemcpyDeviceToHost, s));
            if (owned) std::memcpy(owned, host_queries().data(), 4 * nq);
        } else if (n_own) {
            DBuf<uint32_t> c_ids, c_q;
            DBuf<double> c_dist;
            DBuf<uint8_t> c_pv;
            if (ids || dist) {
                c_ids.ensure(n_own * k_eff);
                c_dist.ensure(n_own * k_eff);
                launch_gather_rows(d_own.p, n_own, k_eff, o_ids.p, o_dist.p, c_ids.p, c_dist.p, s);
                if (ids) KJ_CUDA(cudaMemcpyAsync(ids, c_ids.p, 4 * n_own * k_eff, cudaMemcpyDeviceToHost, s));
                if (dist) KJ_CUDA(cudaMemcpyAsync(dist, c_dist.p, 8 * n_own * k_eff, cudaMemcpyDeviceToHost, s));
            }
            if (prov) {
                c_pv.ensure(n_own);
                launch_gather_u8(d_own.p, d_prov.p, n_own, c_pv.p, s);
                KJ_CUDA(cudaMemcpyAsync(prov, c_pv.p, n_own, cudaMemcpyDeviceToHost, s));
            }
            if (owned) {
                c_q.ensure(n_own);
                launch_map_u32(d_own.p, d_q.p, n_own, c_q.p, s);
                KJ_CUDA(cudaMemcpyAsync(owned, c_q.p, 4 * n_own, cudaMemcpyDeviceToHost, s));
            }
            c->sync();
        }
        I.ms_download = t.ms();
    }
    I.ms_total = t_all.ms();
    I.kernel_launches = g_launches.load() - launches0;
    if (info) *info = I;
}

int knnj_shard_range(const double* cost, uint64_t n_items, uint32_t shard_index,
                     uint32_t shard_count, uint64_t* first, uint64_t* last) {
    if (!first || !last || shard_count < 1 || shard_index >= shard_count || (n_items && !cost))
        return KNNJ_E_USAGE;
    shard_range(cost, n_items, shard_index, shard_count, first, last);
    return KNNJ_OK;
}

int knnj_run(knnj_ctx* c, const knnj_config* cfg, uint32_t* ids, double* dist, uint8_t* prov,
             uint64_t* raw_hist, knnj_run_info* info) {
    return guarded(c, [&] {
        run_impl(c, cfg, 0, 1, nullptr, nullptr, ids, dist, prov, nullptr, raw_hist, info);
    });
}

int knnj_parameter_search(knnj_ctx* c, const knnj_config* base, double f, const double* betas,
                          const double* gammas, uint64_t n_candidates, knnj_search_row* rows,
                          double* best_beta, double* best_gamma) {
    // parameter_search, proj/src/orchestrator.cpp:252-303
    return guarded(c, [&] {
        if (!c || !base || !best_beta || !best_gamma || (n_candidates && (!betas || !gammas || !rows)))
            throw Error(1, "null argument");
        if (!(f > 0.0) || f > 1.0) throw Error(1, "query fraction f must be in (0, 1]");
        if (n_candidates == 0) throw Error(1, "parameter search needs at least one candidate");
        const uint64_t want = (uint64_t)std::floor(f * double(c->N));
        if (want < 50)
            throw Error(7, "parameter search sample of " + std::to_string(want) +
                               " queries is below the floor of 50");
        // kSeedQuerySubset
        const std::vector<uint64_t> picked = sample_seeded(c->N, want, derive_seed(base->seed, 0x04));
        const std::vector<uint32_t> subset(picked.begin(), picked.end());
        bool have = false;
        double best = 0.0;
        for (uint64_t i = 0; i < n_candidates; ++i) {
            knnj_config cfg = *base;
            cfg.mode = KNNJ_HYBRID;
            cfg.beta = betas[i];
            cfg.gamma = gammas[i];
            cfg.rho = 0.5;  // the reference's starting balance
            cfg.query_subset = subset.data();
            cfg.n_query_subset = subset.size();
            knnj_search_row& row = rows[i];
            row = knnj_search_row{};
            row.beta = betas[i];
            row.gamma = gammas[i];
            auto fail = [&](int code, const char* msg) {
                row.status = code;
                std::snprintf(row.error, sizeof row.error, "%s", msg);
            };
            try {
                auto info = std::make_unique<knnj_run_info>();
                run_impl(c, &cfg, 0, 1, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr,
                         nullptr, info.get());
                row.wall_seconds = info->ms_total / 1000.0;
                if (!have || row.wall_seconds < best) {
                    have = true;
                    best = row.wall_seconds;
                    *best_beta = row.beta;
                    *best_gamma = row.gamma;
                }
            } catch (const kj::Error& e) {
                fail(e.code, e.what());
            } catch (const std::exception& e) {
                fail(KNNJ_E_CUDA, e.what());
            }
            alloc_stream() = c->s;
            alloc_cache() = &c->cache;
        }
        if (!have) throw Error(1, "every parameter-search candidate failed");
    });
}

int knnj_run_shard(knnj_ctx* c, const knnj_config* cfg, uint32_t shard_index,
                   uint32_t shard_count, knnj_allreduce_fn allreduce, void* allreduce_user,
                   uint32_t* ids, double* dist, uint8_t* prov, uint32_t* owned_queries,
                   uint64_t* raw_hist, knnj_run_info* info) {
    return guarded(c, [&] {
        run_impl(c, cfg, shard_index, shard_count, allreduce, allreduce_user, ids, dist, prov,
                 owned_queries, raw_hist, info);
    });
}

}  // extern "C"
