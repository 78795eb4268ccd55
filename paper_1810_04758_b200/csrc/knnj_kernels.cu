// Device kernels of the B200 KNN self-join engine (sm_100a).
//
// Hot path:
//   k_join      fused range-join + per-query screened top-K   (execute_batch + filter_keys,
//               proj/src/dense_engine.cpp:86-196; grid walk grid_index.cpp:114-147)
//   k_finalize  exact FP64 (scalar order) re-decision of the screened list
//   k_hist      ε-selection distance histogram (build_distance_histogram, epsilon.cpp:46-120)
//   grid build  cell keys + CUB radix sort + RLE tables (GridIndex::build, grid_index.cpp:13-75)
//
// Exactness model. A candidate pair is first scored with an FP32 "GEMM form"
// distance  key = |a'|^2 + |b'|^2 - 2 a'.b'  on coordinates centred at a
// per-block origin; |key - sq64| <= delta with delta a rigorous bound derived in
// DESIGN.md §3 (input rounding + FP32 dot-product error + FP64 accumulation
// slack). Every decision (top-K membership, ε test, histogram bin) is either
// certain from key±delta or re-decided with the FP64 scalar-order distance, so
// results are bit-identical to the reference scalar kernel.
#include <cub/cub.cuh>
#include <math_constants.h>

#include <atomic>

#include "knnj_internal.cuh"

namespace kj {

std::atomic<unsigned long long> g_launches{0};

// ---------------------------------------------------------------- helpers
__device__ __forceinline__ double exact_sq(const double* __restrict__ a,
                                           const double* __restrict__ b, uint32_t n) {
    // proj/src/kernels_scalar.cpp:9-27, without the early exit (which never
    // changes a finite result): d = a-b; sum += d*d, each op rounded separately.
    double sum = 0.0;
    for (uint32_t i = 0; i < n; ++i) {
        double d = __dsub_rn(a[i], b[i]);
        sum = __dadd_rn(sum, __dmul_rn(d, d));
    }
    return sum;
}

__device__ __forceinline__ bool pair_less(double sa, uint32_t ia, double sb, uint32_t ib) {
    return sa < sb || (sa == sb && ia < ib);
}

__device__ __forceinline__ void cp_async4(void* smem, const void* gmem) {
    unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
    unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n"); }
template <int N>
__device__ __forceinline__ void cp_wait() {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

__device__ __forceinline__ unsigned long long dbl_order(double v) {
    unsigned long long b = __double_as_longlong(v);
    return (b & 0x8000000000000000ull) ? ~b : (b | 0x8000000000000000ull);
}

// Rigorous |key - sq64| bound for one (query, tile): A = |a'|, B = max |b'|.
// gam = 2.02*gamma_{n+2}(fp32); E = erg + eab*(A+B) bounds the input rounding
// of the difference vector; e64 covers the FP64 scalar accumulation.
__device__ __forceinline__ float screen_delta(float A, float B, float gam, float erg, float eab,
                                              float e64) {
    float AB = A + B;
    float E = erg + eab * AB;
    float D = AB + E;
    float d = gam * (A * A + B * B) + 2.f * D * E + E * E + e64 * D * D;
    return d * 1.0625f + 1e-37f;
}

// ---------------------------------------------------------------- join kernel
// One block = one work item: up to QB (128, or 32 for sparse cells) queries of ONE grid cell (one query per
// thread) against the candidate position ranges of that cell's 3^m
// neighbourhood (merged along the last indexed dim). Candidate tiles of T
// points are staged SoA in shared memory (cp.async, double-buffered), centred
// at the block origin, and scored against every query of the block. Per query
// a list of all candidates that can still belong to the exact top-K is kept
// (sorted by key, capacity L), pruned with cut = key_K + 2*delta_max.
template <int NP, int T, int QB>
__global__ void __launch_bounds__(QB) k_join(JoinArgs p) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    float* tile = reinterpret_cast<float*>(smem_raw);          // [2][NP][T]
    float* nbuf = tile + 2 * NP * T;                            // [2][T]
    uint32_t* tpos = reinterpret_cast<uint32_t*>(nbuf + 2 * T); // [2][T]
    float* cen = reinterpret_cast<float*>(tpos + 2 * T);        // [NP] (+pad)
    float* lkey = cen + ((NP + 3) & ~3);                        // [L][QB]
    uint32_t* lpos = reinterpret_cast<uint32_t*>(lkey + p.L * QB);

    __shared__ uint32_t s_ri, s_off, s_cnt[2];
    __shared__ unsigned s_bmax[2];

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint4 it = p.items[blockIdx.x];
    const uint32_t nq = it.y - it.x;
    const bool has_q = (uint32_t)tid < nq;
    const uint32_t row = it.x + (has_q ? tid : 0);
    const uint32_t qp = p.qpos[row];
    const uint32_t n = p.n;
    const uint64_t Npad = p.Npad;

    // zero padded dims of both tile buffers once; block origin = first query
    for (int i = tid; i < 2 * (NP - (int)n) * T; i += QB) {
        int b = i / ((NP - n) * T), r = i % ((NP - n) * T);
        tile[(b * NP + n) * T + r] = 0.f;
    }
    const uint32_t q0 = p.qpos[it.x];
    for (int d = tid; d < NP; d += QB) cen[d] = d < (int)n ? p.Xs[(uint64_t)d * Npad + q0] : 0.f;
    if (tid == 0) {
        s_ri = it.z;
        s_off = 0;
    }
    __syncthreads();

    // query vector (registers): a2 = -2 a', na = |a'|^2
    float a2[NP];
    float na = 0.f;
#pragma unroll
    for (int d = 0; d < NP; ++d) {
        float v = d < (int)n ? p.Xs[(uint64_t)d * Npad + qp] - cen[d] : 0.f;
        a2[d] = -2.f * v;
        na = fmaf(v, v, na);
    }
    const float Aq = sqrtf(na) * 1.0001f;
    const float init_cut = (p.init_cut && has_q) ? p.init_cut[row] : CUDART_INF_F;

    int cnt = 0;
    bool ovf = false;
    float dmax = 0.f;
    float cut_list = CUDART_INF_F;

    auto build = [&](int b) {  // warp 0: next T candidate positions from the cursor
        if (warp == 0) {
            uint32_t ri = s_ri, off = s_off, filled = 0;
            while (filled < (uint32_t)T && ri < it.w) {
                uint2 r = p.adj[ri];
                uint32_t avail = r.y - r.x - off;
                uint32_t take = min(avail, (uint32_t)T - filled);
                for (uint32_t i = lane; i < take; i += 32) tpos[b * T + filled + i] = r.x + off + i;
                filled += take;
                off += take;
                if (off == r.y - r.x) {
                    ++ri;
                    off = 0;
                }
            }
            for (uint32_t i = filled + lane; i < (uint32_t)T; i += 32) tpos[b * T + i] = OVF;
            __syncwarp();
            if (lane == 0) {
                s_ri = ri;
                s_off = off;
                s_cnt[b] = filled;
                s_bmax[b] = 0u;
            }
        }
    };
    auto issue = [&](int b) {
        const uint32_t c = s_cnt[b];
        for (uint32_t i = tid; i < n * (uint32_t)T; i += QB) {
            uint32_t d = i / T, j = i % T;
            float* dst = &tile[(b * NP + d) * T + j];
            uint32_t pj = tpos[b * T + j];
            if (j < c) cp_async4(dst, p.Xs + (uint64_t)d * Npad + pj);
            else *dst = 0.f;
        }
        cp_commit();
    };

    build(0);
    __syncthreads();
    issue(0);
    int buf = 0;
    while (true) {
        const uint32_t c = s_cnt[buf];
        if (c == 0) break;
        build(buf ^ 1);
        __syncthreads();
        issue(buf ^ 1);
        cp_wait<1>();
        __syncthreads();
        // centre candidates, norms, tile max norm
        for (int j = tid; j < T; j += QB) {
            float nb = CUDART_NAN_F;
            if ((uint32_t)j < c) {
                nb = 0.f;
#pragma unroll
                for (int d = 0; d < NP; ++d) {
                    if (d < (int)n) {
                        float v = tile[(buf * NP + d) * T + j] - cen[d];
                        tile[(buf * NP + d) * T + j] = v;
                        nb = fmaf(v, v, nb);
                    }
                }
            }
            nbuf[buf * T + j] = nb;
            float m = (uint32_t)j < c ? nb : 0.f;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
            if (lane == 0) atomicMax(&s_bmax[buf], __float_as_uint(m));
        }
        __syncthreads();
        if (has_q && !ovf) {
            const float Bt = sqrtf(__uint_as_float(s_bmax[buf])) * 1.0001f;
            const float dl = screen_delta(Aq, Bt, p.gam, p.erg, p.eab, p.e64);
            dmax = fmaxf(dmax, dl);
            if (cnt >= (int)p.K) cut_list = __fadd_ru(lkey[(p.K - 1) * QB + tid], 2.f * dmax);
            float cut = fminf(cut_list, __fadd_ru(init_cut, dl));
            float rhs = __fsub_ru(cut, na);
            const float* tb = tile + buf * NP * T;
            const float* nbb = nbuf + buf * T;
            // hits of 4 candidates (j .. j+3), screened against the current rhs
            auto proc4 = [&](uint32_t j, float acc0, float acc1, float acc2, float acc3) {
                const bool s0 = acc0 <= rhs, s1 = acc1 <= rhs, s2 = acc2 <= rhs, s3 = acc3 <= rhs;
                if (!(s0 | s1 | s2 | s3)) return;
                float accs[4] = {acc0, acc1, acc2, acc3};
                bool ss[4] = {s0, s1, s2, s3};
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    if (!ss[u]) continue;
                    const uint32_t pos = tpos[buf * T + j + u];
                    if (pos == qp) continue;  // self pair: excluded by id
                    const float key = accs[u] + na;
                    if (cnt == (int)p.L) {
                        ovf = true;
                        rhs = -CUDART_INF_F;
                        return;
                    }
                    int q = cnt;
                    while (q > 0) {
                        float kq = lkey[(q - 1) * QB + tid];
                        if (kq <= key) break;
                        lkey[q * QB + tid] = kq;
                        lpos[q * QB + tid] = lpos[(q - 1) * QB + tid];
                        --q;
                    }
                    lkey[q * QB + tid] = key;
                    lpos[q * QB + tid] = pos;
                    ++cnt;
                    if (cnt >= (int)p.K) {
                        cut_list = __fadd_ru(lkey[(p.K - 1) * QB + tid], 2.f * dmax);
                        const float ci = __fadd_ru(init_cut, dmax);
                        const float ce = fminf(cut_list, ci);
                        while (cnt > (int)p.K && lkey[(cnt - 1) * QB + tid] > ce) --cnt;
                        cut = fminf(cut_list, __fadd_ru(init_cut, dl));
                        rhs = __fsub_ru(cut, na);
                    }
                }
            };
            // 8 candidates per step: two independent groups of FMA chains (ILP)
            const uint32_t jend = (c + 7) & ~7u;
            for (uint32_t j = 0; j < jend; j += 8) {
                const float4 na4 = *reinterpret_cast<const float4*>(nbb + j);
                const float4 nb4 = *reinterpret_cast<const float4*>(nbb + j + 4);
                float a0 = na4.x, a1 = na4.y, a2v = na4.z, a3 = na4.w;
                float b0 = nb4.x, b1 = nb4.y, b2 = nb4.z, b3 = nb4.w;
#pragma unroll
                for (int d = 0; d < NP; ++d) {
                    const float4 x = *reinterpret_cast<const float4*>(tb + d * T + j);
                    const float4 y = *reinterpret_cast<const float4*>(tb + d * T + j + 4);
                    a0 = fmaf(a2[d], x.x, a0);
                    a1 = fmaf(a2[d], x.y, a1);
                    a2v = fmaf(a2[d], x.z, a2v);
                    a3 = fmaf(a2[d], x.w, a3);
                    b0 = fmaf(a2[d], y.x, b0);
                    b1 = fmaf(a2[d], y.y, b1);
                    b2 = fmaf(a2[d], y.z, b2);
                    b3 = fmaf(a2[d], y.w, b3);
                }
                proc4(j, a0, a1, a2v, a3);
                if (!ovf) proc4(j + 4, b0, b1, b2, b3);
            }
        }
        __syncthreads();
        buf ^= 1;
    }
    cp_wait<0>();
    if (has_q) {
        p.out_cnt[row] = ovf ? OVF : (uint32_t)cnt;
        if (!ovf)
            for (int i = 0; i < cnt; ++i) p.out_pos[(uint64_t)row * p.L + i] = lpos[i * QB + tid];
    }
}

// rank of each of this lane's E entries among all c entries of the warp's list
template <int E, int EMAX>
__device__ __forceinline__ void rank_entries(const double (&sq)[EMAX], const uint32_t (&id)[EMAX],
                                             uint32_t (&rk)[EMAX], uint32_t c) {
#pragma unroll
    for (int e = 0; e < E; ++e) {
        const double ms = sq[e];
        const uint32_t mi = id[e];
        for (int src = 0; src < 32; ++src) {
            const double s = __shfl_sync(0xffffffffu, ms, src);
            const uint32_t t = __shfl_sync(0xffffffffu, mi, src);
            if ((uint32_t)(e * 32 + src) >= c) break;
#pragma unroll
            for (int f = 0; f < E; ++f)
                if (pair_less(s, t, sq[f], id[f])) ++rk[f];
        }
    }
}

// The same ranks with the row's entries staged in shared memory: one broadcast 16-byte
// load per source entry instead of three shuffles (the finalize is bound by its LSU /
// shuffle issue: ncu r02fin, 46% LSU, 80% SM throughput).
template <int E, int EMAX>
__device__ __forceinline__ void rank_entries_smem(const double (&sq)[EMAX], const uint32_t (&id)[EMAX],
                                                  uint32_t (&rk)[EMAX], uint32_t c, uint4* ent) {
    const int lane = threadIdx.x & 31;
    __syncwarp();  // the previous row's reads are done
#pragma unroll
    for (int e = 0; e < E; ++e) {
        const unsigned long long b = (unsigned long long)__double_as_longlong(sq[e]);
        ent[e * 32 + lane] = make_uint4((uint32_t)b, (uint32_t)(b >> 32), id[e], 0u);
    }
    __syncwarp();
#pragma unroll 4
    for (uint32_t src = 0; src < c; ++src) {
        const uint4 v = ent[src];
        const double sv = __longlong_as_double((long long)(((unsigned long long)v.y << 32) | v.x));
#pragma unroll
        for (int f = 0; f < E; ++f)
            if (pair_less(sv, v.z, sq[f], id[f])) ++rk[f];
    }
}

// ---------------------------------------------------------------- finalize

// One warp per launch row: exact FP64 distances for the screened list, exact
// (sq,id) ranks, first K written to the query's output row, status bits.
// status bits and the K-th of one finalized row (lane 0 writes)
__device__ __forceinline__ void finalize_status(const FinalArgs& a, uint32_t c, uint32_t orow, double kth,
                                                int lane) {
    if (lane != 0) return;
    uint8_t st = 0;
    if (c >= a.K) {
        st |= ST_HAS_K;
        if (kth <= a.eps2) st |= ST_IN_EPS;
        if (kth < a.cover2) st |= ST_CERT;
    }
    // bounded pass: the listed top-K is the exact one only if its K-th lies within the
    // bound (every candidate up to it was screened); otherwise re-run unbounded
    if (a.bound2 > 0.0 && !(c >= a.K && kth <= a.bound2)) st = ST_MISS;
    a.out_status[orow] = st;
    a.out_kth[orow] = c >= a.K ? kth : CUDART_INF;
    if (a.out_count) a.out_count[orow] = min(c, a.K);
}

template <int EMAX>
__device__ __forceinline__ void finalize_row(const FinalArgs& a, uint64_t row, int lane,
                                             uint4* ent = nullptr) {
    const uint32_t c = a.cnt[row];
    if (c == SKIP) return;  // a split row: its parts are finalized and merged separately
    const uint32_t orow = a.qrow[row];
    if (c == OVF) {
        if (lane == 0) a.out_status[orow] = a.bound2 > 0.0 ? ST_MISS : ST_OVF;
        return;
    }
    const uint32_t qp = a.qpos[row];
    const double* qx = a.XJ ? a.XJ + (uint64_t)qp * a.n : a.X64 + (uint64_t)a.A[qp] * a.n;
    double sq[EMAX];
    uint32_t id[EMAX];
    uint32_t rk[EMAX];
    const int E = (int)((c + 31) / 32);
#pragma unroll
    for (int e = 0; e < EMAX; ++e) {
        sq[e] = CUDART_INF;
        id[e] = 0xFFFFFFFFu;
        rk[e] = 0;
        const uint32_t i = e * 32 + lane;
        if (e < E && i < c) {
            const uint32_t ps = a.pos[row * a.L + i];
            const uint32_t t = a.A[ps];
            id[e] = t;
            sq[e] = exact_sq(qx, a.XJ ? a.XJ + (uint64_t)ps * a.n : a.X64 + (uint64_t)t * a.n, a.n);
        }
    }
    // exact (sq, id) rank of every entry: compile-time entry count per lane, so the
    // inner comparisons are not issued for empty register slots
    if (ent) {  // staged ranks (lists of at most 64 entries)
        if (E == 1) rank_entries_smem<1, EMAX>(sq, id, rk, c, ent);
        else if (E == 2) rank_entries_smem<2, EMAX>(sq, id, rk, c, ent);
    } else switch (E) {
#define KJ_RANK(EE)                                        \
        case EE:                                           \
            rank_entries<EE, EMAX>(sq, id, rk, c);         \
            break;
        KJ_RANK(1) KJ_RANK(2)
        case 3: if constexpr (EMAX >= 3) rank_entries<3, EMAX>(sq, id, rk, c); break;
        case 4: if constexpr (EMAX >= 4) rank_entries<4, EMAX>(sq, id, rk, c); break;
        case 5: if constexpr (EMAX >= 5) rank_entries<5, EMAX>(sq, id, rk, c); break;
        case 6: if constexpr (EMAX >= 6) rank_entries<6, EMAX>(sq, id, rk, c); break;
        case 7: if constexpr (EMAX >= 7) rank_entries<7, EMAX>(sq, id, rk, c); break;
        case 8: if constexpr (EMAX >= 8) rank_entries<8, EMAX>(sq, id, rk, c); break;
#undef KJ_RANK
        default: break;
    }
    double kth = CUDART_INF;
#pragma unroll
    for (int f = 0; f < EMAX; ++f) {
        const uint32_t i = f * 32 + lane;
        if (f < E && i < c && rk[f] < a.K) {
            const double d = sqrt(sq[f]);
            a.out_ids[(uint64_t)orow * a.K + rk[f]] = id[f];
            a.out_dist[(uint64_t)orow * a.K + rk[f]] = d;
            if (a.out_sq) a.out_sq[(uint64_t)orow * a.K + rk[f]] = sq[f];
            if (rk[f] == a.K - 1) kth = sq[f];
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) kth = fmin(kth, __shfl_xor_sync(0xffffffffu, kth, o));
    finalize_status(a, c, orow, kth, lane);
}

// Warps stride over the launch rows (a bounded grid shares the SMs with a running join).
// EMAX = list entries per lane: 2 for lists of at most 64 (fewer registers, more warps in
// flight for the gathers), else 8.
template <int EMAX>
__global__ void k_finalize(FinalArgs a) {
    const int lane = threadIdx.x & 31;
    const uint64_t nw = (uint64_t(gridDim.x) * blockDim.x) >> 5;
    __shared__ uint4 s_ent[EMAX == 2 ? 8 * 64 : 1];  // 256-thread blocks: 8 warps x 64 entries
    uint4* ent = EMAX == 2 ? s_ent + (threadIdx.x >> 5) * 64 : nullptr;
    for (uint64_t w = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; w < a.nrows; w += nw)
        finalize_row<EMAX>(a, w, lane, ent);
}

// ---------------------------------------------------------------- histogram
// Block = JB sampled queries x one slab of candidates (id order). Per pair the
// FP32 key decides "beyond eps_mean" / bin b whenever key±delta is certain;
// otherwise the FP64 scalar distance decides exactly like epsilon.cpp:86-95.
// Each thread owns a private column of bin counters in shared memory (no
// atomics on the hot path); columns are reduced once per block.
template <int NP, int T>
__global__ void __launch_bounds__(JB) k_hist(HistArgs a) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    float* tile = reinterpret_cast<float*>(smem_raw);  // [2][NP][T]
    float* nbuf = tile + 2 * NP * T;                   // [2][T]
    float* LO = nbuf + 2 * T;                          // [n_bins+1]
    float* HI = LO + a.n_bins + 1;                     // [n_bins+1]
    uint32_t* hist = reinterpret_cast<uint32_t*>(HI + a.n_bins + 1);  // [n_bins][JB]
    __shared__ unsigned s_bmax[2];

    const int tid = threadIdx.x, lane = tid & 31;
    const uint32_t n = a.n, nbins = a.n_bins;
    const uint64_t row = uint64_t(blockIdx.x) * JB + tid;
    const bool has_q = row < a.nq;
    const uint32_t qid = has_q ? a.q[row] : 0;
    const uint64_t cb = uint64_t(blockIdx.y) * a.cand_begin_stride;
    const uint64_t ce = min(a.N, cb + a.cand_begin_stride);

    for (uint32_t i = tid; i < nbins * JB; i += JB) hist[i] = 0;
    for (uint32_t i = tid; i <= nbins; i += JB) {
        LO[i] = a.SU[i];
        HI[i] = a.SD[i];
    }
    for (int i = tid; i < 2 * (NP - (int)n) * T; i += JB) {
        int b = i / ((NP - n) * T), r = i % ((NP - n) * T);
        tile[(b * NP + n) * T + r] = 0.f;
    }
    float a2[NP];
    float na = 0.f;
#pragma unroll
    for (int d = 0; d < NP; ++d) {
        float v = (d < (int)n && has_q) ? a.Xf[(uint64_t)d * a.Npad + qid] : 0.f;
        a2[d] = -2.f * v;
        na = fmaf(v, v, na);
    }
    const float Aq = sqrtf(na) * 1.0001f;
    const uint32_t ncount = a.n_count;
    const float lo_end = a.SU[ncount];  // lower edge of the first uncounted bin
    const float invw = (float)a.inv_width;
    const double* qx = a.X64 + (uint64_t)qid * n;

    auto issue = [&](int b, uint64_t s0) {
        // s0 is a multiple of 4 and Npad a multiple of 4: 16-byte copies
        for (uint32_t i = tid; i < n * (uint32_t)(T / 4); i += JB) {
            uint32_t d = i / (T / 4), j4 = (i % (T / 4)) * 4;
            float* dst = &tile[(b * NP + d) * T + j4];
            cp_async16(dst, a.Xf + (uint64_t)d * a.Npad + s0 + j4);
        }
        cp_commit();
        if (tid == 0) s_bmax[b] = 0u;
    };

    __syncthreads();
    if (cb < ce) issue(0, cb);
    int buf = 0;
    for (uint64_t s0 = cb; s0 < ce; s0 += T) {
        const uint32_t c = (uint32_t)min((uint64_t)T, ce - s0);
        if (s0 + T < ce) issue(buf ^ 1, s0 + T);
        else cp_commit();
        cp_wait<1>();
        __syncthreads();
        for (int j = tid; j < T; j += JB) {
            float nb = CUDART_NAN_F;
            if ((uint32_t)j < c) {
                nb = 0.f;
#pragma unroll
                for (int d = 0; d < NP; ++d) {
                    float v = tile[(buf * NP + d) * T + j];
                    nb = fmaf(v, v, nb);
                }
            }
            nbuf[buf * T + j] = nb;
            float m = (uint32_t)j < c ? nb : 0.f;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
            if (lane == 0) atomicMax(&s_bmax[buf], __float_as_uint(m));
        }
        __syncthreads();
        if (has_q) {
            const float Bt = sqrtf(__uint_as_float(s_bmax[buf])) * 1.0001f;
            const float dl = screen_delta(Aq, Bt, a.gam, a.erg, a.eab, a.e64);
            // key - dl >= lo_end  <=>  acc >= lo_end + dl - na (rounded down: conservative)
            const float skip_at = __fsub_ru(__fadd_ru(lo_end, dl), na);
            const float* tb = tile + buf * NP * T;
            const float* nbb = nbuf + buf * T;
            const uint32_t jend = (c + 3) & ~3u;
            for (uint32_t j = 0; j < jend; j += 4) {
                float4 nb4 = *reinterpret_cast<const float4*>(nbb + j);
                float acc[4] = {nb4.x, nb4.y, nb4.z, nb4.w};
#pragma unroll
                for (int d = 0; d < NP; ++d) {
                    float4 b = *reinterpret_cast<const float4*>(tb + d * T + j);
                    acc[0] = fmaf(a2[d], b.x, acc[0]);
                    acc[1] = fmaf(a2[d], b.y, acc[1]);
                    acc[2] = fmaf(a2[d], b.z, acc[2]);
                    acc[3] = fmaf(a2[d], b.w, acc[3]);
                }
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    if (!(acc[u] < skip_at)) continue;  // beyond eps_mean (or NaN pad)
                    const uint64_t t = s0 + j + u;
                    if (t == qid) continue;
                    const float key = acc[u] + na;
                    const float klo = __fsub_rd(key, dl), khi = __fadd_ru(key, dl);
                    int b = key > 0.f ? (int)(key * rsqrtf(key) * invw) : 0;
                    b = min(max(b, 0), (int)nbins - 1);
                    if (klo >= LO[b] && khi < HI[b]) {
                        if ((uint32_t)b < ncount) hist[b * JB + tid] += 1;
                    } else {
                        const double sq = exact_sq(qx, a.X64 + t * n, n);
                        if (sq > a.limit_sq) continue;
                        const double dist = sqrt(sq);
                        if (dist >= a.eps_mean) continue;
                        uint64_t bb = (uint64_t)(dist * a.inv_width);
                        if (bb >= nbins) bb = nbins - 1;
                        if (bb < ncount) hist[bb * JB + tid] += 1;
                    }
                }
            }
        }
        __syncthreads();
        buf ^= 1;
    }
    cp_wait<0>();
    __syncthreads();
    for (uint32_t b = tid; b < nbins; b += JB) {
        unsigned long long s = 0;
        for (int t = 0; t < JB; ++t) s += hist[b * JB + ((t + b) & (JB - 1))];
        if (s) atomicAdd(&a.counts[b], s);
    }
}

// ---------------------------------------------------------------- dispatch
// Opt a kernel into the dynamic shared memory it needs (static smem counts
// against the same per-block limit).
template <class K>
static void set_smem(K kernel, size_t dyn) {
    int dev = 0, optin = 0;
    KJ_CUDA(cudaGetDevice(&dev));
    KJ_CUDA(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
    cudaFuncAttributes fa;
    KJ_CUDA(cudaFuncGetAttributes(&fa, kernel));
    if (dyn + fa.sharedSizeBytes > (size_t)optin)
        throw Error(1, "configuration needs more shared memory than the device allows");
    KJ_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn));
}
#define KJ_NP_LIST(X) \
    X(1) X(2) X(3) X(4) X(5) X(6) X(7) X(8) X(10) X(12) X(16) X(18) X(20) X(24) X(32) \
    X(48) X(64) X(96) X(128)

int pick_np(uint32_t n) {
    static const int nps[] = {1, 2, 3, 4, 5, 6, 7, 8, 10, 12, 16, 18, 20, 24, 32, 48, 64, 96, 128};
    for (int v : nps)
        if ((uint32_t)v >= n) return v;
    return -1;
}
static int tile_for(int np) { return np <= 32 ? 128 : 64; }

// 32-query blocks over small dims stage 64-candidate tiles: their smem (and with it the
// blocks per SM) is bounded by the per-query lists, so a smaller tile buys occupancy
static int join_tile_for(int np, uint32_t qb) { return (qb == 32 && np <= 16) ? 64 : tile_for(np); }
size_t join_smem_bytes(int np, uint32_t L, uint32_t qb) {
    int T = join_tile_for(np, qb);
    return sizeof(float) * (2 * np * T + 2 * T) + sizeof(uint32_t) * 2 * T +
           sizeof(float) * ((np + 3) & ~3) + (sizeof(float) + sizeof(uint32_t)) * L * qb;
}

template <int NP, int QB>
static void launch_join_np(const JoinArgs& a, uint64_t nitems, cudaStream_t s) {
    constexpr int T = (QB == 32 && NP <= 16) ? 64 : (NP <= 32 ? 128 : 64);
    size_t sm = join_smem_bytes(NP, a.L, QB);
    set_smem(k_join<NP, T, QB>, sm);
    for (uint64_t off = 0; off < nitems; off += 2147483647ull) {
        uint64_t cnt = std::min<uint64_t>(nitems - off, 2147483647ull);
        JoinArgs b = a;
        b.items = a.items + off;
        k_join<NP, T, QB><<<dim3((unsigned)cnt), QB, sm, s>>>(b);
    }
    KJ_CUDA(cudaGetLastError());
    g_launches.fetch_add(1, std::memory_order_relaxed);
}

void launch_join(const JoinArgs& a, uint64_t nitems, uint32_t qb, cudaStream_t s) {
    if (nitems == 0) return;
    int np = pick_np(a.n);
    switch (np) {
#define X(v) \
    case v:                                                         \
        if (qb == 32) launch_join_np<v, 32>(a, nitems, s);          \
        else launch_join_np<v, JB>(a, nitems, s);                   \
        break;
        KJ_NP_LIST(X)
#undef X
        default: throw Error(1, "dimension count above 128 is not supported by the device join");
    }
}

void launch_finalize(const FinalArgs& a, cudaStream_t s, uint32_t max_blocks) {
    if (a.nrows == 0) return;
    uint64_t blocks = (a.nrows * 32 + 255) / 256;
    if (max_blocks) blocks = std::min<uint64_t>(blocks, max_blocks);
    if (a.L <= 64) k_finalize<2><<<(unsigned)blocks, 256, 0, s>>>(a);
    else k_finalize<8><<<(unsigned)blocks, 256, 0, s>>>(a);
    KJ_CUDA(cudaGetLastError());
    g_launches.fetch_add(1, std::memory_order_relaxed);
}

size_t hist_smem_bytes(int np, uint32_t n_bins) {
    int T = tile_for(np);
    return sizeof(float) * (2 * np * T + 2 * T) + sizeof(float) * 2 * (n_bins + 1) +
           sizeof(uint32_t) * n_bins * JB;
}

template <int NP>
static void launch_hist_np(const HistArgs& a, uint64_t n_slabs, cudaStream_t s) {
    constexpr int T = NP <= 32 ? 128 : 64;
    size_t sm = hist_smem_bytes(NP, a.n_bins);
    set_smem(k_hist<NP, T>, sm);
    dim3 grid((unsigned)((a.nq + JB - 1) / JB), (unsigned)n_slabs);
    k_hist<NP, T><<<grid, JB, sm, s>>>(a);
    KJ_CUDA(cudaGetLastError());
    g_launches.fetch_add(1, std::memory_order_relaxed);
}

void launch_histogram(const HistArgs& a, uint64_t n_slabs, cudaStream_t s) {
    if (a.nq == 0) return;
    int np = pick_np(a.n);
    switch (np) {
#define X(v) \
    case v: launch_hist_np<v>(a, n_slabs, s); break;
        KJ_NP_LIST(X)
#undef X
        default: throw Error(1, "dimension count above 128 is not supported by the device histogram");
    }
}

// ---------------------------------------------------------------- grid histogram
__device__ __forceinline__ uint64_t lower_bound_u64(const uint64_t* a, uint64_t n, uint64_t key) {
    uint64_t lo = 0, hi = n;
    while (lo < hi) {
        uint64_t mid = (lo + hi) >> 1;
        if (a[mid] < key) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

// Capped eps-selection histogram over a grid of cell width >= the counted radius r
// (every counted pair, dist < r in all n dims, lies in the query's 3^m cell
// neighbourhood): one warp per sampled query. The warp's lanes first resolve the
// 3^(m-1) rows of the neighbourhood (each row one contiguous position range of the
// grid's sorted order: cells sorted by linear id, the last dim fastest), then stride
// over the candidates. Same screen and exact-bin rule as k_hist (FP32 key +- delta
// certain, else the FP64 scalar distance bins it like epsilon.cpp:86-95); only bins
// [0, n_count) are counted. Used for small n, where the grid neighbourhood is a tight
// superset of the counted ball.
template <int NP>
__global__ void __launch_bounds__(256) k_hist_grid(HistGridArgs a) {
    constexpr int WARPS = 8, MAXR = 243;  // 3^5 rows for m <= 6
    __shared__ uint2 s_rng[WARPS][MAXR];
    __shared__ uint32_t s_hist[WARPS][256];
    __shared__ float s_lo[257], s_hi[257];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t n = a.n, m = a.m, nbins = a.n_bins, ncount = a.n_count;
    for (uint32_t i = threadIdx.x; i < WARPS * 256; i += blockDim.x) (&s_hist[0][0])[i] = 0;
    for (uint32_t i = threadIdx.x; i <= nbins; i += blockDim.x) {
        s_lo[i] = a.SU[i];
        s_hi[i] = a.SD[i];
    }
    __syncthreads();
    const float lo_end = a.SU[ncount];
    const float invw = (float)a.inv_width;
    const uint32_t ml = m - 1;
    uint32_t R = 1;
    for (uint32_t j = 0; j < ml; ++j) R *= 3;
    for (uint64_t row = uint64_t(blockIdx.x) * WARPS + warp; row < a.nq;
         row += uint64_t(gridDim.x) * WARPS) {
        const bool by_id = a.qids != nullptr;
        const uint32_t qp = by_id ? 0xFFFFFFFFu : a.qpos[row];
        const uint32_t qid = by_id ? a.qids[row] : a.A[qp];
        uint64_t c[8];
        if (by_id) {  // the cell rule of k_cell_keys (grid_index.cpp:77-88)
            for (uint32_t j = 0; j < m; ++j) {
                double rel = __ddiv_rn(__dsub_rn(a.X64[(uint64_t)qid * n + j], a.mins[j]), a.w);
                if (rel < 0.0) rel = 0.0;
                uint64_t idx = (uint64_t)floor(rel);
                if (idx > a.cpd[j] - 1) idx = a.cpd[j] - 1;
                c[j] = idx;
            }
        } else {
            uint64_t r = a.B[a.slot[qid]];
            for (uint32_t j = 0; j < m; ++j) {
                c[j] = r / a.strides[j];
                r -= c[j] * a.strides[j];
            }
        }
        const uint64_t lo_l = c[ml] > 0 ? c[ml] - 1 : 0;
        const uint64_t hi_l = min(c[ml] + 1, a.cpd[ml] - 1);
        __syncwarp();
        for (uint32_t r = lane; r < R; r += 32) {
            uint64_t base = 0, t = r;
            bool ok = true;
            for (int j = (int)ml - 1; j >= 0; --j) {
                const uint64_t dig = t % 3;
                t /= 3;
                const int64_t cj = (int64_t)c[j] - 1 + (int64_t)dig;
                if (cj < 0 || cj >= (int64_t)a.cpd[j]) {
                    ok = false;
                    break;
                }
                base += (uint64_t)cj * a.strides[j];
            }
            uint2 rg = make_uint2(0, 0);
            if (ok) {
                const uint64_t i0 = lower_bound_u64(a.B, a.ncells, base + lo_l);
                const uint64_t i1 = lower_bound_u64(a.B, a.ncells, base + hi_l + 1);
                if (i0 < i1) rg = make_uint2(a.G[i0].x, a.G[i1 - 1].y);
            }
            s_rng[warp][r] = rg;
        }
        __syncwarp();
        float a2[NP];
        float na = 0.f;
#pragma unroll
        for (int d = 0; d < NP; ++d) {
            const float v = d < (int)n ? (by_id ? a.Xf[(uint64_t)d * a.Npad + qid]
                                                : a.Xs[(uint64_t)d * a.Npad + qp])
                                       : 0.f;
            a2[d] = -2.f * v;
            na = fmaf(v, v, na);
        }
        const float Aq = sqrtf(na) * 1.0001f;
        const double* qx = a.X64 + (uint64_t)qid * n;
        for (uint32_t r = 0; r < R; ++r) {
            const uint2 rg = s_rng[warp][r];
            for (uint32_t t = rg.x + lane; t < rg.y; t += 32) {
                float nb = 0.f, acc = 0.f;
#pragma unroll
                for (int d = 0; d < NP; ++d) {
                    const float b = d < (int)n ? a.Xs[(uint64_t)d * a.Npad + t] : 0.f;
                    nb = fmaf(b, b, nb);
                    acc = fmaf(a2[d], b, acc);
                }
                acc += nb;
                const float dl = screen_delta(Aq, sqrtf(nb) * 1.0001f, a.gam, a.erg, a.eab, a.e64);
                if (!(acc < __fsub_ru(__fadd_ru(lo_end, dl), na)) || (by_id ? a.A[t] == qid : t == qp))
                    continue;
                const float key = acc + na;
                const float klo = __fsub_rd(key, dl), khi = __fadd_ru(key, dl);
                int b = key > 0.f ? (int)(key * rsqrtf(key) * invw) : 0;
                b = min(max(b, 0), (int)nbins - 1);
                uint32_t bb = nbins;
                if (klo >= s_lo[b] && khi < s_hi[b]) {
                    bb = (uint32_t)b;
                } else {
                    const double sq = exact_sq(qx, a.X64 + (uint64_t)a.A[t] * n, n);
                    if (!(sq > a.limit_sq)) {
                        const double dist = sqrt(sq);
                        if (dist < a.eps_mean) {
                            uint64_t e = (uint64_t)(dist * a.inv_width);
                            bb = e >= nbins ? nbins - 1 : (uint32_t)e;
                        }
                    }
                }
                if (bb < ncount) atomicAdd(&s_hist[warp][bb], 1u);
            }
        }
    }
    __syncthreads();
    for (uint32_t b = threadIdx.x; b < ncount; b += blockDim.x) {
        unsigned long long sum = 0;
        for (int w = 0; w < WARPS; ++w) sum += s_hist[w][b];
        if (sum) atomicAdd(&a.counts[b], sum);
    }
}

void launch_hist_grid(const HistGridArgs& a, cudaStream_t s) {
    if (a.nq == 0) return;
    if (a.m < 1 || a.m > 6 || a.n > 8 || a.n_bins > 256 || a.n_count > a.n_bins)
        throw Error(1, "grid histogram: unsupported shape");
    const unsigned blocks = (unsigned)std::min<uint64_t>((a.nq + 7) / 8, 148ull * 16);
    switch (a.n) {
#define X(v) \
    case v: k_hist_grid<v><<<blocks, 256, 0, s>>>(a); break;
        X(1) X(2) X(3) X(4) X(5) X(6) X(7) X(8)
#undef X
    }
    KJ_CUDA(cudaGetLastError());
    g_launches.fetch_add(1, std::memory_order_relaxed);
}

// ---------------------------------------------------------------- small kernels
__global__ void k_check_finite(const double* X, uint64_t count, unsigned long long* first_bad) {
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < count;
         i += uint64_t(gridDim.x) * blockDim.x)
        if (!isfinite(X[i])) atomicMin(first_bad, (unsigned long long)i);
}
void launch_check_finite(const double* X, uint64_t count, unsigned long long* first_bad,
                         cudaStream_t s) {
    k_check_finite<<<1184, 256, 0, s>>>(X, count, first_bad);
    KJ_CUDA(cudaGetLastError());
    g_launches.fetch_add(1, std::memory_order_relaxed);
}

// Column sums (mean == null) or sums of squared deviations, per row-block:
// partial[blk*n + j]. Fixed partition and order -> deterministic.
__global__ void k_col_sums(const double* X, uint64_t N, uint32_t n, const double* mean,
                           double* partial) {
    __shared__ double red[8][33];
    const uint32_t j = blockIdx.y * 32 + threadIdx.x;
    const uint64_t rows_per = (N + gridDim.x - 1) / gridDim.x;
    const uint64_t r0 = uint64_t(blockIdx.x) * rows_per, r1 = min(N, r0 + rows_per);
    double s = 0.0;
    if (j < n) {
        const double mj = mean ? mean[j] : 0.0;
        for (uint64_t i = r0 + threadIdx.y; i < r1; i += 8) {
            double v = X[i * n + j];
            if (mean) {
                v = v - mj;
                s += v * v;
            } else {
                s += v;
            }
        }
    }
    red[threadIdx.y][threadIdx.x] = s;
    __syncthreads();
    if (threadIdx.y == 0 && j < n) {
        double t = 0.0;
        for (int y = 0; y < 8; ++y) t += red[y][threadIdx.x];
        partial[uint64_t(blockIdx.x) * n + j] = t;
    }
}
void launch_col_sums(const double* X, uint64_t N, uint32_t n, const double* mean,
                     double* partial, uint32_t nblk, cudaStream_t s) {
    dim3 grid(nblk, (n + 31) / 32), block(32, 8);
    k_col_sums<<<grid, block, 0, s>>>(X, N, n, mean, partial);
    KJ_CUDA(cudaGetLastError());
    g_launches.fetch_add(1, std::memory_order_relaxed);
}

__global__ void k_permute_cols(const double* X0, double* X, uint64_t N, uint32_t n,
                               const uint32_t* order) {
    for (uint64_t e = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < N * n;
         e += uint64_t(gridDim.x) * blockDim.x) {
        uint64_t i = e / n;
        uint32_t j = (uint32_t)(e - i * n);
        X[e] = X0[i * n + order[j]];
    }
}
void launch_permute_cols(const double* X0, double* X, uint64_t N, uint32_t n,
                         const uint32_t* order, cudaStream_t s) {
    k_permute_cols<<<2368, 256, 0, s>>>(X0, X, N, n, order);
    KJ_CUDA(cudaGetLastError());
    g_launches.fetch_add(1, std::memory_order_relaxed);
}

__global__ void k_to_float_soa(const double* X, uint64_t N, uint32_t n, const double* g,
                               float* Xf, uint64_t Npad, unsigned long long* rmax_bits) {
    double rmax = 0.0;
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < Npad;
         i += uint64_t(gridDim.x) * blockDim.x) {
        double r2 = 0.0;
        for (uint32_t d = 0; d < n; ++d) {
            float v = 0.f;
            if (i < N) {
                double dv = X[i * n + d] - g[d];
                r2 += dv * dv;
                v = (float)dv;
            }
            Xf[uint64_t(d) * Npad + i] = v;
        }
        rmax = fmax(rmax, r2);
    }
    for (int o = 16; o > 0; o >>= 1) rmax = fmax(rmax, __shfl_xor_sync(0xffffffffu, rmax, o));
    if ((threadIdx.x & 31) == 0) atomicMax(rmax_bits, (unsigned long long)__double_as_longlong(rmax));
}
void launch_to_float_soa(const double* X, uint64_t N, uint32_t n, const double* g, float* Xf,
                         uint64_t Npad, unsigned long long* rmax_bits, cudaStream_t s) {
    k_to_float_soa<<<1184, 256, 0, s>>>(X, N, n, g, Xf, Npad, rmax_bits);
    KJ_CUDA(cudaGetLastError());
    g_launches.fetch_add(1, std::memory_order_relaxed);
}

__global__ void k_pair_sq(const double* X, uint32_t n, const uint64_t* ij, uint64_t npairs,
                          double limit, double* out) {
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < npairs;
         i += uint64_t(gridDim.x) * blockDim.x) {
        double s = exact_sq(X + ij[2 * i] * n, X + ij[2 * i + 1] * n, n);
        out[i] = s > limit ? CUDART_INF : s;
    }
}
void launch_pair_sq(const double* X, uint32_t n, const uint64_t* ij, uint64_t npairs,
                    double limit, double* out, cudaStream_t s) {
    if (!npairs) return;
    k_pair_sq<<<(unsigned)std::min<uint64_t>(4736, (npairs + 255) / 256), 256, 0, s>>>(
        X, n, ij, npairs, limit, out);
    KJ_CUDA(cudaGetLastError());
    g_launches.fetch_add(1, std::memory_order_relaxed);
}

__global__ void k_minmax(const double* X, uint64_t N, uint32_t n, uint32_t m,
                         unsigned long long* mn, unsigned long long* mx) {
    for (uint32_t j = 0; j < m; ++j) {
        unsigned long long lo = ~0ull, hi = 0ull;
        for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < N;
             i += uint64_t(gridDim.x) * blockDim.x) {
            unsigned long long o = dbl_order(X[i * n + j]);
            lo = o < lo ? o : lo;
            hi = o > hi ? o : hi;
        }
        for (int off = 16; off > 0; off >>= 1) {
            unsigned long long l2 = __shfl_xor_sync(0xffffffffu, lo, off);
            unsigned long long h2 = __shfl_xor_sync(0xffffffffu, hi, off);
            lo = l2 < lo ? l2 : lo;
            hi = h2 > hi ? h2 : hi;
        }
        if ((threadIdx.x & 31) == 0) {
            atomicMin(&mn[j], lo);
            atomicMax(&mx[j], hi);
        }
    }
}
void launch_minmax(const double* X, uint64_t N, uint32_t n, uint32_t m, unsigned long long* mn,
                   unsigned long long* mx, cudaStream_t s) {
    k_minmax<<<592, 256, 0, s>>>(X, N, n, m, mn, mx);
    KJ_CUDA(cudaGetLastError());
    g_launches.fetch_add(1, std::memory_order_relaxed);
}

// grid_index.cpp:77-94 (cell_of + linearize), FP64 division and floor
__global__ void k_cell_keys(const double* X, uint64_t N, uint32_t n, uint32_t m,
                            const double* mins, double w, const uint64_t* cpd,
                            const uint64_t* strides, uint64_t* keys, uint32_t* vals, uint32_t base) {
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < N;
         i += uint64_t(gridDim.x) * blockDim.x) {
        uint64_t id = 0;
        for (uint32_t j = 0; j < m; ++j) {
            double rel = __ddiv_rn(__dsub_rn(X[i * n + j], mins[j]), w);
            if (rel < 0.0) rel = 0.0;
            uint64_t idx = (uint64_t)floor(rel);
            if (idx > cpd[j] - 1) idx = cpd[j] - 1;
            id += idx * strides[j];
        }
        keys[i] = id;
        vals[i] = base + (uint32_t)i;
    }
}
// cell keys of arbitrary points (ids), same rule as k_cell_keys
__global__ void k_id_cell_keys(const double* X, const uint32_t* ids, uint64_t cnt, uint32_t n, uint32_t m,
                               const double* mins, double w, const uint64_t* cpd,
                               const uint64_t* strides, uint64_t* keys) {
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < cnt;
         i += uint64_t(gridDim.x) * blockDim.x) {
        const double* x = X + (uint64_t)ids[i] * n;
        uint64_t id = 0;
        for (uint32_t j = 0; j < m; ++j) {
            double rel = __ddiv_rn(__dsub_rn(x[j], mins[j]), w);
            if (rel < 0.0) rel = 0.0;
            uint64_t idx = (uint64_t)floor(rel);
            if (idx > cpd[j] - 1) idx = cpd[j] - 1;
            id += idx * strides[j];
        }
        keys[i] = id;
    }
}
void launch_id_cell_keys(const double* X, const uint32_t* ids, uint64_t cnt, uint32_t n, uint32_t m,
                         const double* mins, double w, const uint64_t* cpd, const uint64_t* strides,
                         uint64_t* keys, cudaStream_t s) {
    if (!cnt) return;
    k_id_cell_keys<<<(unsigned)std::min<uint64_t>((cnt + 255) / 256, 2368), 256, 0, s>>>(
        X, ids, cnt, n, m, mins, w, cpd, strides, keys);
    KJ_CUDA(cudaGetLastError());
    g_launches.fetch_add(1, std::memory_order_relaxed);
}
void launch_cell_keys(const double* X, uint64_t N, uint32_t n, uint32_t m, const double* mins,
                      double w, const uint64_t* cpd, const uint64_t* strides, uint64_t* keys,
                      uint32_t* vals, cudaStream_t s, uint32_t base) {
    k_cell_keys<<<2368, 256, 0, s>>>(X, N, n, m, mins, w, cpd, strides, keys, vals, base);
    KJ_CUDA(cudaGetLastError());
    g_launches.fetch_add(1, std::memory_order_relaxed);
}

__global__ void k_iota(uint32_t* v, uint64_t N) {
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < N;
         i += uint64_t(gridDim.x) * blockDim.x)
        v[i] = (uint32_t)i;
}
void launch_iota(uint32_t* v, uint64_t N, cudaStream_t s) {
    k_iota<<<1184, 256, 0, s>>>(v, N);
    KJ_CUDA(cudaGetLastError());
    g_launches.fetch_add(1, std::memory_order_relaxed);
}

__global__ void k_head_flags(const uint64_t* keys, uint64_t N, uint32_t* flags) {
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < N;
         i += uint64_t(gridDim.x) * blockDim.x)
        flags[i] = (i == 0 || keys[i] != keys[i - 1]) ? 1u : 0u;
}
void launch_head_flags(const uint64_t* keys, uint64_t N, uint32_t* flags, cudaStream_t s) {
    k_head_flags<<<1184, 256, 0, s>>>(keys, N, flags);
    KJ_CUDA(cudaGetLastError());
    g_launches.fetch_add(1, std::memory_order_relaxed);
}

// runidx: inclusive scan of head flags (1-based run number)
__global__ void k_grid_tables(const uint64_t* skeys, const uint32_t* A, const uint32_t* runidx,
                              uint64_t N, uint64_t* B, uint2* G, uint32_t* slot,
                              uint32_t* posOf) {
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < N;
         i += uint64_t(gridDim.x) * blockDim.x) {
        const uint32_t r = runidx[i] - 1;
        const uint64_t k = skeys[i];
        if (i == 0 || skeys[i - 1] != k) {
            B[r] = k;
            G[r].x = (uint32_t)i;
        }
        if (i == N - 1 || skeys[i + 1] != k) G[r].y = (uint32_t)(i + 1);
        if (slot) slot[A[i]] = r;          // (scattered writes: skipped when not needed)
        if (posOf) posOf[A[i]] = (uint32_t)i;
    }
}
void launch_grid_tables(const uint64_t* skeys, const uint32_t* A, const uint32_t* runidx,
                        uint64_t N, uint64_t* B, uint2* G, uint32_t* slot, uint32_t* posOf,
                        cudaStream_t s) {
    k_grid_tables<<<1184, 256, 0, s>>>(skeys, A, runidx, N, B, G, slot, posOf);
    KJ_CUDA(cudaGetLastError());
    g_launches.fetch_add(1, std::memory_order_relaxed);
}

// FP32 SoA rows in a grid's position order (A: position -> point), gathered from the
// FP64 point rows: (float)(x - g), the value k_to_float_soa stores, from one contiguous
// 8n-byte row per point instead of n scattered 4-byte reads of the SoA copy (one sector
// instead of four at n = 4)
__global__ void k_gather_x64(const double* X, const double* g, const uint32_t* A, uint64_t N,
                             uint32_t n, uint64_t Npad, float* Xs) {
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < Npad;
         i += uint64_t(gridDim.x) * blockDim.x) {
        if (i < N) {
            const double* x = X + (uint64_t)A[i] * n;
            for (uint32_t d = 0; d < n; ++d) Xs[uint64_t(d) * Npad + i] = (float)(x[d] - g[d]);
        } else {
            for (uint32_t d = 0; d < n; ++d) Xs[uint64_t(d) * Npad + i] = 0.f;
        }
    }
}
void launch_gather_x64(const double* X, const double* g, const uint32_t* A, uint64_t N, uint32_t n,
                       uint64_t Npad, float* Xs, cudaStream_t s) {
    k_gather_x64<<<2368, 256, 0, s>>>(X, g, A, N, n, Npad, Xs);
    KJ_CUDA(cudaGetLastError());
    g_launches.fetch_add(1, std::memory_order_relaxed);
}

__global__ void k_map_u32(const uint32_t* idx, const uint32_t* table, uint64_t n, uint32_t* out) {
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += uint64_t(gridDim.x) * blockDim.x)
        out[i] = table[idx[i]];
}
void launch_map_u32(const uint32_t* idx, const uint32_t* table, uint64_t n, uint32_t* out,
                    cudaStream_t s) {
    if (!n) return;
    k_map_u32<<<1184, 256, 0, s>>>(idx, table, n, out);
    KJ_CUDA(cudaGetLastError());
    g_launches.fetch_add(1, std::memory_order_relaxed);
}


// One warp per cell: the 3^(m-1) rows of the clamped ±1 neighbourhood over
// the first m-1 indexed dims; each row is the contiguous B-range of linear ids
// [row + lo_last, row + hi_last] (grid_index.cpp:114-147 enumerates exactly
// these cells). The cell's own row is emitted first.
// spans (optional): a work unit is a run of `span` cells along the last dim starting at
// cells[w]; its rows then cover [c - 1, c + span] along that dim (the union of the cells'
// neighbourhoods, a superset for every query of the run)
template <bool FILL>
__global__ void k_adj(const uint64_t* B, const uint2* G, uint64_t ncells, const uint32_t* cells,
                      uint64_t nc, uint32_t m, const uint64_t* cpd, const uint64_t* strides,
                      uint32_t* counts, const uint32_t* offs, uint2* adj,
                      unsigned long long* csize, const uint32_t* spans, const uint16_t* order) {
    const uint64_t w = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (w >= nc) return;
    const uint64_t lin = B[cells[w]];
    uint64_t c[64];
    {
        uint64_t r = lin;
        for (uint32_t j = 0; j < m; ++j) {
            c[j] = r / strides[j];
            r -= c[j] * strides[j];
        }
    }
    const uint32_t ml = m - 1;
    uint64_t R = 1;
    for (uint32_t j = 0; j < ml; ++j) R *= 3;
    const uint64_t own = (R - 1) / 2;
    const uint64_t lo_l = c[ml] > 0 ? c[ml] - 1 : 0;
    const uint64_t hi_l = min(c[ml] + (spans ? spans[w] : 1u), cpd[ml] - 1);
    uint32_t written = 0;
    unsigned long long sz = 0;
    // process own row first (iteration -1), then all rows != own; with `order` (own row
    // first, then by the number of offset dims: the nearer rows first) in one sweep
    for (int64_t base = order ? 0 : -32; base < (int64_t)R; base += 32) {
        int64_t r = base + lane;
        bool valid = false;
        uint2 rng = make_uint2(0, 0);
        if (order) {
            r = r < (int64_t)R ? (int64_t)order[r] : -1;
        } else if (base < 0) {
            if (lane == 0) r = (int64_t)own;
            else r = -1;
        } else if (r >= (int64_t)R || (uint64_t)r == own) {
            r = -1;
        }
        if (r >= 0) {
            uint64_t row = 0, t = (uint64_t)r;
            bool ok = true;
            for (int j = (int)ml - 1; j >= 0; --j) {
                const uint64_t dig = t % 3;
                t /= 3;
                const int64_t cj = (int64_t)c[j] - 1 + (int64_t)dig;
                if (cj < 0 || cj >= (int64_t)cpd[j]) {
                    ok = false;
                    break;
                }
                row += (uint64_t)cj * strides[j];
            }
            if (ok) {
                const uint64_t s_lo = lower_bound_u64(B, ncells, row + lo_l);
                const uint64_t s_hi = lower_bound_u64(B, ncells, row + hi_l + 1);
                if (s_lo < s_hi) {
                    valid = true;
                    if (G) rng = make_uint2(G[s_lo].x, G[s_hi - 1].y);  // (count pass: may be null)
                }
            }
        }
        const unsigned bal = __ballot_sync(0xffffffffu, valid);
        if (FILL && valid) {
            const uint32_t at = offs[w] + written + __popc(bal & ((1u << lane) - 1u));
            adj[at] = rng;
        }
        if (valid) sz += rng.y - rng.x;
        written += __popc(bal);
    }
    for (int o = 16; o > 0; o >>= 1) sz += __shfl_xor_sync(0xffffffffu, sz, o);
    if (lane == 0) {
        if (!FILL) counts[w] = written;
        if (csize) csize[w] = sz;
    }
}
// Per launch row (cells' rows contiguous from ufirst): its cell's neighbourhood size.
__global__ void k_row_walk(const uint32_t* ufirst, const uint32_t* ucnt, uint64_t nuc,
                           const unsigned long long* csize, unsigned long long* rowwalk) {
    for (uint64_t u = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; u < nuc;
         u += uint64_t(gridDim.x) * blockDim.x)
        for (uint32_t i = 0; i < ucnt[u]; ++i) rowwalk[ufirst[u] + i] = csize[u];
}
// sums of rowwalk over n rows: all (out[0]) and those whose output row is dense (out[1])
__global__ void k_walk_sum(const unsigned long long* rowwalk, const uint32_t* qrow, uint64_t n,
                           const uint8_t* dense, unsigned long long* out) {
    unsigned long long a = 0, d = 0;
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += uint64_t(gridDim.x) * blockDim.x) {
        a += rowwalk[i];
        if (dense && dense[qrow[i]]) d += rowwalk[i];
    }
    for (int o = 16; o > 0; o >>= 1) {
        a += __shfl_xor_sync(0xffffffffu, a, o);
        d += __shfl_xor_sync(0xffffffffu, d, o);
    }
    if ((threadIdx.x & 31) == 0) {
        atomicAdd(out, a);
        atomicAdd(out + 1, d);
    }
}
void launch_row_walk(const uint32_t* ufirst, const uint32_t* ucnt, uint64_t nuc,
                     const unsigned long long* csize, unsigned long long* rowwalk, cudaStream_t s) {
    if (!nuc) return;
    k_row_walk<<<(unsigned)std::min<uint64_t>((nuc + 255) / 256, 148 * 16), 256, 0, s>>>(ufirst, ucnt, nuc,
                                                                                         csize, rowwalk);
    KJ_CUDA(cudaGetLastError());
    g_launches.fetch_add(1, std::memory_order_relaxed);
}
void launch_walk_sum(const unsigned long long* rowwalk, const uint32_t* qrow, uint64_t n,
                     const uint8_t* dense, unsigned long long* out, cudaStream_t s) {
    if (!n) return;
    k_walk_sum<<<(unsigned)std::min<uint64_t>((n + 255) / 256, 148 * 8), 256, 0, s>>>(rowwalk, qrow, n,
                                                                                      dense, out);
    KJ_CUDA(cudaGetLastError());
    g_launches.fetch_add(1, std::memory_order_relaxed);
}
void launch_adj_count(const uint64_t* B, uint64_t ncells, const uint32_t* cells, uint64_t nc,
                      uint32_t m, const uint64_t* cpd, const uint64_t* strides,
                      uint32_t* counts, cudaStream_t s, const uint32_t* spans, const uint2* G,
                      unsigned long long* csize) {
    if (!nc) return;
    k_adj<false><<<(unsigned)((nc * 32 + 255) / 256), 256, 0, s>>>(
        B, G, ncells, cells, nc, m, cpd, strides, counts, nullptr, nullptr, csize, spans, nullptr);
    KJ_CUDA(cudaGetLastError());
    g_launches.fetch_add(1, std::memory_order_relaxed);
}
void launch_adj_fill(const uint64_t* B, const uint2* G, uint64_t ncells, const uint32_t* cells,
                     uint64_t nc, uint32_t m, const uint64_t* cpd, const uint64_t* strides,
                     const uint32_t* offs, uint2* adj, unsigned long long* csize,
                     cudaStream_t s, const uint32_t* spans, const uint16_t* order) {
    if (!nc) return;
    k_adj<true><<<(unsigned)((nc * 32 + 255) / 256), 256, 0, s>>>(
        B, G, ncells, cells, nc, m, cpd, strides, nullptr, offs, adj, csize, spans, order);
    KJ_CUDA(cudaGetLastError());
    g_launches.fetch_add(1, std::memory_order_relaxed);
}

__global__ void k_items(const uint32_t* ufirst, const uint32_t* ucnt, const uint32_t* item_off,
                        const uint32_t* adj_off, uint64_t nuc, const unsigned long long* csize,
                        uint4* items, unsigned long long* work, uint32_t chunk) {
    for (uint64_t u = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; u < nuc;
         u += uint64_t(gridDim.x) * blockDim.x) {
        const uint32_t f = ufirst[u], c = ucnt[u];
        const uint32_t i0 = item_off[u];
        const uint32_t nit = (c + chunk - 1) / chunk;
        for (uint32_t t = 0; t < nit; ++t) {
            const uint32_t qb = f + t * chunk, qe = min(f + c, qb + chunk);
            items[i0 + t] = make_uint4(qb, qe, adj_off[u], adj_off[u + 1]);
            work[i0 + t] = (unsigned long long)(qe - qb) * csize[u];
        }
    }
}
void launch_items(const uint32_t* ufirst, const uint32_t* ucnt, const uint32_t* item_off,
                  const uint32_t* adj_off, uint64_t nuc, const unsigned long long* csize,
                  uint4* items, unsigned long long* work, uint32_t chunk, cudaStream_t s) {
    if (!nuc) return;
    k_items<<<592, 256, 0, s>>>(ufirst, ucnt, item_off, adj_off, nuc, csize, items, work, chunk);
    KJ_CUDA(cudaGetLastError());
    g_launches.fetch_add(1, std::memory_order_relaxed);
}

__global__ void k_cell_pop(const uint32_t* pids, uint64_t nq, const uint32_t* slot,
                           const uint2* G, uint32_t* pop) {
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < nq;
         i += uint64_t(gridDim.x) * blockDim.x) {
        const uint2 g = G[slot[pids[i]]];
        pop[i] = g.y - g.x;
    }
}
void launch_cell_pop(const uint32_t* pids, uint64_t nq, const uint32_t* slot, const uint2* G,
                     uint32_t* pop, cudaStream_t s) {
    if (!nq) return;
    k_cell_pop<<<1184, 256, 0, s>>>(pids, nq, slot, G, pop);
    KJ_CUDA(cudaGetLastError());
    g_launches.fetch_add(1, std::memory_order_relaxed);
}

__global__ void k_fill_f32(float* p, uint64_t n, float v) {
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += uint64_t(gridDim.x) * blockDim.x)
        p[i] = v;
}
void launch_fill_f32(float* p, uint64_t n, float v, cudaStream_t s) {
    if (!n) return;
    k_fill_f32<<<1184, 256, 0, s>>>(p, n, v);
    KJ_CUDA(cudaGetLastError());
    g_launches.fetch_add(1, std::memory_order_relaxed);
}

// range_query sizes (self included) over a pass: block per item, warp per query.
__global__ void k_range_count(const double* X64, uint32_t n, const uint32_t* A,
                              const uint32_t* qpos, const uint4* items, const uint2* adj,
                              double eps2, unsigned long long* in_eps) {
    const uint4 it = items[blockIdx.x];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    for (uint32_t r = it.x + warp; r < it.y; r += nw) {
        const uint32_t qid = A[qpos[r]];
        const double* qx = X64 + (uint64_t)qid * n;
        unsigned long long cnt = 0;
        for (uint32_t ri = it.z; ri < it.w; ++ri) {
            const uint2 g = adj[ri];
            for (uint32_t p = g.x + lane; p < g.y; p += 32)
                cnt += exact_sq(qx, X64 + (uint64_t)A[p] * n, n) <= eps2;
        }
        for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
        if (lane == 0) in_eps[r] = cnt;
    }
}
void launch_range_count(const double* X64, uint32_t n, const uint32_t* A, const uint32_t* qpos,
                        const uint4* items, uint64_t nitems, const uint2* adj, double eps2,
                        unsigned long long* in_eps, cudaStream_t s) {
    if (!nitems) return;
    k_range_count<<<(unsigned)nitems, 128, 0, s>>>(X64, n, A, qpos, items, adj, eps2, in_eps);
    KJ_CUDA(cudaGetLastError());
    g_launches.fetch_add(1, std::memory_order_relaxed);
}

// Exact slow path for rows whose screened list overflowed (many exact ties):
// one warp per row, per-lane sorted top-K in shared memory, warp merge.
__global__ void k_slow_exact(const double* X64, uint32_t n, const uint32_t* A,
                             const uint32_t* qpos, const uint32_t* qrow, const uint32_t* rows,
                             uint64_t nrows, const uint4* items, const uint32_t* row_item,
                             const uint2* adj, uint32_t K, double eps2, double cover2,
                             uint32_t* out_ids, double* out_dist, double* out_kth,
                             uint8_t* out_status, double* out_sq, uint32_t* out_count) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    double* ls = reinterpret_cast<double*>(smem_raw);      // [K][32]
    uint32_t* li = reinterpret_cast<uint32_t*>(ls + K * 32);  // [K][32]
    const int lane = threadIdx.x;
    const uint64_t ri = blockIdx.x;
    if (ri >= nrows) return;
    const uint32_t row = rows[ri];
    const uint4 it = items[row_item[row]];
    const uint32_t qp = qpos[row];
    const uint32_t qid = A[qp];
    const double* qx = X64 + (uint64_t)qid * n;
    uint32_t cnt = 0;
    for (uint32_t r = it.z; r < it.w; ++r) {
        const uint2 g = adj[r];
        for (uint32_t p = g.x + lane; p < g.y; p += 32) {
            if (p == qp) continue;
            const uint32_t t = A[p];
            const double s = exact_sq(qx, X64 + (uint64_t)t * n, n);
            if (cnt == K && !pair_less(s, t, ls[(K - 1) * 32 + lane], li[(K - 1) * 32 + lane]))
                continue;
            int q = (int)(cnt < K ? cnt : K - 1);
            while (q > 0 && pair_less(s, t, ls[(q - 1) * 32 + lane], li[(q - 1) * 32 + lane])) {
                ls[q * 32 + lane] = ls[(q - 1) * 32 + lane];
                li[q * 32 + lane] = li[(q - 1) * 32 + lane];
                --q;
            }
            ls[q * 32 + lane] = s;
            li[q * 32 + lane] = t;
            if (cnt < K) ++cnt;
        }
    }
    uint32_t head = 0;
    uint32_t total = cnt;
    for (int o = 16; o > 0; o >>= 1) total += __shfl_xor_sync(0xffffffffu, total, o);
    const uint32_t orow = qrow[row];
    double kth = CUDART_INF;
    const uint32_t outn = min(total, K);
    for (uint32_t r = 0; r < outn; ++r) {
        double s = head < cnt ? ls[head * 32 + lane] : CUDART_INF;
        uint32_t t = head < cnt ? li[head * 32 + lane] : 0xFFFFFFFFu;
        double bs = s;
        uint32_t bt = t;
        for (int o = 16; o > 0; o >>= 1) {
            double s2 = __shfl_xor_sync(0xffffffffu, bs, o);
            uint32_t t2 = __shfl_xor_sync(0xffffffffu, bt, o);
            if (pair_less(s2, t2, bs, bt)) {
                bs = s2;
                bt = t2;
            }
        }
        if (head < cnt && t == bt) ++head;
        if (lane == 0) {
            out_ids[(uint64_t)orow * K + r] = bt;
            out_dist[(uint64_t)orow * K + r] = sqrt(bs);
            if (out_sq) out_sq[(uint64_t)orow * K + r] = bs;
        }
        kth = bs;
    }
    if (lane == 0) {
        uint8_t st = 0;
        if (total >= K) {
            st |= ST_HAS_K;
            if (kth <= eps2) st |= ST_IN_EPS;
            if (kth < cover2) st |= ST_CERT;
        }
        out_status[orow] = st;
        out_kth[orow] = total >= K ? kth : CUDART_INF;
        if (out_count) out_count[orow] = outn;
    }
}
void launch_slow_exact(const double* X64, uint32_t n, const uint32_t* A, const uint32_t* qpos,
                       const uint32_t* qrow, const uint32_t* rows, uint64_t nrows,
                       const uint4* items, const uint32_t* row_item, const uint2* adj,
                       uint32_t K, double eps2, double cover2, uint32_t* out_ids,
                       double* out_dist, double* out_kth, uint8_t* out_status, double* out_sq,
                       uint32_t* out_count, cudaStream_t s) {
    if (!nrows) return;
    size_t sm = (size_t)K * 32 * (sizeof(double) + sizeof(uint32_t));
    set_smem(k_slow_exact, sm);
    k_slow_exact<<<(unsigned)nrows, 32, sm, s>>>(X64, n, A, qpos, qrow, rows, nrows, items,
                                                 row_item, adj, K, eps2, cover2, out_ids,
                                                 out_dist, out_kth, out_status, out_sq, out_count);
    KJ_CUDA(cudaGetLastError());
    g_launches.fetch_add(1, std::memory_order_relaxed);
}

}  // namespace kj

namespace kj {
__global__ void k_row_item(const uint4* items, uint64_t nitems, uint32_t* row_item) {
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < nitems;
         i += uint64_t(gridDim.x) * blockDim.x) {
        const uint4 it = items[i];
        for (uint32_t r = it.x; r < it.y; ++r) row_item[r] = (uint32_t)i;
    }
}
void launch_row_item(const uint4* items, uint64_t nitems, uint32_t* row_item, cudaStream_t s) {
    if (!nitems) return;
    k_row_item<<<592, 256, 0, s>>>(items, nitems, row_item);
    KJ_CUDA(cudaGetLastError());
    g_launches.fetch_add(1, std::memory_order_relaxed);
}
}  // namespace kj

namespace kj {
template <class T>
__global__ void k_gather(const uint32_t* idx, const T* table, uint64_t n, T* out) {
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += uint64_t(gridDim.x) * blockDim.x)
        out[i] = table[idx[i]];
}
void launch_gather_u8(const uint32_t* idx, const uint8_t* table, uint64_t n, uint8_t* out,
                      cudaStream_t s) {
    if (!n) return;
    k_gather<uint8_t><<<592, 256, 0, s>>>(idx, table, n, out);
    KJ_CUDA(cudaGetLastError());
    g_launches.fetch_add(1, std::memory_order_relaxed);
}
void launch_gather_f64(const uint32_t* idx, const double* table, uint64_t n, double* out,
                       cudaStream_t s) {
    if (!n) return;
    k_gather<double><<<592, 256, 0, s>>>(idx, table, n, out);
    KJ_CUDA(cudaGetLastError());
    g_launches.fetch_add(1, std::memory_order_relaxed);
}
void launch_gather_f32(const uint32_t* idx, const float* table, uint64_t n, float* out,
                       cudaStream_t s) {
    if (!n) return;
    k_gather<float><<<592, 256, 0, s>>>(idx, table, n, out);
    KJ_CUDA(cudaGetLastError());
    g_launches.fetch_add(1, std::memory_order_relaxed);
}
}  // namespace kj

namespace kj {
// FP32 roofline denominator: 8 independent FFMA chains per thread, register
// operands (the form the distance kernels issue), full-chip grid.
__global__ void k_ffma_peak(float* out, int iters, float a, float b) {
    float x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5,
          x6 = x0 + 6, x7 = x0 + 7;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int u = 0; u < 16; ++u) {
            x0 = fmaf(x0, a, b); x1 = fmaf(x1, a, b); x2 = fmaf(x2, a, b); x3 = fmaf(x3, a, b);
            x4 = fmaf(x4, a, b); x5 = fmaf(x5, a, b); x6 = fmaf(x6, a, b); x7 = fmaf(x7, a, b);
        }
    }
    float r = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
    if (r == 1234.5f) out[0] = r;
}
double measure_ffma_tflops(cudaStream_t s) {
    int dev = 0, sms = 0;
    KJ_CUDA(cudaGetDevice(&dev));
    KJ_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    float* out = nullptr;
    KJ_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&out), 4, s));
    const int blocks = sms * 8, threads = 256, iters = 4096;
    cudaEvent_t a, b;
    KJ_CUDA(cudaEventCreate(&a));
    KJ_CUDA(cudaEventCreate(&b));
    k_ffma_peak<<<blocks, threads, 0, s>>>(out, 64, 0.999f, 0.001f);  // warm-up
    KJ_CUDA(cudaEventRecord(a, s));
    k_ffma_peak<<<blocks, threads, 0, s>>>(out, iters, 0.999f, 0.001f);
    KJ_CUDA(cudaEventRecord(b, s));
    KJ_CUDA(cudaEventSynchronize(b));
    float ms = 0;
    KJ_CUDA(cudaEventElapsedTime(&ms, a, b));
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    cudaFreeAsync(out, s);
    const double flops = 2.0 * 8 * 16 * double(iters) * blocks * threads;
    return flops / (ms * 1e-3) / 1e12;
}
}  // namespace kj

namespace kj {
__global__ void k_scale_f32(const float* in, uint64_t n, float scale, float* out) {
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += uint64_t(gridDim.x) * blockDim.x)
        out[i] = in[i] * scale;
}
void launch_scale_f32(const float* in, uint64_t n, float scale, float* out, cudaStream_t s) {
    if (!n) return;
    k_scale_f32<<<592, 256, 0, s>>>(in, n, scale, out);
    KJ_CUDA(cudaGetLastError());
    g_launches.fetch_add(1, std::memory_order_relaxed);
}
}  // namespace kj

namespace kj {
// Join-order keys: (cell slot, Morton code of the point over the first `dims`
// working dims, 3 bits each). Points of one cell stay contiguous (same ranges
// as the reference order) but are laid out along a space-filling curve.
__global__ void k_morton_keys(const double* X64, const uint32_t* A, const uint32_t* slot,
                              uint64_t N, uint32_t n, uint32_t dims, const double* lo,
                              const double* inv_range, uint64_t* keys, uint32_t* vals,
                              uint32_t bits) {
    const uint32_t cb = dims * bits;
    const double lv = double(1u << bits);
    const uint32_t qmax = (1u << bits) - 1u;
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < N;
         i += uint64_t(gridDim.x) * blockDim.x) {
        const uint32_t pid = A[i];
        const double* x = X64 + (uint64_t)pid * n;
        uint64_t code = 0;
        for (int bit = (int)bits - 1; bit >= 0; --bit)
            for (uint32_t d = 0; d < dims; ++d) {
                double f = (x[d] - lo[d]) * inv_range[d];
                uint32_t q = f <= 0.0 ? 0u : (f >= 1.0 ? qmax : min(qmax, (uint32_t)(f * lv)));
                code = (code << 1) | ((q >> bit) & 1u);
            }
        keys[i] = (cb >= 64 ? 0ull : ((uint64_t)slot[pid] << cb)) | code;
        vals[i] = pid;
    }
}
void launch_morton_keys(const double* X64, const uint32_t* A, const uint32_t* slot, uint64_t N,
                        uint32_t n, uint32_t dims, const double* lo, const double* inv_range,
                        uint64_t* keys, uint32_t* vals, cudaStream_t s, uint32_t bits) {
    k_morton_keys<<<2368, 256, 0, s>>>(X64, A, slot, N, n, dims, lo, inv_range, keys, vals, bits);
    KJ_CUDA(cudaGetLastError());
    g_launches.fetch_add(1, std::memory_order_relaxed);
}
__global__ void k_inverse(const uint32_t* J, uint64_t N, uint32_t* posJ) {
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < N;
         i += uint64_t(gridDim.x) * blockDim.x)
        posJ[J[i]] = (uint32_t)i;
}
void launch_inverse(const uint32_t* J, uint64_t N, uint32_t* posJ, cudaStream_t s) {
    k_inverse<<<1184, 256, 0, s>>>(J, N, posJ);
    KJ_CUDA(cudaGetLastError());
    g_launches.fetch_add(1, std::memory_order_relaxed);
}
}  // namespace kj

namespace kj {
// ---------------------------------------------------------------- split / classify on device
// split_work (partition.cpp:30-75) without demotion: dense iff double(pop) >= n_thresh,
// pop = population of the query's cell; counts the sparse queries.
__global__ void k_split_flags(const uint32_t* pids, uint64_t nq, const uint32_t* slot,
                              const uint2* G, double n_thresh, uint8_t* dense,
                              unsigned long long* n_sparse) {
    unsigned long long local = 0;
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < nq;
         i += uint64_t(gridDim.x) * blockDim.x) {
        const uint2 g = G[slot[pids[i]]];
        const uint8_t d = double(g.y - g.x) >= n_thresh ? 1 : 0;
        dense[i] = d;
        local += 1 - d;
    }
    for (int o = 16; o > 0; o >>= 1) local += __shfl_xor_sync(0xffffffffu, local, o);
    if ((threadIdx.x & 31) == 0 && local) atomicAdd(n_sparse, local);
}
void launch_split_flags(const uint32_t* pids, uint64_t nq, const uint32_t* slot, const uint2* G,
                        double n_thresh, uint8_t* dense, unsigned long long* n_sparse,
                        cudaStream_t s) {
    if (!nq) return;
    k_split_flags<<<1184, 256, 0, s>>>(pids, nq, slot, G, n_thresh, dense, n_sparse);
    KJ_CUDA(cudaGetLastError());
    g_launches.fetch_add(1, std::memory_order_relaxed);
}

// Provenance and fallback need of the level-0 join rows (orchestrator.cpp:211-234):
// dense rows are solved iff >= K non-self in-eps neighbours (ST_HAS_K & ST_IN_EPS),
// otherwise DenseFailedThenSparse; sparse rows keep the join's list only when it is
// certified globally exact (ST_CERT), else the exact fallback re-solves them.
__global__ void k_classify(const uint32_t* rows, uint64_t n, const uint8_t* st,
                           const uint8_t* dense, uint8_t* prov, uint8_t* need) {
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += uint64_t(gridDim.x) * blockDim.x) {
        const uint32_t r = rows[i];
        const uint8_t s = st[r];
        const bool d = dense ? dense[r] != 0 : true;
        uint8_t pv, nd;
        if (d) {
            const bool ok = (s & ST_HAS_K) && (s & ST_IN_EPS);
            pv = ok ? 0 : 2;
            nd = ok ? 0 : 1;
        } else {
            pv = 1;
            nd = ((s & ST_HAS_K) && (s & ST_CERT)) ? 0 : 1;
        }
        prov[r] = pv;
        need[i] = nd;
    }
}
void launch_classify(const uint32_t* rows, uint64_t n, const uint8_t* st, const uint8_t* dense,
                     uint8_t* prov, uint8_t* need, cudaStream_t s) {
    if (!n) return;
    k_classify<<<1184, 256, 0, s>>>(rows, n, st, dense, prov, need);
    KJ_CUDA(cudaGetLastError());
    g_launches.fetch_add(1, std::memory_order_relaxed);
}

// FP64 rows in a level's position order (same values, contiguous per cell)
__global__ void k_rows_by(const double* X64, const uint32_t* A, uint64_t N, uint32_t n, double* out) {
    const uint64_t total = N * n;
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < total;
         i += uint64_t(gridDim.x) * blockDim.x) {
        const uint64_t r = i / n;
        out[i] = X64[(uint64_t)A[r] * n + (i - r * n)];
    }
}
void launch_rows_by(const double* X64, const uint32_t* A, uint64_t N, uint32_t n, double* out,
                    cudaStream_t s) {
    if (!N) return;
    k_rows_by<<<2368, 256, 0, s>>>(X64, A, N, n, out);
    KJ_CUDA(cudaGetLastError());
    g_launches.fetch_add(1, std::memory_order_relaxed);
}

// rows whose list is not yet globally exact (fine cascade: they go on to level 0)
__global__ void k_item_delta(const uint4* items, const float* r2, uint64_t nitems, double inv_s2,
                             double A, double B, double C, double lim, uint32_t min_q, float* delta,
                             uint8_t* tc_ok) {
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < nitems;
         i += uint64_t(gridDim.x) * blockDim.x) {
        const double R2 = (double)r2[i] * inv_s2 * (1.0 + 1e-12);
        const double d = (A * R2 + B * sqrt(R2) * (1.0 + 1e-15) + C) * (1.0 + 1e-6);
        const float df = __double2float_ru(d);
        delta[i] = df;
        const uint4 it = items[i];
        tc_ok[i] = (2.0 * (double)df <= lim && it.y - it.x >= min_q) ? 1 : 0;
    }
}
void launch_item_delta(const uint4* items, const float* r2, uint64_t nitems, double inv_s2,
                       double A, double B, double C, double lim, uint32_t min_q, float* delta,
                       uint8_t* tc_ok, cudaStream_t s) {
    if (!nitems) return;
    k_item_delta<<<(unsigned)std::min<uint64_t>((nitems + 255) / 256, 148 * 16), 256, 0, s>>>(
        items, r2, nitems, inv_s2, A, B, C, lim, min_q, delta, tc_ok);
    KJ_CUDA(cudaGetLastError());
    g_launches.fetch_add(1, std::memory_order_relaxed);
}
// per work item: the largest per-row K-th bound (cut_by_row, by output row) over its launch
// rows (virtual split-part rows map to their real row through vsrc)
__global__ void k_item_max_cut(const uint4* items, uint64_t nitems, const uint32_t* qrow, uint64_t nq,
                               const uint32_t* vsrc, const float* cut_by_row, float* out) {
    const uint64_t item = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (item >= nitems) return;
    const uint4 it = items[item];
    float m = 0.f;
    for (uint32_t r = it.x + lane; r < it.y; r += 32) {
        const uint32_t rr = r < nq ? r : vsrc[r - nq];
        m = fmaxf(m, cut_by_row[qrow[rr]]);
    }
    for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    // widened like the scalar radius (an FP64 sum can sit below the true squared distance)
    if (lane == 0) out[item] = it.y > it.x ? __fmul_ru(m, 1.0f + 0x1p-20f) : 0.f;
}
void launch_item_max_cut(const uint4* items, uint64_t nitems, const uint32_t* qrow, uint64_t nq,
                         const uint32_t* vsrc, const float* cut_by_row, float* out, cudaStream_t s) {
    if (!nitems) return;
    k_item_max_cut<<<(unsigned)((nitems * 32 + 255) / 256), 256, 0, s>>>(items, nitems, qrow, nq, vsrc,
                                                                         cut_by_row, out);
    KJ_CUDA(cudaGetLastError());
    g_launches.fetch_add(1, std::memory_order_relaxed);
}
__global__ void k_range_len(const uint2* r, uint64_t n, uint32_t* out) {
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += uint64_t(gridDim.x) * blockDim.x)
        out[i] = r[i].y - r[i].x;
}
void launch_range_len(const uint2* r, uint64_t n, uint32_t* out, cudaStream_t s) {
    if (!n) return;
    k_range_len<<<(unsigned)std::min<uint64_t>((n + 255) / 256, 148 * 16), 256, 0, s>>>(r, n, out);
    KJ_CUDA(cudaGetLastError());
    g_launches.fetch_add(1, std::memory_order_relaxed);
}
__global__ void k_miss_flags(const uint32_t* rows, uint64_t n, const uint8_t* st, uint8_t* flags) {
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += uint64_t(gridDim.x) * blockDim.x)
        flags[i] = (st[rows[i]] & ST_MISS) ? 1 : 0;
}
void launch_miss_flags(const uint32_t* rows, uint64_t n, const uint8_t* st, uint8_t* flags,
                       cudaStream_t s) {
    if (!n) return;
    k_miss_flags<<<(unsigned)std::min<uint64_t>((n + 255) / 256, 148 * 16), 256, 0, s>>>(rows, n, st, flags);
    KJ_CUDA(cudaGetLastError());
    g_launches.fetch_add(1, std::memory_order_relaxed);
}
__global__ void k_uncert_flags(const uint32_t* rows, uint64_t n, const uint8_t* st, uint8_t* flags) {
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += uint64_t(gridDim.x) * blockDim.x) {
        const uint8_t v = st[rows[i]];
        flags[i] = ((v & ST_HAS_K) && (v & ST_CERT)) ? 0 : 1;
    }
}
void launch_uncert_flags(const uint32_t* rows, uint64_t n, const uint8_t* st, uint8_t* flags,
                         cudaStream_t s) {
    if (!n) return;
    k_uncert_flags<<<1184, 256, 0, s>>>(rows, n, st, flags);
    KJ_CUDA(cudaGetLastError());
    g_launches.fetch_add(1, std::memory_order_relaxed);
}

// candidates_examined over the dense queries of a pass: sum over items of
// (candidate-set size) x (dense rows in the item).
__global__ void k_dense_cand(const uint4* items, const unsigned long long* work, uint64_t nitems,
                             const uint32_t* qrow, const uint8_t* dense,
                             unsigned long long* out) {
    unsigned long long local = 0;
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < nitems;
         i += uint64_t(gridDim.x) * blockDim.x) {
        const uint4 it = items[i];
        const uint32_t q = it.y - it.x;
        if (!q) continue;
        const unsigned long long cs = work[i] / q;
        uint32_t nd = 0;
        for (uint32_t r = it.x; r < it.y; ++r) nd += dense[qrow[r]] ? 1u : 0u;
        local += cs * nd;
    }
    for (int o = 16; o > 0; o >>= 1) local += __shfl_xor_sync(0xffffffffu, local, o);
    if ((threadIdx.x & 31) == 0 && local) atomicAdd(out, local);
}
void launch_dense_cand(const uint4* items, const unsigned long long* work, uint64_t nitems,
                       const uint32_t* qrow, const uint8_t* dense, unsigned long long* out,
                       cudaStream_t s) {
    if (!nitems) return;
    k_dense_cand<<<592, 256, 0, s>>>(items, work, nitems, qrow, dense, out);
    KJ_CUDA(cudaGetLastError());
    g_launches.fetch_add(1, std::memory_order_relaxed);
}

// Output rows of one shard, compacted: out[i*K..] = src[rows[i]*K..] (ids + dist).
__global__ void k_gather_rows(const uint32_t* rows, uint64_t n, uint32_t K, const uint32_t* ids,
                              const double* dist, uint32_t* oids, double* odist) {
    const uint64_t total = n * K;
    for (uint64_t e = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < total;
         e += uint64_t(gridDim.x) * blockDim.x) {
        const uint64_t i = e / K, j = e - i * K;
        const uint64_t src = (uint64_t)rows[i] * K + j;
        oids[e] = ids[src];
        odist[e] = dist[src];
    }
}
void launch_gather_rows(const uint32_t* rows, uint64_t n, uint32_t K, const uint32_t* ids,
                        const double* dist, uint32_t* oids, double* odist, cudaStream_t s) {
    if (!n || !K) return;
    k_gather_rows<<<2368, 256, 0, s>>>(rows, n, K, ids, dist, oids, odist);
    KJ_CUDA(cudaGetLastError());
    g_launches.fetch_add(1, std::memory_order_relaxed);
}
// One warp per output row, rows taken in the given (ascending) order: the row's K ids and
// K distances from device memory to the same row of mapped host memory, one coalesced
// store per 128 bytes. Ascending rows keep the host stores sweeping the address space in
// order (~49 GB/s over PCIe; random rows ~15 GB/s, tools/micro/pcie_write.cu).
__global__ void k_rows_to_host(const uint32_t* rows, uint64_t n, uint32_t K, const uint32_t* ids,
                               const double* dist, uint32_t* hids, double* hdist) {
    const int lane = threadIdx.x & 31;
    const uint64_t nw = (uint64_t(gridDim.x) * blockDim.x) >> 5;
    for (uint64_t w = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; w < n; w += nw) {
        const uint64_t base = (uint64_t)rows[w] * K;
        for (uint32_t i = lane; i < K; i += 32) hids[base + i] = ids[base + i];
        for (uint32_t i = lane; i < K; i += 32) hdist[base + i] = dist[base + i];
    }
}
void launch_rows_to_host(const uint32_t* rows, uint64_t n, uint32_t K, const uint32_t* ids,
                         const double* dist, uint32_t* hids, double* hdist, uint32_t max_blocks,
                         cudaStream_t s) {
    if (!n || !K) return;
    uint64_t blocks = (n * 32 + 255) / 256;
    if (max_blocks) blocks = std::min<uint64_t>(blocks, max_blocks);
    k_rows_to_host<<<(unsigned)blocks, 256, 0, s>>>(rows, n, K, ids, dist, hids, hdist);
    KJ_CUDA(cudaGetLastError());
    g_launches.fetch_add(1, std::memory_order_relaxed);
}
// rows[i] of (ids, dist) to the same rows of (oids, odist) (e.g. mapped host memory)
__global__ void k_scatter_rows(const uint32_t* rows, uint64_t n, uint32_t K, const uint32_t* ids,
                               const double* dist, uint32_t* oids, double* odist) {
    const uint64_t total = n * K;
    for (uint64_t e = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < total;
         e += uint64_t(gridDim.x) * blockDim.x) {
        const uint64_t i = e / K, j = e - i * K;
        const uint64_t at = (uint64_t)rows[i] * K + j;
        oids[at] = ids[at];
        odist[at] = dist[at];
    }
}
void launch_scatter_rows(const uint32_t* rows, uint64_t n, uint32_t K, const uint32_t* ids,
                         const double* dist, uint32_t* oids, double* odist, cudaStream_t s) {
    if (!n || !K) return;
    k_scatter_rows<<<1184, 256, 0, s>>>(rows, n, K, ids, dist, oids, odist);
    KJ_CUDA(cudaGetLastError());
    g_launches.fetch_add(1, std::memory_order_relaxed);
}
}  // namespace kj

namespace kj {
// Rows whose screened list overflowed (cnt == OVF), appended in any order (each is
// re-solved independently by k_slow_exact, so the order never reaches the output).
__global__ void k_find_ovf(const uint32_t* cnt, uint64_t n, uint32_t* rows,
                           unsigned long long* count) {
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += uint64_t(gridDim.x) * blockDim.x) {
        if (cnt[i] == OVF) rows[atomicAdd(count, 1ull)] = (uint32_t)i;
    }
}
void launch_find_ovf(const uint32_t* cnt, uint64_t n, uint32_t* rows, unsigned long long* count,
                     cudaStream_t s) {
    if (!n) return;
    k_find_ovf<<<1184, 256, 0, s>>>(cnt, n, rows, count);
    KJ_CUDA(cudaGetLastError());
    g_launches.fetch_add(1, std::memory_order_relaxed);
}
}  // namespace kj

namespace kj {
// Rows whose work item was split into candidate-range parts (pass build): each part
// was finalized exactly into its own sorted (sq, id) top-K; this merges the parts'
// lists per query (warp argmin over the part heads, K steps) into the real row.
// splits[i] = (first real row, queries, parts, first virtual row - nq).
__global__ void k_merge_parts(const uint4* splits, uint64_t nsplits, uint32_t K,
                              const uint32_t* t_ids, const double* t_sq, const uint32_t* t_count,
                              const uint32_t* qrow, double eps2, double cover2,
                              uint32_t* out_ids, double* out_dist, double* out_kth,
                              uint8_t* out_status) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
    for (uint64_t si = blockIdx.x; si < nsplits; si += gridDim.x) {
        const uint4 sp = splits[si];
        for (uint32_t qi = w; qi < sp.y; qi += nw) {
            // lane p < parts follows part p's list
            const bool act = (uint32_t)lane < sp.z;
            const uint64_t v = act ? (uint64_t)sp.w + (uint64_t)lane * sp.y + qi : 0;
            const uint32_t cnt = act ? t_count[v] : 0u;
            uint32_t head = 0;
            uint32_t total = cnt;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) total += __shfl_xor_sync(0xffffffffu, total, o);
            const uint32_t orow = qrow[sp.x + qi];
            const uint32_t outn = min(total, K);
            double kth = CUDART_INF;
            for (uint32_t r = 0; r < outn; ++r) {
                const double s0 = head < cnt ? t_sq[v * K + head] : CUDART_INF;
                const uint32_t i0 = head < cnt ? t_ids[v * K + head] : 0xFFFFFFFFu;
                double bs = s0;
                uint32_t bt = i0;
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) {
                    const double s2 = __shfl_xor_sync(0xffffffffu, bs, o);
                    const uint32_t t2 = __shfl_xor_sync(0xffffffffu, bt, o);
                    if (pair_less(s2, t2, bs, bt)) {
                        bs = s2;
                        bt = t2;
                    }
                }
                // parts hold disjoint candidates, so exactly one head carries (bs, bt)
                if (head < cnt && i0 == bt && s0 == bs) ++head;
                if (lane == 0) {
                    out_ids[(uint64_t)orow * K + r] = bt;
                    out_dist[(uint64_t)orow * K + r] = sqrt(bs);
                }
                kth = bs;
            }
            if (lane == 0) {
                uint8_t st = 0;
                if (total >= K) {
                    st |= ST_HAS_K;
                    if (kth <= eps2) st |= ST_IN_EPS;
                    if (kth < cover2) st |= ST_CERT;
                }
                out_status[orow] = st;
                out_kth[orow] = total >= K ? kth : CUDART_INF;
            }
        }
    }
}
void launch_merge_parts(const uint4* splits, uint64_t nsplits, uint32_t K, const uint32_t* t_ids,
                        const double* t_sq, const uint32_t* t_count, const uint32_t* qrow,
                        double eps2, double cover2, uint32_t* out_ids, double* out_dist,
                        double* out_kth, uint8_t* out_status, cudaStream_t s) {
    if (!nsplits) return;
    k_merge_parts<<<(unsigned)std::min<uint64_t>(nsplits, 4096), 256, 0, s>>>(
        splits, nsplits, K, t_ids, t_sq, t_count, qrow, eps2, cover2, out_ids, out_dist, out_kth,
        out_status);
    KJ_CUDA(cudaGetLastError());
    g_launches.fetch_add(1, std::memory_order_relaxed);
}
}  // namespace kj

namespace kj {
__global__ void k_fill_u32(uint32_t* p, uint64_t n, uint32_t v) {
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += uint64_t(gridDim.x) * blockDim.x)
        p[i] = v;
}
void launch_fill_u32(uint32_t* p, uint64_t n, uint32_t v, cudaStream_t s) {
    if (!n) return;
    k_fill_u32<<<1184, 256, 0, s>>>(p, n, v);
    KJ_CUDA(cudaGetLastError());
    g_launches.fetch_add(1, std::memory_order_relaxed);
}
}  // namespace kj

namespace kj {
__global__ void k_scatter_f32(const uint32_t* idx, const float* vals, uint64_t n, float* out) {
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += uint64_t(gridDim.x) * blockDim.x)
        out[idx[i]] = vals[i];
}
void launch_scatter_f32(const uint32_t* idx, const float* vals, uint64_t n, float* out,
                        cudaStream_t s) {
    if (!n) return;
    k_scatter_f32<<<592, 256, 0, s>>>(idx, vals, n, out);
    KJ_CUDA(cudaGetLastError());
    g_launches.fetch_add(1, std::memory_order_relaxed);
}
}  // namespace kj

namespace kj {
// ---------------------------------------------------------------- candidate box filter
// Boxes are FP32, rounded outward from the FP64 coordinates (lo down, hi up), stored
// dimension-major so a warp testing 32 consecutive blocks reads coalesced rows.
__device__ __forceinline__ void box_of(const double* X64, const uint32_t* ids_pos, const uint32_t* J,
                                       uint64_t p0, uint64_t p1, uint32_t n, uint32_t d, int lane,
                                       float& lo, float& hi) {
    double l = CUDART_INF, h = -CUDART_INF;
    for (uint64_t p = p0 + lane; p < p1; p += 32) {
        const uint32_t pos = ids_pos ? ids_pos[p] : (uint32_t)p;
        const double v = X64[(uint64_t)J[pos] * n + d];
        l = fmin(l, v);
        h = fmax(h, v);
    }
    for (int o = 16; o > 0; o >>= 1) {
        l = fmin(l, __shfl_xor_sync(0xffffffffu, l, o));
        h = fmax(h, __shfl_xor_sync(0xffffffffu, h, o));
    }
    lo = __double2float_rd(l);
    hi = __double2float_ru(h);
}

// Per FB-position block of a level's join order (J): box[d * nblk + b] (lo), then
// box[(n + d) * nblk + b] (hi). One warp per block.
__global__ void k_block_boxes(const double* X64, const uint32_t* J, uint64_t N, uint32_t n,
                              float* box) {
    const uint64_t nblk = (N + FB - 1) / FB;
    const uint64_t w = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (w >= nblk) return;
    for (uint32_t d = 0; d < n; ++d) {
        float lo, hi;
        box_of(X64, nullptr, J, w * FB, min(N, (w + 1) * FB), n, d, lane, lo, hi);
        if (lane == 0) {
            box[(uint64_t)d * nblk + w] = lo;
            box[(uint64_t)(n + d) * nblk + w] = hi;
        }
    }
}
void launch_block_boxes(const double* X64, const uint32_t* J, uint64_t N, uint32_t n, float* box,
                        cudaStream_t s) {
    const uint64_t nblk = (N + FB - 1) / FB;
    if (!nblk) return;
    k_block_boxes<<<(unsigned)((nblk * 32 + 255) / 256), 256, 0, s>>>(X64, J, N, n, box);
    KJ_CUDA(cudaGetLastError());
    g_launches.fetch_add(1, std::memory_order_relaxed);
}

// Per work item, the box of its queries (qpos rows [x, y)): qbox[item * 2n + d] lo, [+ n] hi.
__global__ void k_item_boxes(const uint4* items, uint64_t nitems, const uint32_t* qpos,
                             const uint32_t* J, const double* X64, uint32_t n, float* qbox) {
    const uint64_t item = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (item >= nitems) return;
    const uint4 it = items[item];
    for (uint32_t d = 0; d < n; ++d) {
        float lo, hi;
        box_of(X64, qpos, J, it.x, it.y, n, d, lane, lo, hi);
        if (lane == 0) {
            qbox[item * 2 * n + d] = lo;
            qbox[item * 2 * n + n + d] = hi;
        }
    }
}

// One warp per work item: every FB-block of its candidate ranges is tested against
// the item's query box (lanes = 32 consecutive blocks); blocks whose squared box gap
// (rounded down, early exit) exceeds r2 are dropped, the survivors re-emitted as
// merged ranges. COUNT: out_cnt[item] = ranges kept. FILL: ranges written at
// out_off[item], (abeg, aend) of the item rewritten, kept pairs summed into screened.
// ORDER: one range per kept block plus a sweep-order key (squared distance between the
// item box centre and the block box centre), for a per-item sort nearest-first.
// FILL with item_r2: also the squared radius (rounded up) of the item's data about the
// global centre, max over its query box and its kept blocks' boxes, from g rounded
// outward (g_lo, g_hi): the per-item tensor-core screen bound.
__device__ __forceinline__ float box_radius2(const float* lo, const float* hi, size_t stride,
                                             const float* g_lo, const float* g_hi, uint32_t n,
                                             uint32_t d0 = 0) {
    float acc = 0.f;
    for (uint32_t d = d0; d < n; ++d) {
        const float r = fmaxf(fmaxf(__fsub_ru(g_hi[d], lo[d * stride]), __fsub_ru(hi[d * stride], g_lo[d])), 0.f);
        acc = __fadd_ru(acc, __fmul_ru(r, r));
    }
    return acc;
}
template <bool FILL, bool ORDER>
__global__ void k_filter_ranges(uint4* items, uint64_t nitems, const float* qbox, uint32_t n,
                                const uint2* adj, const float* box, uint64_t nblk, float r2,
                                uint32_t* out_cnt, const uint32_t* out_off, uint2* out_adj,
                                unsigned long long* screened, float* out_key, const float* gbox,
                                float* item_r2, uint32_t r_m, float r_2w, const float* dbox,
                                const float* item_rad2) {
    const int lane = threadIdx.x & 31;
    const uint64_t item = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    if (item >= nitems) return;
    const uint4 it = items[item];
    const float* ql = qbox + item * 2 * n;
    const float* qh = ql + n;
    if (item_rad2) r2 = fminf(r2, item_rad2[item]);  // the item's rows' K-th bound
    uint32_t kept = 0;
    unsigned long long span = 0;
    float rmax = 0.f;  // item_r2: max over kept blocks
    const bool want_r = FILL && item_r2 != nullptr;
    const uint32_t base = FILL ? out_off[item] : 0;
    for (uint32_t ri = it.z; ri < it.w; ++ri) {
        const uint2 rg = adj[ri];
        if (rg.x >= rg.y) continue;
        const uint32_t b0 = rg.x / FB, b1 = (rg.y - 1) / FB;
        // 32-block chunks independently: a kept run crossing a chunk boundary becomes two
        // ranges (block-aligned, so no extra partial tiles in the join)
        for (uint32_t c0 = b0; c0 <= b1; c0 += 32) {
            const uint32_t blk = c0 + lane;
            bool keep = false;
            float ck = 0.f;
            if (blk <= b1) {
                float acc = 0.f;
                for (uint32_t d = 0; d < n && acc <= r2; ++d) {
                    const float lo = __ldg(box + (uint64_t)d * nblk + blk);
                    const float hi = __ldg(box + (uint64_t)(n + d) * nblk + blk);
                    const float g = fmaxf(0.f, fmaxf(__fsub_rd(lo, qh[d]), __fsub_rd(ql[d], hi)));
                    acc = __fadd_rd(acc, __fmul_rd(g, g));
                    if (ORDER && FILL) {  // sweep key from the same loads (complete for kept blocks)
                        const float dc = 0.5f * ((lo + hi) - (ql[d] + qh[d]));
                        ck = fmaf(dc, dc, ck);
                    }
                }
                keep = acc <= r2;
                if (want_r && keep && r_m < n)
                    rmax = fmaxf(rmax, box_radius2(box + blk, box + (uint64_t)n * nblk + blk, nblk,
                                                   gbox, gbox + n, n, r_m));
            }
            const unsigned m = __ballot_sync(0xffffffffu, keep);
            if (ORDER) {
                if (FILL && keep) {
                    const uint32_t rank = kept + __popc(m & ((1u << lane) - 1u));
                    const uint2 o = make_uint2(max(rg.x, blk * FB), min(rg.y, (blk + 1) * FB));
                    out_adj[base + rank] = o;
                    out_key[base + rank] = ck;
                    span += o.y - o.x;
                }
                kept += __popc(m);
                continue;
            }
            const unsigned starts = m & ~(m << 1);  // first block of each kept run
            if (FILL && ((starts >> lane) & 1u)) {
                const unsigned above = lane == 31 ? 0u : ~m & ~((2u << lane) - 1u);
                const uint32_t e = above ? c0 + (uint32_t)(__ffs(above) - 2) : min(c0 + 31, b1);
                const uint32_t rank = kept + __popc(starts & ((1u << lane) - 1u));
                const uint2 o = make_uint2(max(rg.x, blk * FB), min(rg.y, (e + 1) * FB));
                out_adj[base + rank] = o;
                span += o.y - o.x;
            }
            kept += __popc(starts);
        }
    }
    if (FILL && screened) {
        for (int o = 16; o > 0; o >>= 1) span += __shfl_xor_sync(0xffffffffu, span, o);
        if (lane == 0 && span) atomicAdd(screened, span * (unsigned long long)(it.y - it.x));
    }
    if (want_r) {
        // grid dims d < r_m: every candidate lies in the cells next to a query's cell. In
        // the dims where all the item's queries share one cell coordinate (all but the last:
        // an item is one cell or a run of cells along the last dim) that is within
        // [qh - 2w, ql + 2w]; along the last dim within [ql - 2w, qh + 2w]. The other dims:
        // the kept blocks' boxes (and the query box). All clipped to the data range (dbox).
        for (int o = 16; o > 0; o >>= 1) rmax = fmaxf(rmax, __shfl_xor_sync(0xffffffffu, rmax, o));
        if (lane == 0) {
            float low = 0.f;
            for (uint32_t d = 0; d < r_m; ++d) {
                const bool run_dim = d + 1 == r_m;
                const float lo = fmaxf(__fsub_rd(run_dim ? ql[d] : qh[d], r_2w), dbox[d]);
                const float hi = fminf(__fadd_ru(run_dim ? qh[d] : ql[d], r_2w), dbox[r_m + d]);
                const float r = fmaxf(fmaxf(__fsub_ru(gbox[n + d], lo), __fsub_ru(hi, gbox[d])), 0.f);
                low = __fadd_ru(low, __fmul_ru(r, r));
            }
            const float high = r_m < n ? fmaxf(rmax, box_radius2(ql, qh, 1, gbox, gbox + n, n, r_m)) : 0.f;
            item_r2[item] = __fadd_ru(low, high);
        }
    }
    if (lane == 0) {
        if (FILL) items[item] = make_uint4(it.x, it.y, base, base + kept);
        else out_cnt[item] = kept;
        if (!FILL && screened) atomicAdd(screened, (unsigned long long)kept);  // 64-bit total
    }
}
void launch_item_boxes(const uint4* items, uint64_t nitems, const uint32_t* qpos, const uint32_t* J,
                       const double* X64, uint32_t n, float* qbox, cudaStream_t s) {
    if (!nitems) return;
    k_item_boxes<<<(unsigned)((nitems * 32 + 255) / 256), 256, 0, s>>>(items, nitems, qpos, J, X64, n,
                                                                       qbox);
    KJ_CUDA(cudaGetLastError());
    g_launches.fetch_add(1, std::memory_order_relaxed);
}
void launch_filter_ranges(uint4* items, uint64_t nitems, const float* qbox, uint32_t n,
                          const uint2* adj, const float* box, uint64_t nblk, float r2,
                          uint32_t* out_cnt, const uint32_t* out_off, uint2* out_adj,
                          unsigned long long* screened, bool fill, cudaStream_t s,
                          float* out_key, unsigned long long* count_total, const float* gbox,
                          float* item_r2, uint32_t r_m, float r_2w, const float* dbox,
                          const float* item_rad2) {
    if (!nitems) return;
    const unsigned grid = (unsigned)((nitems * 32 + 255) / 256);
    if (!fill) screened = count_total;  // the count pass sums kept ranges there (if given)
#define KJ_FR(F, O)                                                                       \
    k_filter_ranges<F, O><<<grid, 256, 0, s>>>(items, nitems, qbox, n, adj, box, nblk, r2, \
                                               out_cnt, out_off, out_adj, screened, out_key, gbox, \
                                               item_r2, r_m, r_2w, dbox, item_rad2)
    if (out_key) {
        if (fill) KJ_FR(true, true);
        else KJ_FR(false, true);
    } else {
        if (fill) KJ_FR(true, false);
        else KJ_FR(false, false);
    }
#undef KJ_FR
    KJ_CUDA(cudaGetLastError());
    g_launches.fetch_add(1, std::memory_order_relaxed);
}
}  // namespace kj
