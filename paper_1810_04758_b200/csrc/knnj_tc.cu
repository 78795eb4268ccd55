// tcgen05 (5th-gen tensor core) screen for the fused range-join + top-K.
//
// Same contract as k_join (knnj_kernels.cu): per query, the list of every
// candidate that can belong to the exact (sq,id) top-K of its 3^m
// neighbourhood; k_finalize re-decides it in FP64 scalar order.
//
// Distance screen as a GEMM on the tensor cores. Coordinates are centred at
// the global mean g and scaled by a power of two S (|x~| <= 1), then split
// x~ = hi + lo with hi, lo FP16. Per candidate (B operand, precomputed once per
// grid level, K-major, streamed by TMA):    [hi, lo, hi, nb_hi, nb_lo, 0...]
// per query (A operand, built in smem):     [-2hi, -2hi, -2lo, 1, 1, 0...]
// so one UMMA chain accumulates (FP32, in TMEM)
//     D = |b|^2 - 2 (a_hi.b_hi + a_hi.b_lo + a_lo.b_hi)  ~  |b|^2 - 2 a.b
// and key = D + |a|^2 ~ |a-b|^2 / S^2 with a rigorously bounded error
// (DESIGN.md §3). 128 queries (TMEM lanes) x 128 candidates (columns) per
// tile; two TMEM accumulators and two smem stages so the next tile's TMA +
// MMA overlap the current tile's epilogue (TMEM -> registers -> screen).
#include <cuda.h>
#include <cuda_fp16.h>
#include <cudaTypedefs.h>
#include <math_constants.h>

#include "knnj_internal.cuh"

namespace kj {

namespace {

constexpr int TC_M = 128;     // queries per block (= TMEM lanes = threads)
constexpr int TC_N = 128;     // candidates per tile (= accumulator columns)
constexpr int KBLK = 64;      // fp16 elements per 128-byte swizzle row
constexpr int KB_BYTES = TC_M * 128;  // one k-block of a 128-row operand: 16 KB

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
#ifdef KNNJ_MBAR_SUSPEND
    asm volatile(
        "{\n\t.reg .pred P;\n\t"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1, %2;\n\t"
        "@!P bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
        "r"(parity), "r"(KNNJ_MBAR_SUSPEND)
        : "memory");
#else
    asm volatile(
        "{\n\t.reg .pred P;\n\t"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n\t"
        "@!P bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
#endif
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar,
                                            int c0, int c1) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(dst)),
        "l"(map), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
        : "memory");
}
__device__ __forceinline__ void fence_before() {
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void fence_after() {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}

// UMMA shared-memory descriptor, K-major, 128B swizzle (8-row atoms of 128 B,
// SBO = 1024 B between atoms), sm_100 descriptor version 1.
__device__ __forceinline__ uint64_t umma_desc_sw128(uint32_t saddr) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFF);   // start address
    d |= (uint64_t)1 << 16;                   // LBO (unused for swizzled K-major)
    d |= (uint64_t)(1024 >> 4) << 32;         // SBO
    d |= (uint64_t)1 << 46;                   // version
    d |= (uint64_t)2 << 61;                   // SWIZZLE_128B
    return d;
}

// kind::f16: A=F16, B=F16, D=F32, both K-major, M=128, N=128
template <int TN>
constexpr uint32_t idesc_f16() {
    return (1u << 4) | (0u << 7) | (0u << 10) | ((uint32_t)(TN >> 3) << 17) |
           ((uint32_t)(TC_M >> 4) << 24);
}

template <int TN>
__device__ __forceinline__ void umma_f16(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(da), "l"(db), "r"(idesc_f16<TN>()), "r"(acc));
}
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                     smem_u32(bar))
                 : "memory");
}

// two 32-column loads in flight, one wait (both in one asm: no use before the wait)
__device__ __forceinline__ void tmem_ld64(uint32_t taddr, float (&v0)[32], float (&v1)[32]) {
    uint32_t r[64];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%64];\n\t"
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%32,%33,%34,%35,%36,%37,%38,%39,%40,%41,%42,%43,%44,%45,%46,%47,%48,%49,%50,%51,%52,%53,%54,%55,%56,%57,%58,%59,%60,%61,%62,%63}, [%65];\n\t"
        "tcgen05.wait::ld.sync.aligned;"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31]), "=r"(r[32]), "=r"(r[33]), "=r"(r[34]), "=r"(r[35]), "=r"(r[36]), "=r"(r[37]), "=r"(r[38]), "=r"(r[39]), "=r"(r[40]), "=r"(r[41]), "=r"(r[42]), "=r"(r[43]), "=r"(r[44]), "=r"(r[45]), "=r"(r[46]), "=r"(r[47]), "=r"(r[48]), "=r"(r[49]), "=r"(r[50]), "=r"(r[51]), "=r"(r[52]), "=r"(r[53]), "=r"(r[54]), "=r"(r[55]), "=r"(r[56]), "=r"(r[57]), "=r"(r[58]), "=r"(r[59]), "=r"(r[60]), "=r"(r[61]), "=r"(r[62]), "=r"(r[63])
        : "r"(taddr), "r"(taddr + 32u)
        : "memory");
#pragma unroll
    for (int i = 0; i < 32; ++i) {
        v0[i] = __uint_as_float(r[i]);
        v1[i] = __uint_as_float(r[32 + i]);
    }
}
__device__ __forceinline__ float tmem_ld1(uint32_t taddr) {
    uint32_t r;
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(r) : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    return __uint_as_float(r);
}

// dev instrumentation (-DKNNJ_TC_CLOCKS, KNNJ_JOIN_STATS): cycles per role phase into stats[8..]
#ifdef KNNJ_TC_CLOCKS
#define TCK(v) const long long v = clock64()
#define TCADD(i, a, b) (ck[i] += (unsigned long long)((b) - (a)))
#else
#define TCK(v)
#define TCADD(i, a, b)
#endif

// v[j] for a warp-uniform runtime j, from registers: a 5-level select tree (31 SELs)
// instead of a local-memory array or a TMEM re-read plus its wait
__device__ __forceinline__ float pick32(const float (&v)[32], int j) {
    float a[16], b[8], c[4], d[2];
#pragma unroll
    for (int i = 0; i < 16; ++i) a[i] = (j & 16) ? v[i + 16] : v[i];
#pragma unroll
    for (int i = 0; i < 8; ++i) b[i] = (j & 8) ? a[i + 8] : a[i];
#pragma unroll
    for (int i = 0; i < 4; ++i) c[i] = (j & 4) ? b[i + 4] : b[i];
#pragma unroll
    for (int i = 0; i < 2; ++i) d[i] = (j & 2) ? c[i + 2] : c[i];
    return (j & 1) ? d[1] : d[0];
}

// 3-input FP32 min (FMNMX3 on sm_100; a NaN input is ignored like fminf)
__device__ __forceinline__ float fmin3(float a, float b, float c) {
    float d;
    asm("min.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
    return d;
}
// minimum of a 64-column slab (NaN columns ignored): a 3-ary tree, 32 FMNMX3/FMNMX
__device__ __forceinline__ float slab_min64(const float (&v0)[32], const float (&v1)[32]) {
    float t[22];
#pragma unroll
    for (int i = 0; i < 21; ++i) {
        const int a = 3 * i, b = 3 * i + 1, c = 3 * i + 2;
        t[i] = fmin3(a < 32 ? v0[a] : v1[a - 32], b < 32 ? v0[b] : v1[b - 32], c < 32 ? v0[c] : v1[c - 32]);
    }
    t[21] = v1[31];
    float u[8];
#pragma unroll
    for (int i = 0; i < 7; ++i) u[i] = fmin3(t[3 * i], t[3 * i + 1], t[3 * i + 2]);
    u[7] = t[21];
    return fmin3(fmin3(u[0], u[1], u[2]), fmin3(u[3], u[4], u[5]), fminf(u[6], u[7]));
}

// K-th smallest (1-based k) of the 32*R values a[r] (element index r*32 + lane)
// held across a warp: bitonic sort network, ascending.
template <int R>
__device__ __forceinline__ float warp_kth(float (&a)[R], uint32_t k) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int kk = 2; kk <= 32 * R; kk <<= 1) {
#pragma unroll
        for (int j = kk >> 1; j > 0; j >>= 1) {
            if (j >= 32) {
                // partner in register r ^ (j/32) of the same lane
                const int rj = j >> 5;
#pragma unroll
                for (int r = 0; r < R; ++r) {
                    if (r & rj) continue;
                    const int e = r * 32 + lane;
                    const bool up = (e & kk) == 0;
                    const float lo = fminf(a[r], a[r | rj]), hi = fmaxf(a[r], a[r | rj]);
                    a[r] = up ? lo : hi;
                    a[r | rj] = up ? hi : lo;
                }
            } else {
                const bool lower = (lane & j) == 0;
#pragma unroll
                for (int r = 0; r < R; ++r) {
                    const float pv = __shfl_xor_sync(0xffffffffu, a[r], j);
                    const int e = r * 32 + lane;
                    const bool up = (e & kk) == 0;
                    a[r] = (lower == up) ? fminf(a[r], pv) : fmaxf(a[r], pv);
                }
            }
        }
    }
    const uint32_t i = k - 1;
    float v = 0.f;
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const float t = __shfl_sync(0xffffffffu, a[r], i & 31);
        if ((i >> 5) == (uint32_t)r) v = t;
    }
    return v;
}

}  // namespace

// B-operand rows for one grid level, sorted order: [lo | hi | hi | nb_hi nb_lo | 0]
// (K = 3n+2, ~22-bit products). The small hi x lo products come first in K and the
// large hi x hi products and |b|^2 last, which keeps the accumulated partial sums small
// for most of the UMMA chain (the accumulation term of tc_delta).
__global__ void k_prep_tc(const double* X64, const uint32_t* A, uint64_t N, uint32_t n,
                          const double* g, double inv_S, uint32_t row_halfs, __half* Bh,
                          uint32_t write_halfs) {
    // one thread per row; the row is emitted as 16-byte chunks of 8 halfs, so a warp
    // writes whole 128-byte rows instead of scattered 2-byte stores
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < N;
         i += uint64_t(gridDim.x) * blockDim.x) {
        const double* x = X64 + (uint64_t)A[i] * n;
        double nb = 0.0;
        for (uint32_t d = 0; d < n; ++d) {
            const double v = (x[d] - g[d]) * inv_S;
            nb += v * v;
        }
        const __half nh = __double2half(nb);
        const __half nl = __double2half(nb - (double)__half2float(nh));
        const uint32_t o = 3 * n;
        uint4* row = reinterpret_cast<uint4*>(Bh + i * row_halfs);
        // (write_halfs < row_halfs: the rest of the row is known zero from an earlier build)
        for (uint32_t c0 = 0; c0 < write_halfs; c0 += 8) {
            uint32_t w[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                uint32_t pair = 0;
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const uint32_t k = c0 + 2 * e + h;
                    __half hv = __float2half(0.f);
                    if (k < o) {
                        const uint32_t d = k % n, part = k / n;  // lo | hi | hi
                        const double v = (x[d] - g[d]) * inv_S;
                        const __half hi = __double2half(v);
                        hv = part == 0 ? __double2half(v - (double)__half2float(hi)) : hi;
                    } else if (k == o) {
                        hv = nh;
                    } else if (k == o + 1) {
                        hv = nl;
                    }
                    pair |= (uint32_t)__half_as_ushort(hv) << (16 * h);
                }
                w[e] = pair;
            }
            row[c0 / 8] = make_uint4(w[0], w[1], w[2], w[3]);
        }
    }
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// Exact bin of one histogram pair (epsilon.cpp:86-95), off the hot path.
__device__ __noinline__ uint32_t exact_bin(const double* X64, uint32_t n, uint32_t q, uint32_t t,
                                           double em, double limit_sq, double inv_width,
                                           uint32_t nb) {
    const double* a = X64 + (uint64_t)q * n;
    const double* b = X64 + (uint64_t)t * n;
    double sum = 0.0;
    for (uint32_t i = 0; i < n; ++i) {
        const double d = __dsub_rn(a[i], b[i]);
        sum = __dadd_rn(sum, __dmul_rn(d, d));
    }
    if (sum > limit_sq) return nb;
    const double dist = sqrt(sum);
    if (dist >= em) return nb;
    uint64_t bb = (uint64_t)(dist * inv_width);
    return bb >= nb ? nb - 1 : (uint32_t)bb;
}

// Warp-specialised tensor-core kernel (one block = one work item):
//   warp 0      TMA producer: candidate tiles (128 rows of the level's B operand)
//               into a STAGES-deep smem ring (also owns the TMEM allocation)
//   warp 1      MMA issuer: per tile and query group g, 4*KB UMMAs (M=128,N=128,K=16)
//               into accumulator (g, t&1) of TMEM; commits free the smem stage and
//               signal the epilogue
//   warps 2..   epilogue, 4 warps per query group (TMEM lane quarters):
//               JOIN: screened top-K list insertion; HIST: exact-certain binning
// Every role walks the same deterministic tile sequence (ranges of the item,
// <=TN positions per tile, tiles never straddle a range). Only the first p.ksteps
// K=16 steps of the operand rows hold non-zero columns (ceil((3n+2)/16)); the MMA
// warp issues just those (n = 4: one UMMA per tile instead of four).
// TN = 64: wide operands (KB >= 3), so that A + the B ring fit in shared memory.
template <int KB, int G, int STAGES, bool HIST, int LR, int TN = 128>
__global__ void __launch_bounds__(32 * (1 + G) + 128 * G, 1)
    k_tc(const __grid_constant__ CUtensorMap tmB, TcJoinArgs p) {
    constexpr int NQ = 128 * G;                    // queries per block
    constexpr int BK = TN * 128;                   // bytes of one k-block of a candidate tile
    // accumulator buffers per group: all 512 TMEM columns when the CTA has the SM to itself
    // (G = 2, or a deep B ring whose shared memory admits one CTA); 256 for the two-per-SM
    // shape (STAGES = 2). More buffers let a group's epilogue warps drift further apart
    // (one warp's rare path no longer stalls the MMA into the next buffer).
    constexpr int NB = (G == 2 || STAGES > 2 ? 512 : 256) / (G * TN);
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    // 1024-byte alignment for the 128B-swizzle atoms, staying in the shared state space
    unsigned char* base = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    unsigned char* sA = base;                                   // G x KB x 16 KB
    unsigned char* sB = sA + G * KB * KB_BYTES;                 // STAGES x KB x BK
    unsigned char* tail = sB + STAGES * KB * BK;
    // accumulator barriers per (query group, buffer): the groups' pipelines are decoupled
    __shared__ uint64_t bar_full[STAGES], bar_empty[STAGES], bar_accf[G * NB], bar_acce[G * NB];
    __shared__ uint32_t s_tmem;

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
#ifdef KNNJ_TC_CLOCKS
    unsigned long long ck[16] = {};
    const long long ck_start = clock64();
#endif
    const uint4 it = p.items[blockIdx.x];
    const uint32_t nq = it.y - it.x;
    constexpr uint32_t TMEM_COLS = G * NB * TN;

    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         smem_u32(&s_tmem)),
                     "n"(TMEM_COLS));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (tid == 32) {
        for (int i = 0; i < STAGES; ++i) {
            mbar_init(&bar_full[i], 1);
            mbar_init(&bar_empty[i], G);  // one MMA commit per query group
        }
        for (int i = 0; i < G * NB; ++i) {
            mbar_init(&bar_accf[i], 1);
            mbar_init(&bar_acce[i], 4);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&tmB) : "memory");
    }

    // epilogue identity
    // warp 0: TMA producer; warps 1 .. G: MMA issuers (one per query group, so a group
    // waiting on its epilogue never stalls the other's issue through lane divergence);
    // then 4 epilogue warps per group (any 4 consecutive warps cover the 4 TMEM lane quarters)
    constexpr int NSPEC = 1 + G;
    const int e = warp - NSPEC;                  // epilogue warp index (valid if >= 0)
    const int g = e >= 0 ? e >> 2 : 0;           // query group
    const int quarter = warp & 3;                // TMEM lane quarter this warp may access
    const uint32_t r = quarter * 32 + lane;      // accumulator row (= TMEM lane)
    const uint32_t qi = g * 128 + r;             // query index inside the item
    const bool epi = e >= 0 && e < 4 * G;
    const bool has_q = epi && qi < nq;
    const uint32_t row = it.x + (has_q ? qi : 0);
    const uint32_t qp = p.qpos[row];
    float na = 0.f;
    if (epi) {
        // A operand row r of group g: [-2hi, -2lo, -2hi, 1, 1, 0...] against the B row
        // [lo, hi, hi, nb_hi, nb_lo, 0...], with the 128B swizzle
        const __half* qrow_g = p.Bh + (uint64_t)qp * p.row_halfs;
        const uint32_t n = p.n;
        for (int kb = 0; kb < KB; ++kb) {
            unsigned char* blk =
                sA + (g * KB + kb) * KB_BYTES + (r >> 3) * 1024 + (r & 7) * 128;
#pragma unroll
            for (int c = 0; c < 8; ++c) {
                uint32_t w[4];
#pragma unroll
                for (int e2 = 0; e2 < 4; ++e2) {
                    uint32_t pair = 0;
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        const uint32_t k = kb * KBLK + c * 8 + e2 * 2 + h;
                        __half v = __float2half(0.f);
                        if (has_q) {
                            // x2 is exact in FP16: the operand carries -2a unrounded
                            if (k < n) v = __hmul(__float2half(-2.f), qrow_g[k + n]);         // -2 a_hi
                            else if (k < 2 * n) v = __hmul(__float2half(-2.f), qrow_g[k - n]);  // -2 a_lo
                            else if (k < 3 * n) v = __hmul(__float2half(-2.f), qrow_g[k]);      // -2 a_hi
                            else if (k < 3 * n + 2) v = __float2half(1.f);
                        }
                        pair |= (uint32_t)__half_as_ushort(v) << (16 * h);
                    }
                    w[e2] = pair;
                }
                *reinterpret_cast<uint4*>(blk + ((c ^ (r & 7)) * 16)) =
                    make_uint4(w[0], w[1], w[2], w[3]);
            }
        }
    }
    if (has_q) {
        const __half* qrow_g = p.Bh + (uint64_t)qp * p.row_halfs;
        na = __half2float(qrow_g[3 * p.n]) + __half2float(qrow_g[3 * p.n + 1]);
    }
    if (HIST) {
        uint32_t* hist = reinterpret_cast<uint32_t*>(tail);
        float* tab = reinterpret_cast<float*>(hist + p.n_bins * NQ);
        for (uint32_t i = tid; i < p.n_bins * NQ; i += blockDim.x) hist[i] = 0;
        for (uint32_t i = tid; i < 2 * (p.n_bins + 1); i += blockDim.x) tab[i] = p.tables[i];
        float2* lh = reinterpret_cast<float2*>(tab + 2 * (p.n_bins + 1));
        for (uint32_t i = tid; i < p.n_bins; i += blockDim.x)
            lh[i] = make_float2(p.tables[i], p.tables[p.n_bins + 1 + i]);
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    fence_before();
    __syncthreads();
    fence_after();
    const uint32_t tmem = s_tmem;
#ifdef KNNJ_TC_CLOCKS
    const long long ck_loop = clock64();
    ck[11] += ck_loop - ck_start;
#endif

    // Deterministic tile sequence over the item's ranges. In the first range (the
    // item's own cell row, where its queries live) the sweep starts at the tile
    // holding the item's first query and wraps around: with the within-cell
    // locality order the nearest candidates come first and the top-K cut
    // converges after one tile.
    uint32_t cur_ri = it.z, cur_off = 0, first_start = 0, first_done = 0;
    if (!HIST && it.z < it.w) {
        const uint2 rg0 = p.adj[it.z];
        const uint32_t q0pos = p.qpos[it.x];
        if (q0pos >= rg0.x && q0pos < rg0.y) first_start = ((q0pos - rg0.x) / TN) * TN;
    }
    auto next_tile = [&](uint32_t& s, uint32_t& c) -> bool {
        if (cur_ri == it.z && cur_ri < it.w) {  // first range: [first_start, len) then [0, first_start)
            const uint2 rg = p.adj[cur_ri];
            const uint32_t len = rg.y - rg.x;
            while (first_done < len) {
                const uint32_t off = (first_start + first_done) % len;
                const uint32_t seg_end = off >= first_start ? len : first_start;
                s = rg.x + off;
                c = min((uint32_t)TN, seg_end - off);
                first_done += c;
                return true;
            }
            ++cur_ri;
            cur_off = 0;
        }
        while (cur_ri < it.w) {
            const uint2 rg = p.adj[cur_ri];
            const uint32_t len = rg.y - rg.x;
            if (cur_off < len) {
                s = rg.x + cur_off;
                c = min((uint32_t)TN, len - cur_off);
                cur_off += c;
                if (cur_off == len) {
                    ++cur_ri;
                    cur_off = 0;
                }
                return true;
            }
            ++cur_ri;
            cur_off = 0;
        }
        return false;
    };

    if (warp == 0) {
        // ------------------------------------------------ TMA producer
        if (lane == 0) {
            uint32_t s, c;
            for (uint32_t t = 0; next_tile(s, c); ++t) {
                const int st = t % STAGES;
                TCK(w0);
                mbar_wait(&bar_empty[st], ((t / STAGES) & 1) ^ 1);
                TCK(w1);
                TCADD(8, w0, w1);
                mbar_expect_tx(&bar_full[st], KB * BK);
#pragma unroll
                for (int kb = 0; kb < KB; ++kb)
                    tma_load_2d(sB + (st * KB + kb) * BK, &tmB, &bar_full[st], kb * KBLK, (int)s);
            }
        }
    } else if (warp <= G) {
        // ------------------------------------------------ MMA issuer
        // one issuing warp per query group: a group whose epilogue is in its rare path
        // holds only its own accumulators; the other runs ahead within the stage ring
        if (lane == 0) {
            const int gg = warp - 1;
            uint32_t s, c;
            const uint32_t a0 = smem_u32(sA);
            for (uint32_t t = 0; next_tile(s, c); ++t) {
                const int st = t % STAGES, b = t % NB;
                TCK(w0);
                mbar_wait(&bar_full[st], (t / STAGES) & 1);
                TCK(w1);
                mbar_wait(&bar_acce[gg * NB + b], ((t / NB) & 1) ^ 1);
                TCK(w2);
                TCADD(9, w0, w1);
                TCADD(10, w1, w2);
                fence_after();
                const uint32_t b0 = smem_u32(sB + st * KB * BK);
                const uint32_t dcol = tmem + (gg * NB + b) * TN;
#pragma unroll
                for (int kb = 0; kb < KB; ++kb)
#pragma unroll
                    for (int kk = 0; kk < KBLK / 16; ++kk)
                        if ((uint32_t)(kb * (KBLK / 16) + kk) < p.ksteps)
                            umma_f16<TN>(dcol, umma_desc_sw128(a0 + (gg * KB + kb) * KB_BYTES + kk * 32),
                                         umma_desc_sw128(b0 + kb * BK + kk * 32), (kb | kk) ? 1u : 0u);
                umma_commit(&bar_empty[st]);
                umma_commit(&bar_accf[gg * NB + b]);
            }
        }
    } else if (!HIST) {
        // ------------------------------------------------ JOIN epilogue
        // Per query an UNSORTED buffer (capacity p.L <= 64) of every candidate
        // that passed the cut; the cut tightens when a full buffer is
        // compacted warp-cooperatively (K-th key + 2 delta). Fast path: one
        // FMNMX per pair; survivors are re-read from TMEM one warp-uniform
        // column at a time (no per-lane dynamic indexing).
        // lists in shared memory, [NQ][L]
        float* lkey = reinterpret_cast<float*>(tail);
        uint32_t* lpos = reinterpret_cast<uint32_t*>(lkey + p.L * NQ);
        const uint32_t LB = p.L;
        float* mykey = lkey + (size_t)qi * LB;
        uint32_t* mypos = lpos + (size_t)qi * LB;
        uint32_t cnt = 0;
        bool ovf = false;
        const float init_cut = (p.init_cut && has_q) ? p.init_cut[row] : CUDART_INF_F;
        const float dl = p.item_delta ? p.item_delta[blockIdx.x] : p.delta;
        const float cap = __fadd_ru(init_cut, dl);        // U + delta
        float cut = cap;
        float rhs = has_q ? __fsub_ru(cut, na) : -CUDART_INF_F;
        // compact the buffer of query column `src_lane` (all lanes cooperate)
        auto compact = [&](int src) {
            __syncwarp();  // the src lane's appends are visible to the warp
            const uint32_t c_src = __shfl_sync(0xffffffffu, cnt, src);
            const uint32_t col = g * 128 + quarter * 32 + src;
            float* kb = lkey + (size_t)col * LB;
            uint32_t* pb = lpos + (size_t)col * LB;
            float kv[LR];
            uint32_t pv[LR];
#pragma unroll
            for (int r = 0; r < LR; ++r) {
                const uint32_t i = r * 32 + lane;
                kv[r] = i < c_src ? kb[i] : CUDART_INF_F;
                pv[r] = i < c_src ? pb[i] : 0u;
            }
            float srt[LR];
#pragma unroll
            for (int r = 0; r < LR; ++r) srt[r] = kv[r];
            const float kth = warp_kth<LR>(srt, p.K);
            const float cap_src = __shfl_sync(0xffffffffu, cap, src);
            const float nc = fminf(__fadd_ru(kth, 2.f * dl), cap_src);
            unsigned bal[LR];
#pragma unroll
            for (int r = 0; r < LR; ++r) bal[r] = __ballot_sync(0xffffffffu, kv[r] <= nc);
            const unsigned lt = (1u << lane) - 1u;
            __syncwarp();
            uint32_t at = 0;
#pragma unroll
            for (int r = 0; r < LR; ++r) {
                if (kv[r] <= nc) {
                    kb[at + __popc(bal[r] & lt)] = kv[r];
                    pb[at + __popc(bal[r] & lt)] = pv[r];
                }
                at += __popc(bal[r]);
            }
            __syncwarp();
            if (lane == src) {
                cnt = at;
                cut = nc;
                rhs = __fsub_ru(cut, na);
                if (cnt >= LB) {  // every entry inside the band: exact ties, slow path
                    ovf = true;
                    rhs = -CUDART_INF_F;
                }
            }
        };
        uint32_t s, c;
        unsigned long long st_slab = 0, st_rare = 0, st_bits = 0, st_ins = 0, st_cmp = 0;
        for (uint32_t t = 0; next_tile(s, c); ++t) {
            const int b = t % NB;
            TCK(e0);
            mbar_wait(&bar_accf[g * NB + b], (t / NB) & 1);
            TCK(e1);
            TCADD(0, e0, e1);
            fence_after();
            const uint32_t tbase = tmem + ((uint32_t)(quarter * 32) << 16) + (g * NB + b) * TN;
            for (uint32_t j0 = 0; j0 < c; j0 += 64) {
                float v0[32], v1[32];
                TCK(l0);
                tmem_ld64(tbase + j0, v0, v1);
                TCK(l1);
                TCADD(1, l0, l1);
                if (p.dbg && blockIdx.x == 0 && t == 0 && g == 0)
#pragma unroll
                    for (int j = 0; j < 32; ++j) {
                        p.dbg[r * TC_N + j0 + j] = v0[j];
                        p.dbg[r * TC_N + j0 + 32 + j] = v1[j];
                    }
                const uint32_t lim = c - j0;  // valid columns in this 64-column slab
                if (lim < 64) {
#pragma unroll
                    for (int j = 0; j < 32; ++j) {
                        if ((uint32_t)j >= lim) v0[j] = CUDART_NAN_F;
                        if ((uint32_t)(j + 32) >= lim) v1[j] = CUDART_NAN_F;
                    }
                }
                const bool hit = has_q && !ovf && slab_min64(v0, v1) <= rhs;
                ++st_slab;
                const bool any_hit = __any_sync(0xffffffffu, hit);
                TCK(l2);
                TCADD(2, l1, l2);
                if (!any_hit) continue;
                ++st_rare;
                // rare path: each lane walks its own hit columns, the values picked from
                // registers; the warp loops max-over-lanes times, not once per column any
                // lane hit. A lane's inserts keep their column order, so its list and cut
                // evolve exactly as in a column-at-a-time walk.
                unsigned mk[2] = {0u, 0u};
                if (hit) {
#pragma unroll
                    for (int j = 0; j < 32; ++j) {
                        mk[0] |= (v0[j] <= rhs ? 1u : 0u) << j;
                        mk[1] |= (v1[j] <= rhs ? 1u : 0u) << j;
                    }
                }
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    unsigned m = mk[h];
                    while (__any_sync(0xffffffffu, m != 0u)) {
                        const bool act = m != 0u;
                        const int j = act ? __ffs(m) - 1 : 0;
                        m &= m - 1u;
                        ++st_bits;
                        const float x = pick32(h ? v1 : v0, j);
                        const uint32_t pos = s + j0 + h * 32 + j;
                        bool want = act && x <= rhs && pos != qp;
                        // make room: cooperative compaction of every full buffer that needs it
                        unsigned full = __ballot_sync(0xffffffffu, want && cnt == LB);
                        TCK(r1);
                        while (full) {
                            const int src = __ffs(full) - 1;
                            full &= full - 1;
                            ++st_cmp;
                            compact(src);
                        }
                        TCK(r2);
                        TCADD(5, r1, r2);
                        want = want && !ovf && x <= rhs;  // cut may have tightened
                        if (want) {
                            mykey[cnt] = x + na;
                            mypos[cnt] = pos;
                            ++cnt;
                            ++st_ins;
                        }
                    }
                }
                TCK(l3);
                TCADD(3, l2, l3);
            }
            fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&bar_acce[g * NB + b]);
            TCK(e2);
            TCADD(4, e0, e2);
        }
        if (p.stats) {  // bits: warp iterations of the rare loop; inserts: list appends
            atomicAdd(p.stats + 3, st_ins);
            if (lane == 0) {
                atomicAdd(p.stats + 2, st_bits);
                atomicAdd(p.stats + 0, st_slab);
                atomicAdd(p.stats + 1, st_rare);
                atomicAdd(p.stats + 4, st_cmp);
            }
        }
        if (has_q) {
            p.out_cnt[row] = ovf ? OVF : cnt;
            if (!ovf)
                for (uint32_t i = 0; i < cnt; ++i) p.out_pos[(uint64_t)row * LB + i] = mypos[i];
        }
    } else {
        // ------------------------------------------------ HISTOGRAM epilogue
        uint32_t* hist = reinterpret_cast<uint32_t*>(tail);          // [n_bins][NQ]
        const float* LO = reinterpret_cast<const float*>(hist + p.n_bins * NQ);
        const float* HI = LO + p.n_bins + 1;
        const float2* LH = reinterpret_cast<const float2*>(HI + p.n_bins + 1);  // [n_bins]
        uint2* qbuf = reinterpret_cast<uint2*>(const_cast<float2*>(LH + p.n_bins)) + e * 32;
        const uint32_t nbins = p.n_bins, ncount = p.n_count;
        const bool capped = ncount < nbins;  // counts only the low bins select_eps_beta needs
        const float dl = p.delta;
        const float skip_at = has_q ? __fsub_ru(__fadd_ru(LO[ncount], dl), na) : -CUDART_INF_F;
        const float invw = p.inv_width_scaled;
        uint32_t qn = 0;  // warp-uniform queue fill
        // resolve queued pairs: one per lane, FP64 scalar order, exact bin
        auto flush = [&]() {
            if (lane < qn) {
                const uint2 pr = qbuf[lane];  // (query column, candidate position)
                const uint32_t qcol = pr.x & 0xFFFFu;
                const uint32_t qps = p.qpos[it.x + qcol];
                const uint32_t qid = p.A ? p.A[qps] : qps;   // positions -> point ids
                const uint32_t cid = p.A ? p.A[pr.y] : pr.y;
                const uint32_t bb =
                    exact_bin(p.X64, p.n, qid, cid, p.eps_mean, p.limit_sq, p.inv_width, nbins);
                if (bb < ncount) atomicAdd(&hist[bb * NQ + qcol], 1u);
            }
            __syncwarp();
            qn = 0;
        };
        // warp-cooperative append of one ambiguous pair per lane (need = this lane has one)
        auto enqueue = [&](bool need, uint32_t pos) {
            const unsigned m = __ballot_sync(0xffffffffu, need);
            if (!m) return;
            if (qn + __popc(m) > 32) flush();
            if (need) qbuf[qn + __popc(m & ((1u << lane) - 1u))] = make_uint2(qi, pos);
            __syncwarp();
            qn += __popc(m);
        };
        uint32_t s, c;
        for (uint32_t t = 0; next_tile(s, c); ++t) {
            const int b = t % NB;
            mbar_wait(&bar_accf[g * NB + b], (t / NB) & 1);
            fence_after();
            const uint32_t tbase = tmem + ((uint32_t)(quarter * 32) << 16) + (g * NB + b) * TN;
            for (uint32_t j0 = 0; j0 < c; j0 += 64) {
                float v[2][32];
                tmem_ld64(tbase + j0, v[0], v[1]);
                const uint32_t lim = has_q ? c - j0 : 0;
                const uint32_t selfj = qp - (s + j0);  // column of the self pair (if any)
                if (capped) {
                    // Sparse path: nearly every pair lies beyond the cap edge. One FMNMX
                    // per pair decides the slab; survivors are re-read from TMEM one
                    // warp-uniform column at a time and binned like the dense path.
                    if (lim < 64) {
#pragma unroll
                        for (int j = 0; j < 32; ++j) {
                            if ((uint32_t)j >= lim) v[0][j] = CUDART_NAN_F;
                            if ((uint32_t)(j + 32) >= lim) v[1][j] = CUDART_NAN_F;
                        }
                    }
                    const bool hit = slab_min64(v[0], v[1]) < skip_at;
                    if (!__any_sync(0xffffffffu, hit)) continue;
                    unsigned mk[2] = {0u, 0u};
                    if (hit) {
#pragma unroll
                        for (int j = 0; j < 32; ++j) {
                            mk[0] |= (v[0][j] < skip_at ? 1u : 0u) << j;
                            mk[1] |= (v[1][j] < skip_at ? 1u : 0u) << j;
                        }
                    }
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        unsigned um = __reduce_or_sync(0xffffffffu, mk[h]);
                        while (um) {
                            const int j = __ffs(um) - 1;
                            um &= um - 1;
                            const uint32_t jj = h * 32 + j;
                            const float x = tmem_ld1(tbase + j0 + jj);
                            const bool valid = ((mk[h] >> j) & 1u) && jj != selfj;
                            const float key = x + na;
                            const float klo = __fsub_rd(key, dl), khi = __fadd_ru(key, dl);
                            const float rt = fmaxf(key, 1e-30f);
                            int bin = __float2int_rz(rt * rsqrtf(rt) * invw);
                            bin = min(bin, (int)nbins - 1);
                            const float2 edge = LH[bin];
                            const bool certain = valid && klo >= edge.x && khi < edge.y;
                            if (certain && (uint32_t)bin < ncount) hist[(uint32_t)bin * NQ + qi] += 1u;
                            enqueue(valid && !certain, s + j0 + jj);
                        }
                    }
                    continue;
                }
                unsigned am[2] = {0u, 0u};
                // branch-free per pair: in range & not self -> exact-certain bin from
                // key +- delta against the interleaved (LO,HI) edge table, else queue
#pragma unroll
                for (int h = 0; h < 2; ++h)
#pragma unroll
                    for (int j = 0; j < 32; ++j) {
                        const uint32_t jj = h * 32 + j;
                        const float key = v[h][j] + na;
                        const bool valid = (jj < lim) & (v[h][j] < skip_at) & (jj != selfj);
                        const float klo = __fsub_rd(key, dl), khi = __fadd_ru(key, dl);
                        const float rt = fmaxf(key, 1e-30f);
                        int bin = __float2int_rz(rt * rsqrtf(rt) * invw);
                        bin = min(bin, (int)nbins - 1);
                        const float2 edge = LH[bin];
                        const bool certain = valid & (klo >= edge.x) & (khi < edge.y);
                        const uint32_t hidx = (uint32_t)bin * NQ + qi;
                        hist[hidx] += certain ? 1u : 0u;
                        am[h] |= ((valid & !certain) ? 1u : 0u) << j;
                    }
                // queue ambiguous pairs (one per lane per round), resolve 32 at a time
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    unsigned mine = am[h];
                    while (true) {
                        const bool has = mine != 0u;
                        const unsigned m = __ballot_sync(0xffffffffu, has);
                        if (!m) break;
                        if (qn + __popc(m) > 32) flush();
                        if (has) {
                            const int j = __ffs(mine) - 1;
                            mine &= mine - 1;
                            qbuf[qn + __popc(m & ((1u << lane) - 1u))] =
                                make_uint2(qi, s + j0 + h * 32 + j);
                        }
                        __syncwarp();
                        qn += __popc(m);
                    }
                }
            }
            fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&bar_acce[g * NB + b]);
        }
        flush();
    }
#ifdef KNNJ_TC_CLOCKS
    ck[12] += clock64() - ck_loop;
    if (p.stats && lane == 0 && !HIST) {
        // epilogue warps: 0 accf wait, 1 ld64, 2 fast, 3 rare, 4 loop total, 11 prologue,
        // 12 role total; producer 8 (empty waits) + 13 total; MMA 9 full, 10 acce + 14 total
        const int role = warp == 0 ? 0 : (warp <= G ? 1 : 2);
        if (role == 2)
            for (int i : {0, 1, 2, 3, 4, 5, 6, 11, 12}) atomicAdd(p.stats + 8 + i, ck[i]);
        else if (role == 0) {
            atomicAdd(p.stats + 8 + 8, ck[8]);
            atomicAdd(p.stats + 8 + 13, ck[12]);
        } else {
            atomicAdd(p.stats + 8 + 9, ck[9]);
            atomicAdd(p.stats + 8 + 10, ck[10]);
            atomicAdd(p.stats + 8 + 14, ck[12]);
        }
        if (role == 2) atomicAdd(p.stats + 8 + 15, 1ull);  // epilogue warps
    }
#endif
    fence_before();
    __syncthreads();
    if (HIST) {
        uint32_t* hist = reinterpret_cast<uint32_t*>(tail);
        for (uint32_t bb = tid; bb < p.n_bins; bb += blockDim.x) {
            unsigned long long sum = 0;
            for (int q = 0; q < NQ; ++q) sum += hist[bb * NQ + ((q + bb) & (NQ - 1))];
            if (sum) atomicAdd(&p.counts[bb], sum);
        }
    }
    if (warp == 0) {
        fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                     "n"(TMEM_COLS));
    }
}

// ---------------------------------------------------------------- host side
size_t tc_smem_bytes(const TcShape& sh, uint32_t L, uint32_t n_bins, bool hist) {
    const size_t NQ = 128 * sh.G;
    size_t b = 1024 + (size_t)sh.G * sh.KB * KB_BYTES + (size_t)sh.STAGES * sh.KB * sh.TN * 128;
    if (hist) b += NQ * n_bins * 4 + 8 * (n_bins + 1) + 8 * n_bins + 8 + (size_t)4 * sh.G * 32 * 8;
    else b += NQ * L * 8;
    return b;
}

// k_prep_tc for a compile-time n <= 8: the row's halfs from registers (no per-half
// division by n, no re-reads of the point row); the same values, bit for bit
template <int NN>
__global__ void k_prep_tc_n(const double* X64, const uint32_t* A, uint64_t N, const double* g,
                            double inv_S, uint32_t row_halfs, __half* Bh, uint32_t write_halfs) {
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < N;
         i += uint64_t(gridDim.x) * blockDim.x) {
        const double* x = X64 + (uint64_t)A[i] * NN;
        double nb = 0.0;
        __half hi[NN], lo[NN];
#pragma unroll
        for (int d = 0; d < NN; ++d) {
            const double v = (x[d] - g[d]) * inv_S;
            nb += v * v;
            hi[d] = __double2half(v);
            lo[d] = __double2half(v - (double)__half2float(hi[d]));
        }
        const __half nh = __double2half(nb);
        const __half nl = __double2half(nb - (double)__half2float(nh));
        constexpr int O = 3 * NN;
        constexpr int NZ = ((O + 2 + 7) / 8) * 8;  // the 16-byte chunks holding non-zeros
        uint4* row = reinterpret_cast<uint4*>(Bh + i * row_halfs);
#pragma unroll
        for (int c0 = 0; c0 < NZ; c0 += 8) {
            uint32_t w[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                uint32_t pair = 0;
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const int k = c0 + 2 * e + h;  // lo | hi | hi | nb_hi | nb_lo | 0...
                    const __half hv = k < NN ? lo[k < NN ? k : 0]
                                      : k < 2 * NN ? hi[k < 2 * NN ? k - NN : 0]
                                      : k < O ? hi[k < O ? k - 2 * NN : 0]
                                      : k == O ? nh : k == O + 1 ? nl : __float2half(0.f);
                    pair |= (uint32_t)__half_as_ushort(hv) << (16 * h);
                }
                w[e] = pair;
            }
            row[c0 / 8] = make_uint4(w[0], w[1], w[2], w[3]);
        }
        // (write_halfs < row_halfs: the rest of the row is known zero from an earlier build)
        for (uint32_t c0 = NZ; c0 < write_halfs; c0 += 8) row[c0 / 8] = make_uint4(0u, 0u, 0u, 0u);
    }
}

void launch_prep_tc(const double* X64, const uint32_t* A, uint64_t N, uint32_t n, const double* g,
                    double inv_S, uint32_t row_halfs, __half* Bh, cudaStream_t s, uint32_t write_halfs) {
    if (write_halfs == 0 || write_halfs > row_halfs) write_halfs = row_halfs;
    switch (n) {
#define KJ_PREP(NN)                                                                            \
    case NN:                                                                                   \
        k_prep_tc_n<NN><<<2368, 256, 0, s>>>(X64, A, N, g, inv_S, row_halfs, Bh, write_halfs); \
        break;
        KJ_PREP(1) KJ_PREP(2) KJ_PREP(3) KJ_PREP(4) KJ_PREP(5) KJ_PREP(6) KJ_PREP(7) KJ_PREP(8)
#undef KJ_PREP
        default: k_prep_tc<<<2368, 256, 0, s>>>(X64, A, N, n, g, inv_S, row_halfs, Bh, write_halfs);
    }
    KJ_CUDA(cudaGetLastError());
    g_launches.fetch_add(1, std::memory_order_relaxed);
}

static PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    if (!fn) {
        cudaDriverEntryPointQueryResult q;
        void* ptr = nullptr;
        KJ_CUDA(cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &ptr, 12000,
                                                 cudaEnableDefault, &q));
        if (q != cudaDriverEntryPointSuccess || !ptr)
            throw Error(9, "cuTensorMapEncodeTiled unavailable");
        fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(ptr);
    }
    return fn;
}

template <int KB, int G, int STAGES, bool HIST, int LR, int TN = 128>
static void launch_tc_t(const TcJoinArgs& a, uint64_t nitems, uint64_t N, cudaStream_t s) {
    CUtensorMap map;
    cuuint64_t dims[2] = {(cuuint64_t)a.row_halfs, (cuuint64_t)N};
    cuuint64_t strides[1] = {(cuuint64_t)a.row_halfs * 2};
    cuuint32_t box[2] = {KBLK, (cuuint32_t)TN};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = get_encode()(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, (void*)a.Bh, dims, strides,
                              box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                              CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw Error(9, "cuTensorMapEncodeTiled failed: " + std::to_string((int)r));
    const size_t sm = tc_smem_bytes(TcShape{KB, G, STAGES, TN}, a.L, a.n_bins, HIST);
    if (sm > 227 * 1024) throw Error(1, "tensor-core kernel needs too much shared memory");
    KJ_CUDA(cudaFuncSetAttribute(k_tc<KB, G, STAGES, HIST, LR, TN>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    for (uint64_t off = 0; off < nitems; off += 2147483647ull) {
        const uint64_t cnt = std::min<uint64_t>(nitems - off, 2147483647ull);
        TcJoinArgs b = a;
        b.items = a.items + off;
        k_tc<KB, G, STAGES, HIST, LR, TN><<<(unsigned)cnt, 32 * (1 + G) + 128 * G, sm, s>>>(map, b);
    }
    KJ_CUDA(cudaGetLastError());
    g_launches.fetch_add(1, std::memory_order_relaxed);
}

void launch_join_tc(const TcJoinArgs& a, const TcShape& sh, uint64_t nitems, uint64_t N,
                    cudaStream_t s) {
    if (!nitems) return;
    const bool wide = a.L > 64;  // list compaction over 128 entries
    if (sh.TN == 64) {  // wide operands (KB >= 3), 64-candidate tiles
        if (sh.KB == 3 && sh.G == 1 && sh.STAGES == 3 && !wide) launch_tc_t<3, 1, 3, false, 2, 64>(a, nitems, N, s);
        else if (sh.KB == 4 && sh.G == 1 && sh.STAGES == 3 && !wide) launch_tc_t<4, 1, 3, false, 2, 64>(a, nitems, N, s);
        else if (sh.KB == 5 && sh.G == 1 && sh.STAGES == 2 && !wide) launch_tc_t<5, 1, 2, false, 2, 64>(a, nitems, N, s);
        else throw Error(1, "no wide-operand tensor-core join instance for this shape");
        return;
    }
    if (sh.KB == 1 && sh.G == 2 && sh.STAGES == 4 && !wide) launch_tc_t<1, 2, 4, false, 2>(a, nitems, N, s);
    else if (sh.KB == 1 && sh.G == 1 && sh.STAGES == 2 && !wide) launch_tc_t<1, 1, 2, false, 2>(a, nitems, N, s);
    else if (sh.KB == 1 && sh.G == 1 && sh.STAGES == 4 && wide) launch_tc_t<1, 1, 4, false, 4>(a, nitems, N, s);
    else if (sh.KB == 2 && sh.G == 1 && sh.STAGES == 3 && !wide) launch_tc_t<2, 1, 3, false, 2>(a, nitems, N, s);
    else if (sh.KB == 2 && sh.G == 1 && sh.STAGES == 2 && wide) launch_tc_t<2, 1, 2, false, 4>(a, nitems, N, s);
    else throw Error(1, "no tensor-core join instance for this shape");
}

void launch_hist_tc(const TcJoinArgs& a, const TcShape& sh, uint64_t nitems, uint64_t N,
                    cudaStream_t s) {
    if (!nitems) return;
    if (sh.KB == 1 && sh.G == 2 && sh.STAGES == 4) launch_tc_t<1, 2, 4, true, 2>(a, nitems, N, s);
    else if (sh.KB == 2 && sh.G == 1 && sh.STAGES == 3) launch_tc_t<2, 1, 3, true, 2>(a, nitems, N, s);
    else throw Error(1, "no tensor-core histogram instance for this shape");
}

}  // namespace kj
