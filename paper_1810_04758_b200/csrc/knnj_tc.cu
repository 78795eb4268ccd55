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
    asm volatile(
        "{\n\t.reg .pred P;\n\t"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n\t"
        "@!P bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
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
constexpr uint32_t IDESC = (1u << 4) | (0u << 7) | (0u << 10) | ((uint32_t)(TC_N >> 3) << 17) |
                           ((uint32_t)(TC_M >> 4) << 24);

__device__ __forceinline__ void umma_f16(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(da), "l"(db), "r"(IDESC), "r"(acc));
}
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                     smem_u32(bar))
                 : "memory");
}

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float (&v)[32]) {
    uint32_t r[32];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
          "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]),
          "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]),
          "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
          "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]),
          "=r"(r[31])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

}  // namespace

// B-operand rows for one grid level, sorted order: [hi | lo | hi | nb_hi nb_lo | 0]
__global__ void k_prep_tc(const double* X64, const uint32_t* A, uint64_t N, uint32_t n,
                          const double* g, double inv_S, uint32_t row_halfs, __half* Bh) {
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < N;
         i += uint64_t(gridDim.x) * blockDim.x) {
        const double* x = X64 + (uint64_t)A[i] * n;
        __half* row = Bh + i * row_halfs;
        double nb = 0.0;
        for (uint32_t d = 0; d < n; ++d) {
            const double v = (x[d] - g[d]) * inv_S;
            const __half hi = __double2half(v);
            const __half lo = __double2half(v - (double)__half2float(hi));
            row[d] = hi;
            row[n + d] = lo;
            row[2 * n + d] = hi;
            nb += v * v;
        }
        const __half nh = __double2half(nb);
        row[3 * n] = nh;
        row[3 * n + 1] = __double2half(nb - (double)__half2float(nh));
        for (uint32_t c = 3 * n + 2; c < row_halfs; ++c) row[c] = __float2half(0.f);
    }
}

// One block = one work item (<=128 queries of one cell).
template <int KB>
__global__ void __launch_bounds__(TC_M, 2)
    k_join_tc(const __grid_constant__ CUtensorMap tmB, TcJoinArgs p) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    // 1024-byte alignment for the 128B-swizzle atoms
    unsigned char* base = reinterpret_cast<unsigned char*>(
        (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    unsigned char* sA = base;                         // KB x 16 KB
    unsigned char* sB = sA + KB * KB_BYTES;           // 2 stages x KB x 16 KB
    float* lkey = reinterpret_cast<float*>(sB + 2 * KB * KB_BYTES);  // [L][128]
    uint32_t* lpos = reinterpret_cast<uint32_t*>(lkey + p.L * TC_M);
    float* scr = reinterpret_cast<float*>(lpos + p.L * TC_M);        // [32][128] survivor scratch

    __shared__ uint64_t bar_full[2], bar_mma[2];
    __shared__ uint32_t s_tmem;
    __shared__ uint32_t s_tile_s[4], s_tile_c[4];   // ring of tile descriptors
    __shared__ uint32_t s_ri, s_off;

    const int tid = threadIdx.x, warp = tid >> 5;
    const uint4 it = p.items[blockIdx.x];
    const uint32_t nq = it.y - it.x;
    const bool has_q = (uint32_t)tid < nq;
    const uint32_t row = it.x + (has_q ? tid : 0);
    const uint32_t qp = p.qpos[row];

    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(
            smem_u32(&s_tmem)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (tid == 0) {
        mbar_init(&bar_full[0], 1);
        mbar_init(&bar_full[1], 1);
        mbar_init(&bar_mma[0], 1);
        mbar_init(&bar_mma[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&tmB) : "memory");
        s_ri = it.z;
        s_off = 0;
    }
    // A operand: this thread's query row, written with the 128B swizzle
    const __half* qrow_g = p.Bh + (uint64_t)qp * p.row_halfs;
    float na = 0.f;
    {
        const uint32_t n = p.n;
        for (int kb = 0; kb < KB; ++kb) {
            unsigned char* blk = sA + kb * KB_BYTES + (tid >> 3) * 1024 + (tid & 7) * 128;
#pragma unroll
            for (int c = 0; c < 8; ++c) {  // 16-byte chunks of this 128-byte row
                __half h[8];
#pragma unroll
                for (int e = 0; e < 8; ++e) {
                    const uint32_t k = kb * KBLK + c * 8 + e;
                    __half v = __float2half(0.f);
                    if (has_q) {
                        if (k < 2 * n) v = __hmul(__float2half(-2.f), qrow_g[k < n ? k : k - n]);
                        else if (k < 3 * n) v = __hmul(__float2half(-2.f), qrow_g[n + (k - 2 * n)]);
                        else if (k < 3 * n + 2) v = __float2half(1.f);
                    }
                    h[e] = v;
                }
                uint4 pk;
                pk.x = (uint32_t)__half_as_ushort(h[0]) | ((uint32_t)__half_as_ushort(h[1]) << 16);
                pk.y = (uint32_t)__half_as_ushort(h[2]) | ((uint32_t)__half_as_ushort(h[3]) << 16);
                pk.z = (uint32_t)__half_as_ushort(h[4]) | ((uint32_t)__half_as_ushort(h[5]) << 16);
                pk.w = (uint32_t)__half_as_ushort(h[6]) | ((uint32_t)__half_as_ushort(h[7]) << 16);
                *reinterpret_cast<uint4*>(blk + ((c ^ (tid & 7)) * 16)) = pk;
            }
        }
        if (has_q) na = __half2float(qrow_g[3 * n]) + __half2float(qrow_g[3 * n + 1]);
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    fence_before();
    __syncthreads();
    fence_after();
    const uint32_t tmem = s_tmem;

    // tile cursor (thread 0): next chunk of <=128 positions inside one range
    auto next_tile = [&](uint32_t& s, uint32_t& c) {
        c = 0;
        while (s_ri < it.w) {
            const uint2 r = p.adj[s_ri];
            if (s_off < r.y - r.x) {
                s = r.x + s_off;
                c = min((uint32_t)TC_N, r.y - r.x - s_off);
                s_off += c;
                if (s_off == r.y - r.x) {
                    ++s_ri;
                    s_off = 0;
                }
                return;
            }
            ++s_ri;
            s_off = 0;
        }
    };
    auto issue_tma = [&](int stage, uint32_t s) {
        mbar_expect_tx(&bar_full[stage], KB * KB_BYTES);
#pragma unroll
        for (int kb = 0; kb < KB; ++kb)
            tma_load_2d(sB + (stage * KB + kb) * KB_BYTES, &tmB, &bar_full[stage], kb * KBLK,
                        (int)s);
    };
    auto issue_mma = [&](int stage, int acc_buf) {
        const uint32_t a0 = smem_u32(sA), b0 = smem_u32(sB + stage * KB * KB_BYTES);
        const uint32_t dcol = tmem + acc_buf * TC_N;
#pragma unroll
        for (int kb = 0; kb < KB; ++kb)
#pragma unroll
            for (int kk = 0; kk < KBLK / 16; ++kk) {
                const uint64_t da = umma_desc_sw128(a0 + kb * KB_BYTES + kk * 32);
                const uint64_t db = umma_desc_sw128(b0 + kb * KB_BYTES + kk * 32);
                umma_f16(dcol, da, db, (kb | kk) ? 1u : 0u);
            }
        umma_commit(&bar_mma[acc_buf]);
    };

    if (tid == 0) {
        for (int t = 0; t < 2; ++t) {
            uint32_t s, c;
            next_tile(s, c);
            s_tile_s[t] = s;
            s_tile_c[t] = c;
            if (c) issue_tma(t, s);
        }
        if (s_tile_c[0]) {
            mbar_wait(&bar_full[0], 0);
            fence_after();
            issue_mma(0, 0);
        }
    }
    __syncthreads();

    int cnt = 0;
    bool ovf = false;
    float cut_list = CUDART_INF_F;
    const float init_cut = (p.init_cut && has_q) ? p.init_cut[row] : CUDART_INF_F;
    const float dl = p.delta;
    float rhs = fminf(cut_list, __fadd_ru(init_cut, dl));
    rhs = __fsub_ru(rhs, na);
    if (!has_q) rhs = -CUDART_INF_F;

    for (uint32_t t = 0;; ++t) {
        const uint32_t c = s_tile_c[t & 3];
        if (c == 0) break;
        const uint32_t s = s_tile_s[t & 3];
        const int buf = t & 1;
        // issue MMA for tile t+1 (its accumulator was drained at the end of t-1)
        if (tid == 0 && s_tile_c[(t + 1) & 3]) {
            mbar_wait(&bar_full[(t + 1) & 1], ((t + 1) >> 1) & 1);
            fence_after();
            issue_mma((t + 1) & 1, (t + 1) & 1);
        }
        mbar_wait(&bar_mma[buf], (t >> 1) & 1);
        fence_after();
        // stage `buf` is free again: prefetch tile t+2 into it
        if (tid == 0) {
            uint32_t s2, c2;
            next_tile(s2, c2);
            s_tile_s[(t + 2) & 3] = s2;
            s_tile_c[(t + 2) & 3] = c2;
            if (c2) issue_tma(buf, s2);
        }
        // epilogue: this warp's 32 TMEM lanes, columns [0, c)
        const uint32_t tbase = tmem + ((uint32_t)(warp * 32) << 16) + buf * TC_N;
        for (uint32_t j0 = 0; j0 < c; j0 += 32) {
            float v[32];
            tmem_ld32(tbase + j0, v);
            if (p.dbg && blockIdx.x == 0 && t == 0)
#pragma unroll
                for (int j = 0; j < 32; ++j) p.dbg[tid * TC_N + j0 + j] = v[j];
            if (!has_q || ovf) continue;
            const uint32_t lim = c - j0;
            if (lim < 32) {
#pragma unroll
                for (int j = 0; j < 32; ++j)
                    if ((uint32_t)j >= lim) v[j] = CUDART_NAN_F;  // never passes a <= test
            }
            // fast path: one FMNMX per pair
            float m[16];
#pragma unroll
            for (int j = 0; j < 16; ++j) m[j] = fminf(v[j], v[j + 16]);
#pragma unroll
            for (int w = 8; w > 0; w >>= 1)
#pragma unroll
                for (int j = 0; j < w; ++j) m[j] = fminf(m[j], m[j + w]);
            if (!(m[0] <= rhs)) continue;
            // rare path: survivors through this thread's smem scratch row
            uint32_t mask = 0;
#pragma unroll
            for (int j = 0; j < 32; ++j) {
                mask |= (v[j] <= rhs ? 1u : 0u) << j;
                scr[j * TC_M + tid] = v[j];
            }
            while (mask) {
                const int j = __ffs(mask) - 1;
                mask &= mask - 1;
                const float vj = scr[j * TC_M + tid];
                if (!(vj <= rhs)) continue;  // rhs may have tightened
                const uint32_t pos = s + j0 + j;
                if (pos == qp) continue;  // self pair: excluded by id
                if (cnt == (int)p.L) {
                    ovf = true;
                    rhs = -CUDART_INF_F;
                    break;
                }
                const float key = vj + na;
                int q = cnt;
                while (q > 0) {
                    const float kq = lkey[(q - 1) * TC_M + tid];
                    if (kq <= key) break;
                    lkey[q * TC_M + tid] = kq;
                    lpos[q * TC_M + tid] = lpos[(q - 1) * TC_M + tid];
                    --q;
                }
                lkey[q * TC_M + tid] = key;
                lpos[q * TC_M + tid] = pos;
                ++cnt;
                if (cnt >= (int)p.K) {
                    cut_list = __fadd_ru(lkey[(p.K - 1) * TC_M + tid], 2.f * dl);
                    const float ce = fminf(cut_list, __fadd_ru(init_cut, dl));
                    while (cnt > (int)p.K && lkey[(cnt - 1) * TC_M + tid] > ce) --cnt;
                    rhs = __fsub_ru(ce, na);
                }
            }
        }
        fence_before();
        __syncthreads();
    }
    if (has_q) {
        p.out_cnt[row] = ovf ? OVF : (uint32_t)cnt;
        if (!ovf)
            for (int i = 0; i < cnt; ++i) p.out_pos[(uint64_t)row * p.L + i] = lpos[i * TC_M + tid];
    }
    fence_before();
    __syncthreads();
    if (warp == 0) {
        fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tmem));
    }
}

// ---------------------------------------------------------------- host side
size_t tc_join_smem_bytes(int KB, uint32_t L) {
    return 1024 + (size_t)3 * KB * KB_BYTES + (size_t)L * TC_M * 8 + 32 * TC_M * 4;
}

void launch_prep_tc(const double* X64, const uint32_t* A, uint64_t N, uint32_t n, const double* g,
                    double inv_S, uint32_t row_halfs, __half* Bh, cudaStream_t s) {
    k_prep_tc<<<2368, 256, 0, s>>>(X64, A, N, n, g, inv_S, row_halfs, Bh);
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

template <int KB>
static void launch_tc_kb(const TcJoinArgs& a, uint64_t nitems, uint64_t N, cudaStream_t s) {
    CUtensorMap map;
    cuuint64_t dims[2] = {(cuuint64_t)a.row_halfs, (cuuint64_t)N};
    cuuint64_t strides[1] = {(cuuint64_t)a.row_halfs * 2};
    cuuint32_t box[2] = {KBLK, TC_N};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = get_encode()(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, (void*)a.Bh, dims, strides,
                              box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                              CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw Error(9, "cuTensorMapEncodeTiled failed: " + std::to_string((int)r));
    const size_t sm = tc_join_smem_bytes(KB, a.L);
    KJ_CUDA(cudaFuncSetAttribute(k_join_tc<KB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    for (uint64_t off = 0; off < nitems; off += 2147483647ull) {
        const uint64_t cnt = std::min<uint64_t>(nitems - off, 2147483647ull);
        TcJoinArgs b = a;
        b.items = a.items + off;
        k_join_tc<KB><<<(unsigned)cnt, TC_M, sm, s>>>(map, b);
    }
    KJ_CUDA(cudaGetLastError());
    g_launches.fetch_add(1, std::memory_order_relaxed);
}

void launch_join_tc(const TcJoinArgs& a, uint64_t nitems, uint64_t N, cudaStream_t s) {
    if (!nitems) return;
    const int KB = (int)(a.row_halfs / KBLK);
    if (KB == 1) launch_tc_kb<1>(a, nitems, N, s);
    else if (KB == 2) launch_tc_kb<2>(a, nitems, N, s);
    else throw Error(1, "tensor-core join supports up to 42 dimensions");
}

}  // namespace kj
