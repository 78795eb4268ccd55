/* TEST INFRASTRUCTURE ONLY — the CPU oracle for the KNN self-join hot path.
 *
 * A plain-C restatement of the reference algorithm (arXiv 1810.04758,
 * /root/reference/proj), used exclusively by tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline leg as the CHECKER. The product library
 * (paper_1810_04758_b200/libknnj_b200.so) never links or calls it.
 *
 * Pinned against: the reference's own known-answer tests (see
 * tests/test_oracle_golden.py) and the outputs of the unmodified reference
 * compiled by oracle/Makefile (the tests/golden fixtures made by
 * tests/golden/make_golden.py). Every function cites the reference file:line
 * it restates.
 */
#ifndef KNNJ_ORACLE_H
#define KNNJ_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* proj/src/kernels_scalar.cpp:9-27 */
double orc_sq_dist_limited(const double* a, const double* b, size_t n, double limit_sq);

/* std::mt19937_64 (fully specified by [rand.eng.mers]) */
typedef struct {
    uint64_t mt[312];
    int mti;
} orc_mt64;
void orc_mt_seed(orc_mt64* s, uint64_t seed);
uint64_t orc_mt_next(orc_mt64* s);
/* libstdc++ 13 uniform_int_distribution<uint64_t>{a,b}(mt19937_64) (Lemire, bits/uniform_int_dist.h) */
uint64_t orc_uniform_u64(orc_mt64* s, uint64_t a, uint64_t b);
/* proj/include/knnjoin/util.hpp:15-30 */
uint64_t orc_derive_seed(uint64_t master, uint64_t tag);
/* proj/include/knnjoin/util.hpp:70-92; out ascending, returns count */
uint64_t orc_sample_without_replacement(uint64_t n, uint64_t k, orc_mt64* rng, uint64_t* out);

/* proj/src/dataset.cpp:58-111: variances and the descending-variance order */
void orc_variance_order(const double* X, uint64_t N, uint32_t n, uint32_t* order, double* var);
void orc_permute_columns(const double* X, uint64_t N, uint32_t n, const uint32_t* order,
                         double* out);

/* proj/src/epsilon.cpp:14-44 */
int orc_eps_mean(const double* X, uint64_t N, uint32_t n, uint64_t pairs, uint64_t seed,
                 double* out);
/* proj/src/epsilon.cpp:46-120: raw integer bin counts (before normalisation) */
int orc_histogram(const double* X, uint64_t N, uint32_t n, double eps_mean, uint32_t n_bins,
                  double frac, uint64_t seed, uint32_t threads, uint64_t* raw,
                  uint64_t* query_count);
/* proj/src/epsilon.cpp:122-141 and orchestrator.cpp:49-63 (fallback) */
int orc_histogram_queries(const double* X, uint64_t N, uint32_t n, double eps_mean,
                          uint32_t n_bins, const uint64_t* queries, uint64_t nq,
                          uint32_t threads, uint64_t* raw);
int orc_select_eps(const double* cum, uint32_t n_bins, double bin_width, uint32_t k, double beta,
                   int allow_fallback, double* eps_beta, double* eps_final, uint64_t* bin,
                   int* fell_back);

/* proj/src/grid_index.cpp:13-75 */
typedef struct {
    uint32_t m;
    double eps;
    double mins[64], maxs[64];
    uint64_t cpd[64], strides[64];
    uint64_t ncells;
    uint64_t* B;    /* ncells */
    uint64_t* G;    /* 2*ncells: begin,end */
    uint32_t* A;    /* N */
    uint32_t* slot; /* N */
} orc_grid;
int orc_grid_build(const double* X, uint64_t N, uint32_t n, uint32_t m, double eps, orc_grid* g,
                   char* err, size_t errlen);
void orc_grid_free(orc_grid* g);

/* proj/src/partition.cpp:12-75 */
double orc_n_min(uint32_t k, uint32_t m);
double orc_n_thresh(double n_min, double gamma);

enum { ORC_HYBRID = 0, ORC_SPARSE = 1, ORC_DENSE = 2, ORC_ORACLE = 3 };

typedef struct {
    uint32_t k, m, mode, threads, n_bins;
    double beta, gamma, rho, hist_frac;
    uint64_t seed, eps_mean_cap;
} orc_cfg;

typedef struct {
    uint32_t k_eff, m_used, eps_fallback;
    double eps_mean, bin_width, eps_default, eps_beta, eps_used, n_min, n_thresh;
    uint64_t hist_query_count, q_gpu, q_cpu, demoted, failed_count, candidates_examined;
    uint32_t perm[1024];
} orc_info;

/* proj/src/orchestrator.cpp:67-250 (run_hybrid). Queries are all points, in id order.
 * ids/dist: N*k_eff (k_eff neighbours per query, stride k_eff). prov: 0 dense, 1 sparse,
 * 2 dense-failed-then-sparse. raw_hist: n_bins (may be NULL). The sparse engine's
 * kd-tree and the brute oracle both return the exact (sq,id)-ordered KNN; the
 * restatement computes that by brute force (proj/src/dense_engine.cpp:322-346). */
int orc_run(const double* X, uint64_t N, uint32_t n, const orc_cfg* cfg, uint32_t* ids,
            double* dist, uint8_t* prov, uint64_t* raw_hist, orc_info* info, char* err,
            size_t errlen);

/* proj/src/dense_engine.cpp:322-346 over an already-reordered dataset */
int orc_brute_knn(const double* X, uint64_t N, uint32_t n, const uint32_t* q, uint64_t nq,
                  uint32_t k, uint32_t threads, uint32_t* ids, double* dist);

#ifdef __cplusplus
}
#endif
#endif
