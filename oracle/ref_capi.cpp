// TEST INFRASTRUCTURE ONLY — never linked into the product library.
//
// Thin extern "C" wrapper over the UNMODIFIED reference library, compiled from
// the sources where they lie under /root/reference/proj (see oracle/Makefile).
// The result is oracle/_ref/libknnjoin_ref.so, used for three things only:
//   * generating the golden fixtures in tests/golden/ (tests/golden/make_golden.py),
//   * cross-checking the C restatement (oracle/knnj_oracle.c) in tests/,
//   * the CPU "reference" arm of bench.py (`--impl reference`, cpu_baseline).
// Every function calls straight into the reference's public API; no algorithm
// lives here.
#include <cmath>
#include <cstdint>
#include <cstring>
#include <exception>
#include <memory>
#include <string>
#include <vector>

#include "knnjoin/dataset.hpp"
#include "knnjoin/dense_engine.hpp"
#include "knnjoin/epsilon.hpp"
#include "knnjoin/errors.hpp"
#include "knnjoin/grid_index.hpp"
#include "knnjoin/io.hpp"
#include "knnjoin/kdtree.hpp"
#include "knnjoin/kernels.hpp"
#include "knnjoin/orchestrator.hpp"
#include "knnjoin/partition.hpp"
#include "knnjoin/sparse_engine.hpp"
#include "knnjoin/synthetic.hpp"
#include "knnjoin/util.hpp"

using namespace knnjoin;

namespace {

thread_local std::string g_err;

int code_of(const std::exception& e) {
    if (dynamic_cast<const UsageError*>(&e)) return 1;
    if (dynamic_cast<const IngestError*>(&e)) return 2;
    if (dynamic_cast<const IndexingError*>(&e)) return 3;
    if (dynamic_cast<const DegenerateProfileError*>(&e)) return 4;
    if (dynamic_cast<const TargetUnreachableError*>(&e)) return 5;
    if (dynamic_cast<const BatchOverflowError*>(&e)) return 6;
    if (dynamic_cast<const SampleTooSmallError*>(&e)) return 7;
    if (dynamic_cast<const OracleCapError*>(&e)) return 8;
    return 9;
}

template <class F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return code_of(e);
    }
}

Dataset make_ds(const double* X, uint64_t N, uint32_t n) {
    return Dataset(std::vector<double>(X, X + N * n), n);
}

}  // namespace

extern "C" {

struct ref_cfg {
    uint32_t k, m;
    double beta, gamma, rho;
    uint32_t mode;  // 0 hybrid 1 sparse 2 dense 3 oracle
    uint32_t workers;
    uint64_t seed;
    uint32_t n_bins;
    double hist_frac, batch_frac;
    uint64_t buffer_size, eps_mean_cap;
    uint32_t policy_dynamic;
    uint64_t policy_count;
    const uint32_t* subset;
    uint64_t n_subset;
    uint64_t force_n_batches;  // 0 = estimate
};

struct ref_info {
    uint64_t n_queries;
    uint32_t k_eff, m_used;
    double eps_used, eps_mean, eps_default, eps_beta, bin_width;
    uint64_t hist_query_count;
    uint64_t q_gpu, q_cpu, demoted, failed_count;
    double n_min, n_thresh;
    uint32_t eps_fallback, has_profile;
    uint64_t candidates_examined, estimate_e, n_batches;
    double t_reorder, t_eps, t_grid, t_kd, t_split, t_dense, t_sparse, t_reassign, t_merge,
        measured_total;
    uint32_t perm[1024];
};

const char* ref_last_error() { return g_err.c_str(); }

// ingest_dataset (io.cpp:99-106) into a caller buffer: sizes always, coordinates when
// `cap` is large enough (used by tests/golden/make_ingest_golden.py)
int ref_ingest(const char* path, const char* fmt, double* out, uint64_t cap, uint64_t* N,
               uint64_t* n) {
    return guarded([&] {
        Dataset d = ingest_dataset(path, format_from_string(fmt));
        *N = d.size();
        *n = d.dims();
        if (out && cap >= d.raw().size()) std::memcpy(out, d.raw().data(), 8 * d.raw().size());
    });
}


int ref_set_kernel(const char* name) { return kernels::set_active_kernel(name) ? 0 : 1; }

double ref_sq_dist_limited(const double* a, const double* b, uint64_t n, double limit) {
    return kernels::sq_dist_limited(a, b, n, limit);
}

int ref_generate(const char* spec, uint64_t size, uint32_t dims, uint64_t seed, double* out) {
    return guarded([&] {
        Dataset d = generate_synthetic(SyntheticSpec::parse(spec), size, dims, seed);
        std::memcpy(out, d.raw().data(), d.raw().size() * sizeof(double));
    });
}

// Full run_hybrid. Outputs are sized by the caller: ids/dist [n_queries*k],
// counts [n_queries] (neighbours per query), prov [n_queries], qids [n_queries],
// hist_counts/hist_cum [n_bins].
int ref_run(const double* X, uint64_t N, uint32_t n, const ref_cfg* c, uint32_t* qids,
            uint32_t* ids, double* dist, uint32_t* counts, uint8_t* prov, double* hist_counts,
            double* hist_cum, ref_info* info) {
    return guarded([&] {
        Dataset d = make_ds(X, N, n);
        RunConfig cfg;
        cfg.k = c->k;
        cfg.m = c->m;
        cfg.beta = c->beta;
        cfg.gamma = c->gamma;
        cfg.rho = c->rho;
        cfg.mode = EngineMode(c->mode);
        cfg.workers = c->workers;
        cfg.seed = c->seed;
        cfg.n_bins = c->n_bins;
        cfg.hist_query_fraction = c->hist_frac;
        cfg.batch_sample_fraction = c->batch_frac;
        cfg.buffer_size = c->buffer_size;
        cfg.eps_mean_pair_cap = c->eps_mean_cap;
        cfg.policy = c->policy_dynamic ? GranularityPolicy::tdynamic(c->policy_count)
                                       : GranularityPolicy::tstatic(c->policy_count);
        if (c->subset) cfg.query_subset = std::vector<PointId>(c->subset, c->subset + c->n_subset);
        if (c->force_n_batches) cfg.force_n_batches = c->force_n_batches;

        KnnRunResult r = run_hybrid(d, cfg);
        std::memset(info, 0, sizeof(*info));
        info->n_queries = r.queries.size();
        info->k_eff = uint32_t(r.k_effective);
        info->m_used = uint32_t(r.m_used);
        info->eps_used = r.eps_used;
        if (r.profile) {
            info->has_profile = 1;
            info->eps_mean = r.profile->eps_mean;
            info->eps_default = r.profile->eps_default;
            info->eps_beta = r.profile->eps_beta;
            info->bin_width = r.profile->bin_width;
            info->hist_query_count = r.profile->query_count;
            for (std::size_t b = 0; b < r.profile->counts.size(); ++b) {
                if (hist_counts) hist_counts[b] = r.profile->counts[b];
                if (hist_cum) hist_cum[b] = r.profile->cumulative[b];
            }
        }
        if (r.partition) {
            info->q_gpu = r.partition->q_gpu;
            info->q_cpu = r.partition->q_cpu;
            info->n_min = r.partition->n_min;
            info->n_thresh = r.partition->n_thresh;
            info->demoted = r.partition->demoted;
        }
        info->failed_count = r.failed_count;
        info->eps_fallback = r.eps_fallback;
        if (r.dense_stats) {
            info->candidates_examined = r.dense_stats->candidates_examined;
            info->estimate_e = r.dense_stats->estimate_e;
            info->n_batches = r.dense_stats->batch_pair_counts.size();
        }
        info->t_reorder = r.timings.reorder;
        info->t_eps = r.timings.eps_select;
        info->t_grid = r.timings.grid_build;
        info->t_kd = r.timings.kd_build;
        info->t_split = r.timings.split;
        info->t_dense = r.timings.dense;
        info->t_sparse = r.timings.sparse;
        info->t_reassign = r.timings.reassign;
        info->t_merge = r.timings.merge;
        info->measured_total = r.timings.measured_total;
        const auto& perm = r.working->dim_permutation();
        for (std::size_t j = 0; j < perm.size() && j < 1024; ++j) info->perm[j] = perm[j];
        const std::size_t k = c->k;
        for (std::size_t i = 0; i < r.queries.size(); ++i) {
            qids[i] = r.queries[i];
            counts[i] = uint32_t(r.neighbors[i].size());
            prov[i] = uint8_t(r.provenance[i]);
            for (std::size_t j = 0; j < r.neighbors[i].size(); ++j) {
                ids[i * k + j] = r.neighbors[i][j].id;
                dist[i * k + j] = r.neighbors[i][j].dist;
            }
        }
    });
}

int ref_tsv(const double* X, uint64_t N, uint32_t n, const ref_cfg* c, char* out,
            uint64_t cap, uint64_t* len) {
    return guarded([&] {
        Dataset d = make_ds(X, N, n);
        RunConfig cfg;
        cfg.k = c->k;
        cfg.m = c->m;
        cfg.beta = c->beta;
        cfg.gamma = c->gamma;
        cfg.rho = c->rho;
        cfg.mode = EngineMode(c->mode);
        cfg.workers = c->workers;
        cfg.seed = c->seed;
        cfg.n_bins = c->n_bins;
        cfg.hist_query_fraction = c->hist_frac;
        cfg.batch_sample_fraction = c->batch_frac;
        cfg.buffer_size = c->buffer_size;
        cfg.eps_mean_pair_cap = c->eps_mean_cap;
        std::string s = tsv_string(run_hybrid(d, cfg));
        *len = s.size();
        if (out && cap >= s.size()) std::memcpy(out, s.data(), s.size());
    });
}

int ref_variance_order(const double* X, uint64_t N, uint32_t n, uint32_t m, uint32_t* perm,
                       double* var) {
    return guarded([&] {
        Dataset d = make_ds(X, N, n);
        auto v = d.column_variances();
        Dataset w = reorder_by_variance(d, m);
        for (uint32_t j = 0; j < n; ++j) {
            perm[j] = w.dim_permutation()[j];
            if (var) var[j] = v[j];
        }
    });
}

int ref_eps_mean(const double* X, uint64_t N, uint32_t n, uint64_t pairs, uint64_t seed,
                 double* out) {
    return guarded([&] { *out = estimate_eps_mean(make_ds(X, N, n), pairs, seed); });
}

int ref_histogram(const double* X, uint64_t N, uint32_t n, double eps_mean, uint32_t n_bins,
                  double frac, uint64_t seed, uint32_t threads, double* counts, double* cum,
                  uint64_t* qcount) {
    return guarded([&] {
        EpsilonProfile p =
            build_distance_histogram(make_ds(X, N, n), eps_mean, n_bins, frac, seed, threads);
        for (uint32_t b = 0; b < n_bins; ++b) {
            counts[b] = p.counts[b];
            cum[b] = p.cumulative[b];
        }
        *qcount = p.query_count;
    });
}

int ref_select_eps(const double* cum, uint32_t n_bins, double bin_width, uint32_t k, double beta,
                   double* eps_beta, double* eps_final, uint64_t* bin, double* achievable) {
    return guarded([&] {
        EpsilonProfile p;
        p.n_bins = n_bins;
        p.bin_width = bin_width;
        p.cumulative.assign(cum, cum + n_bins);
        p.counts.assign(n_bins, 0.0);
        try {
            auto s = select_eps_beta(p, k, beta);
            *eps_beta = s.eps_beta;
            *eps_final = s.eps_final;
            *bin = s.bin;
        } catch (const TargetUnreachableError& e) {
            *achievable = e.achievable_max;
            throw;
        }
    });
}

int ref_sample(uint64_t n, uint64_t k, uint64_t seed, uint64_t* out) {
    return guarded([&] {
        std::mt19937_64 rng(seed);
        auto v = sample_without_replacement(n, k, rng);
        std::memcpy(out, v.data(), v.size() * sizeof(uint64_t));
    });
}

uint64_t ref_derive_seed(uint64_t master, uint64_t tag) { return derive_seed(master, tag); }

// Grid: first call with B == nullptr returns the cell count.
int ref_grid(const double* X, uint64_t N, uint32_t n, uint32_t m, double eps, uint64_t* ncells,
             uint64_t* B, uint64_t* G, uint32_t* A, uint64_t* cpd, double* mins, double* maxs) {
    return guarded([&] {
        Dataset d = make_ds(X, N, n);
        GridIndex g = GridIndex::build(d, m, eps);
        *ncells = g.nonempty_cell_ids().size();
        if (!B) return;
        for (std::size_t i = 0; i < g.nonempty_cell_ids().size(); ++i) {
            B[i] = g.nonempty_cell_ids()[i];
            G[2 * i] = g.cell_ranges()[i].first;
            G[2 * i + 1] = g.cell_ranges()[i].second;
        }
        for (std::size_t i = 0; i < N; ++i) A[i] = g.point_lookup()[i];
        for (uint32_t j = 0; j < m; ++j) {
            cpd[j] = g.cells_per_dim()[j];
            mins[j] = g.mins()[j];
            maxs[j] = g.maxs()[j];
        }
    });
}

// Per query: number of candidates examined and in-eps results (self included).
int ref_range_counts(const double* X, uint64_t N, uint32_t n, uint32_t m, double eps,
                     const uint32_t* q, uint64_t nq, uint64_t* cand, uint64_t* in_eps) {
    return guarded([&] {
        Dataset d = make_ds(X, N, n);
        GridIndex g = GridIndex::build(d, m, eps);
        for (uint64_t i = 0; i < nq; ++i) {
            RangeQueryStats st;
            in_eps[i] = g.range_query(q[i], eps, &st).size();
            cand[i] = st.candidates_examined;
        }
    });
}

int ref_split(const double* X, uint64_t N, uint32_t n, uint32_t m, double eps, uint32_t k,
              double beta, double gamma, double rho, const uint32_t* q, uint64_t nq,
              uint8_t* is_dense, uint64_t* pop, double* n_min, double* n_thresh,
              uint64_t* demoted) {
    return guarded([&] {
        Dataset d = make_ds(X, N, n);
        GridIndex g = GridIndex::build(d, m, eps);
        WorkPartition p = split_work(g, k, {beta, gamma, rho}, std::span<const PointId>(q, nq));
        std::vector<uint8_t> dense(N, 0);
        for (PointId x : p.q_gpu) dense[x] = 1;
        for (uint64_t i = 0; i < nq; ++i) {
            is_dense[i] = dense[q[i]];
            pop[i] = p.cell_population[i];
        }
        *n_min = p.n_min;
        *n_thresh = p.n_thresh;
        *demoted = p.demoted_count;
    });
}

// Dense join over the given queries with a pinned batch count; per query the
// solved flag and, when solved, its k neighbours.
int ref_dense_join(const double* X, uint64_t N, uint32_t n, uint32_t m, double eps, uint32_t k,
                   const uint32_t* q, uint64_t nq, uint32_t threads, uint8_t* solved,
                   uint32_t* ids, double* dist, uint64_t* candidates) {
    return guarded([&] {
        Dataset d = make_ds(X, N, n);
        GridIndex g = GridIndex::build(d, m, eps);
        std::span<const PointId> qs(q, nq);
        BatchPlan plan = plan_with_batches(qs, 3, ~uint64_t(0) >> 1);
        DenseJoinResult r =
            run_dense_join(g, qs, eps, k, GranularityPolicy::tstatic(8), plan, threads);
        std::vector<int64_t> pos(N, -1);
        for (uint64_t i = 0; i < nq; ++i) pos[q[i]] = int64_t(i);
        for (uint64_t i = 0; i < nq; ++i) solved[i] = 0;
        for (const auto& qn : r.solved) {
            int64_t i = pos[qn.id];
            solved[i] = 1;
            for (std::size_t j = 0; j < qn.neighbors.size(); ++j) {
                ids[i * k + j] = qn.neighbors[j].id;
                dist[i * k + j] = qn.neighbors[j].dist;
            }
        }
        *candidates = r.stats.candidates_examined;
    });
}

int ref_brute_knn(const double* X, uint64_t N, uint32_t n, const uint32_t* q, uint64_t nq,
                  uint32_t k, uint32_t threads, uint32_t* ids, double* dist) {
    return guarded([&] {
        Dataset d = make_ds(X, N, n);
        auto r = brute_force_knn(d, std::span<const PointId>(q, nq), k, threads);
        for (uint64_t i = 0; i < nq; ++i)
            for (std::size_t j = 0; j < r[i].size(); ++j) {
                ids[i * k + j] = r[i][j].id;
                dist[i * k + j] = r[i][j].dist;
            }
    });
}

// kd-tree (the paper's RefImpl / SparseOnly engine) on an already-reordered
// dataset: build excluded from *seconds, as in the reference's measured_total.
int ref_sparse_knn(const double* X, uint64_t N, uint32_t n, const uint32_t* q, uint64_t nq,
                   uint32_t k, uint32_t threads, uint32_t* ids, double* dist, double* seconds) {
    return guarded([&] {
        Dataset d = make_ds(X, N, n);
        KdTree t = KdTree::build(d, 16);
        Stopwatch sw;
        SparseRunResult r = run_sparse_knn(t, std::span<const PointId>(q, nq), k, threads);
        *seconds = sw.seconds();
        for (uint64_t i = 0; i < nq; ++i)
            for (std::size_t j = 0; j < r.neighbors[i].size(); ++j) {
                ids[i * k + j] = r.neighbors[i][j].id;
                dist[i * k + j] = r.neighbors[i][j].dist;
            }
    });
}

unsigned ref_hardware_concurrency() { return default_worker_count(); }

// Persistent RefImpl (SparseOnly) state for timing: the reference's
// reorder_by_variance + KdTree::build once, then run_sparse_knn on query
// samples (orchestrator.cpp:114-129; build excluded like measured_total).
struct RefKd {
    std::unique_ptr<Dataset> d;
    std::unique_ptr<KdTree> t;
};

void* ref_kd_create(const double* X, uint64_t N, uint32_t n, uint32_t m, double* t_reorder,
                    double* t_build) {
    try {
        auto h = new RefKd;
        Dataset raw = make_ds(X, N, n);
        Stopwatch a;
        h->d = std::make_unique<Dataset>(reorder_by_variance(raw, m));
        *t_reorder = a.seconds();
        Stopwatch b;
        h->t = std::make_unique<KdTree>(KdTree::build(*h->d, 16));
        *t_build = b.seconds();
        return h;
    } catch (const std::exception& e) {
        g_err = e.what();
        return nullptr;
    }
}

int ref_kd_query(void* hp, const uint32_t* q, uint64_t nq, uint32_t k, uint32_t threads,
                 uint32_t* ids, double* dist, double* seconds) {
    return guarded([&] {
        auto* h = static_cast<RefKd*>(hp);
        SparseRunResult r = run_sparse_knn(*h->t, std::span<const PointId>(q, nq), k, threads);
        *seconds = r.t1_seconds * double(nq);
        for (uint64_t i = 0; i < nq; ++i)
            for (std::size_t j = 0; j < r.neighbors[i].size(); ++j) {
                if (ids) ids[i * k + j] = r.neighbors[i][j].id;
                if (dist) dist[i * k + j] = r.neighbors[i][j].dist;
            }
    });
}

void ref_kd_destroy(void* hp) { delete static_cast<RefKd*>(hp); }

}  // extern "C"
