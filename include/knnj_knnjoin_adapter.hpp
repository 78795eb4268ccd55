// knnj_knnjoin_adapter.hpp — drop-in for the reference's run_hybrid on the B200 engine.
//
// Header-only C++ adapter a maintainer of the reference library adds to its tree
// (it includes the reference's own headers, proj/include/knnjoin/*.hpp) to route
// knnjoin::run_hybrid (proj/include/knnjoin/orchestrator.hpp:95,
// proj/src/orchestrator.cpp:67-250) through libknnj_b200.so's C ABI (knnj_c.h).
// Same inputs (Dataset, RunConfig), same KnnRunResult fields, same exception
// types; see INTEGRATION.md for the build line.
//
// What maps where:
//   RunConfig.k/m/beta/gamma/rho/mode/n_bins/hist_query_fraction/
//   eps_mean_pair_cap/seed/query_subset        -> knnj_config (same meaning)
//   RunConfig.policy/buffer_size/batch_sample_fraction/force_n_batches/workers/
//   kd_bucket_capacity/duplicate_kd_index      -> no device analogue (the fused join
//                                                 has no pair buffer and no batches;
//                                                 results never depended on them,
//                                                 acceptance C6/C9)
//   KnnRunResult.neighbors/provenance/queries/k_effective/eps_used/m_used/
//   failed_count/eps_fallback/profile/partition/dense_stats.candidates_examined
//                                               <- knnj_run outputs
//   KnnRunResult.t1/t2/rho_model/sparse_worker_counts: CPU load-balance model,
//                                                 left empty (no CPU engine runs)
#pragma once

#include <algorithm>
#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <memory>
#include <span>
#include <string>
#include <utility>
#include <vector>

#include "knnj_c.h"
#include "knnjoin/dataset.hpp"
#include "knnjoin/errors.hpp"
#include "knnjoin/orchestrator.hpp"
#include "knnjoin/util.hpp"

namespace knnjoin_b200 {

// knnj_status -> the reference exception type (proj/include/knnjoin/errors.hpp:11-62)
[[noreturn]] inline void rethrow(int rc, const std::string& msg) {
    switch (rc) {
        case KNNJ_E_USAGE: throw knnjoin::UsageError(msg);
        case KNNJ_E_INGEST: throw knnjoin::IngestError(msg);
        case KNNJ_E_INDEXING: throw knnjoin::IndexingError(msg);
        case KNNJ_E_DEGENERATE: throw knnjoin::DegenerateProfileError(msg);
        case KNNJ_E_TARGET_UNREACHABLE: throw knnjoin::TargetUnreachableError(msg, 0.0);
        case KNNJ_E_BATCH_OVERFLOW: throw knnjoin::BatchOverflowError(msg, 0);
        case KNNJ_E_SAMPLE_TOO_SMALL: throw knnjoin::SampleTooSmallError(msg);
        case KNNJ_E_ORACLE_CAP: throw knnjoin::OracleCapError(msg);
        default: throw std::runtime_error("knnj: " + msg);
    }
}

// One device context (RAII over knnj_create / knnj_destroy).
class Engine {
public:
    explicit Engine(int device = 0) {
        const int rc = knnj_create(device, &ctx_);
        if (rc) rethrow(rc, "cannot create a context on device " + std::to_string(device));
    }
    ~Engine() { knnj_destroy(ctx_); }
    Engine(const Engine&) = delete;
    Engine& operator=(const Engine&) = delete;
    knnj_ctx* get() const { return ctx_; }
    void check(int rc) const {
        if (rc) rethrow(rc, knnj_last_error(ctx_));
    }

private:
    knnj_ctx* ctx_ = nullptr;
};

// knnjoin::run_hybrid with the hot path on the GPU (semantics of
// proj/src/orchestrator.cpp:67-250; outputs bit-identical to the reference run
// with kernel "scalar").
inline knnjoin::KnnRunResult run_hybrid(Engine& eng, const knnjoin::Dataset& d,
                                        const knnjoin::RunConfig& cfg) {
    knnj_ctx* ctx = eng.get();
    eng.check(knnj_set_points(ctx, d.raw().data(), d.size(), (uint32_t)d.dims()));
    knnj_config c{};
    c.k = (uint32_t)cfg.k;
    c.m = (uint32_t)cfg.m;
    c.beta = cfg.beta;
    c.gamma = cfg.gamma;
    c.rho = cfg.rho;
    switch (cfg.mode) {
        case knnjoin::EngineMode::Hybrid: c.mode = KNNJ_HYBRID; break;
        case knnjoin::EngineMode::SparseOnly: c.mode = KNNJ_SPARSE_ONLY; break;
        case knnjoin::EngineMode::DenseOnly: c.mode = KNNJ_DENSE_ONLY; break;
        case knnjoin::EngineMode::BruteOracle: c.mode = KNNJ_BRUTE_ORACLE; break;
    }
    c.n_bins = (uint32_t)cfg.n_bins;
    c.hist_query_fraction = cfg.hist_query_fraction;
    c.eps_mean_pair_cap = cfg.eps_mean_pair_cap;
    c.seed = cfg.seed;
    if (cfg.query_subset) {
        c.query_subset = cfg.query_subset->data();
        c.n_query_subset = cfg.query_subset->size();
    }
    std::vector<knnjoin::PointId> queries;
    if (cfg.query_subset) {
        queries = *cfg.query_subset;
        std::sort(queries.begin(), queries.end());
        queries.erase(std::unique(queries.begin(), queries.end()), queries.end());
    } else {
        queries.resize(d.size());
        for (std::size_t i = 0; i < d.size(); ++i) queries[i] = (knnjoin::PointId)i;
    }
    const std::size_t nq = queries.size();
    const std::size_t k_cap = std::min<std::size_t>(cfg.k, d.size() ? d.size() - 1 : 0);
    std::vector<uint32_t> ids(nq * k_cap);
    std::vector<double> dist(nq * k_cap);
    std::vector<uint8_t> prov(nq);
    std::vector<uint64_t> raw(cfg.n_bins);
    const bool profiled = cfg.mode == knnjoin::EngineMode::Hybrid ||
                          cfg.mode == knnjoin::EngineMode::DenseOnly;
    auto info = std::make_unique<knnj_run_info>();
    eng.check(knnj_run(ctx, &c, ids.data(), dist.data(), prov.data(),
                       profiled ? raw.data() : nullptr, info.get()));

    knnjoin::KnnRunResult r;
    r.queries = queries;
    r.k_effective = info->k_effective;
    r.neighbors.resize(nq);
    r.provenance.resize(nq);
    for (std::size_t i = 0; i < nq; ++i) {
        auto& row = r.neighbors[i];
        row.resize(info->k_effective);
        for (uint32_t j = 0; j < info->k_effective; ++j)
            row[j] = knnjoin::Neighbor{ids[i * info->k_effective + j], dist[i * info->k_effective + j]};
        r.provenance[i] = static_cast<knnjoin::Provenance>(prov[i]);
    }
    // working (variance-reordered) dataset, as the reference keeps it
    std::vector<double> w(d.size() * d.dims());
    eng.check(knnj_get_points(ctx, w.data()));
    std::vector<uint32_t> perm(info->perm, info->perm + d.dims());
    r.working = std::make_shared<const knnjoin::Dataset>(std::move(w), d.dims(), std::move(perm));
    r.mode = cfg.mode;
    r.m_used = info->m_used;
    r.eps_used = info->eps_used;
    r.failed_count = info->failed_count;
    r.eps_fallback = info->eps_fallback != 0;
    if (info->k_clamped)
        r.warnings.push_back("k clamped to |D|-1 = " + std::to_string(info->k_effective));
    if (info->eps_fallback)
        r.warnings.push_back("beta target unreachable within eps_mean; clamped to the histogram maximum");
    // k_eff == 0 (|D| == 1): the reference returns before eps selection and the split
    // (orchestrator.cpp:94-97), so there is no profile, partition or dense stats
    if (profiled && info->k_effective > 0) {
        knnjoin::EpsilonProfile p;
        p.eps_mean = info->eps_mean;
        p.n_bins = cfg.n_bins;
        p.bin_width = info->bin_width;
        p.sample_fraction = cfg.hist_query_fraction;
        p.query_count = info->hist_query_count;
        p.seed = knnjoin::derive_seed(cfg.seed, knnjoin::kSeedHistogram);  // the histogram sub-stream
        p.counts.resize(cfg.n_bins);
        p.cumulative.resize(cfg.n_bins);
        uint64_t run = 0;
        for (std::size_t b = 0; b < cfg.n_bins; ++b) {
            run += raw[b];
            p.counts[b] = double(raw[b]) / double(info->hist_query_count);
            p.cumulative[b] = double(run) / double(info->hist_query_count);
        }
        p.eps_default = info->eps_default;
        p.beta = cfg.beta;
        p.eps_beta = info->eps_beta;
        p.eps_final = info->eps_final;
        r.profile = std::move(p);
        knnjoin::PartitionSummary ps;
        ps.q_gpu = info->q_gpu;
        ps.q_cpu = info->q_cpu;
        ps.n_min = info->n_min;
        ps.n_thresh = info->n_thresh;
        ps.demoted = info->demoted;
        r.partition = ps;
        knnjoin::DenseJoinStats st;
        st.candidates_examined = info->candidates_examined;
        st.kernel_seconds = info->ms_join_kernel * 1e-3;
        r.dense_stats = std::move(st);
    }
    r.timings.reorder = info->ms_reorder * 1e-3;
    r.timings.eps_select = (info->ms_eps_mean + info->ms_histogram) * 1e-3;
    r.timings.grid_build = info->ms_grid * 1e-3;
    r.timings.split = info->ms_split * 1e-3;
    r.timings.dense = info->ms_join * 1e-3;
    r.timings.reassign = info->ms_fallback * 1e-3;
    r.timings.measured_total = info->ms_total * 1e-3;
    return r;
}

// knnjoin::parameter_search (proj/include/knnjoin/orchestrator.hpp:116-118,
// proj/src/orchestrator.cpp:252-303) on the GPU: the same seeded query subset and
// candidate runs (hybrid, rho = 0.5); wall_seconds is the device run time. t1/t2/
// rho_model (the CPU load-balance model) stay empty.
inline knnjoin::ParameterSearchResult parameter_search(
    Engine& eng, const knnjoin::Dataset& d, std::size_t k, double f,
    std::span<const std::pair<double, double>> candidates, const knnjoin::RunConfig& base) {
    knnj_ctx* ctx = eng.get();
    eng.check(knnj_set_points(ctx, d.raw().data(), d.size(), (uint32_t)d.dims()));
    knnj_config c{};
    c.k = (uint32_t)k;
    c.m = (uint32_t)base.m;
    c.beta = base.beta;
    c.gamma = base.gamma;
    c.rho = base.rho;
    c.mode = KNNJ_HYBRID;
    c.n_bins = (uint32_t)base.n_bins;
    c.hist_query_fraction = base.hist_query_fraction;
    c.eps_mean_pair_cap = base.eps_mean_pair_cap;
    c.seed = base.seed;
    std::vector<double> betas, gammas;
    for (const auto& [b, g] : candidates) {
        betas.push_back(b);
        gammas.push_back(g);
    }
    std::vector<knnj_search_row> rows(std::max<std::size_t>(1, candidates.size()));
    double bb = 0.0, bg = 0.0;
    eng.check(knnj_parameter_search(ctx, &c, f, betas.data(), gammas.data(), candidates.size(),
                                    rows.data(), &bb, &bg));
    knnjoin::ParameterSearchResult out;
    out.best_beta = bb;
    out.best_gamma = bg;
    for (std::size_t i = 0; i < candidates.size(); ++i) {
        knnjoin::CandidateOutcome o;
        o.beta = rows[i].beta;
        o.gamma = rows[i].gamma;
        o.wall_seconds = rows[i].wall_seconds;
        o.error = rows[i].error;
        out.candidates.push_back(std::move(o));
    }
    return out;
}

}  // namespace knnjoin_b200
