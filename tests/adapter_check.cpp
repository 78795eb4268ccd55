// TEST INFRASTRUCTURE — drop-in check of include/knnj_knnjoin_adapter.hpp.
//
// Links the UNMODIFIED reference library (compiled by path, oracle/Makefile) and
// the B200 engine, then for each case runs the reference's own
// knnjoin::run_hybrid (kernel "scalar") and knnjoin_b200::run_hybrid on the same
// knnjoin::Dataset (drawn by the reference's generate_synthetic) and requires
// byte-identical io::tsv_string output, identical provenance, eps and failed
// counts. Built only where /root/reference exists (oracle/_ref/adapter_check);
// run on the GPU box by tests/test_gpu_adapter.py.
#include <cstdio>
#include <string>
#include <utility>
#include <vector>

#include "knnj_knnjoin_adapter.hpp"
#include "knnjoin/io.hpp"
#include "knnjoin/report.hpp"
#include "knnjoin/kernels.hpp"
#include "knnjoin/synthetic.hpp"

int main() {
    knnjoin::kernels::set_active_kernel("scalar");
    struct Case {
        const char* spec;
        std::size_t size, dims, k, m;
        double beta, gamma, rho;
        knnjoin::EngineMode mode;
    };
    const Case cases[] = {
        {"uniform", 4000, 2, 5, 0, 0.0, 0.0, 0.0, knnjoin::EngineMode::Hybrid},
        {"clusters:16:0.05", 3000, 18, 32, 0, 0.0, 0.0, 0.0, knnjoin::EngineMode::Hybrid},
        {"mixture", 2000, 6, 10, 0, 0.2, 0.5, 0.3, knnjoin::EngineMode::Hybrid},
        {"clusters:4:0.1", 1500, 24, 16, 4, 0.0, 0.0, 0.0, knnjoin::EngineMode::DenseOnly},
        {"mixture", 1200, 90, 8, 0, 0.0, 0.0, 0.0, knnjoin::EngineMode::SparseOnly},
        {"uniform", 900, 3, 7, 0, 0.0, 0.0, 0.0, knnjoin::EngineMode::BruteOracle},
        // k >= |D|: k clamped to |D|-1 with the reference's warning text (orchestrator.cpp:77-82)
        {"uniform", 24, 3, 40, 0, 0.0, 0.0, 0.0, knnjoin::EngineMode::Hybrid},
        {"clusters:2:0.1", 30, 5, 30, 0, 0.0, 0.0, 0.0, knnjoin::EngineMode::DenseOnly},
        // |D| == 1: k_eff = 0, empty lists, Sparse provenance, no profile (orchestrator.cpp:94-97)
        {"uniform", 1, 4, 3, 0, 0.0, 0.0, 0.0, knnjoin::EngineMode::Hybrid},
    };
    knnjoin_b200::Engine eng(0);
    int bad = 0, n = 0;
    for (const Case& c : cases) {
        // (the reference generator needs two points; a one-point dataset is built directly)
        const knnjoin::Dataset d =
            c.size == 1 ? knnjoin::Dataset(std::vector<double>(c.dims, 0.25), c.dims)
                        : knnjoin::generate_synthetic(knnjoin::SyntheticSpec::parse(c.spec), c.size,
                                                      c.dims, 11);
        knnjoin::RunConfig cfg;
        cfg.k = c.k;
        cfg.m = c.m;
        cfg.beta = c.beta;
        cfg.gamma = c.gamma;
        cfg.rho = c.rho;
        cfg.mode = c.mode;
        cfg.seed = 5;
        cfg.buffer_size = 100'000'000;
        const knnjoin::KnnRunResult ref = knnjoin::run_hybrid(d, cfg);
        const knnjoin::KnnRunResult got = knnjoin_b200::run_hybrid(eng, d, cfg);
        const bool tsv = knnjoin::tsv_string(ref) == knnjoin::tsv_string(got);
        const bool prov = ref.provenance == got.provenance;
        const bool meta = ref.eps_used == got.eps_used && ref.failed_count == got.failed_count &&
                          ref.k_effective == got.k_effective && ref.m_used == got.m_used;
        // ε-profile text (epsilon.cpp:149-164) and the run report's deterministic view
        // (report.cpp:18-134). The reference's batch plan and worker round-robin are
        // CPU-engine artefacts with no device analogue: dropped before comparing.
        const bool prof = (!ref.profile && !got.profile) ||
                          (ref.profile && got.profile && ref.profile->to_text() == got.profile->to_text());
        auto view = [&](const knnjoin::KnnRunResult& r) {
            auto j = knnjoin::deterministic_view(knnjoin::make_run_report(d, cfg, r));
            if (j.contains("dense")) {
                j["dense"].erase("n_batches");
                j["dense"].erase("estimate_e");
                j["dense"].erase("batch_pair_counts");
            }
            j.erase("sparse");
            return j.dump();
        };
        const bool rep = view(ref) == view(got);
        const bool ok = tsv && prov && meta && prof && rep;
        std::printf("%s %s |D|=%zu n=%zu k=%zu mode=%s tsv=%d prov=%d meta=%d profile=%d report=%d\n",
                    ok ? "ok " : "BAD", c.spec, c.size, c.dims, c.k, knnjoin::to_string(c.mode), tsv,
                    prov, meta, prof, rep);
        if (!rep) std::printf("  ref: %s\n  got: %s\n", view(ref).c_str(), view(got).c_str());
        if (!prof && ref.profile && got.profile)
            std::printf("  ref profile:\n%.400s\n  got profile:\n%.400s\n", ref.profile->to_text().c_str(),
                        got.profile->to_text().c_str());
        bad += !ok;
        ++n;
    }
    // parameter_search: same candidates (one invalid), same per-candidate errors; the
    // winner is timing-dependent, so it only has to be one of the valid candidates
    {
        const knnjoin::Dataset d =
            knnjoin::generate_synthetic(knnjoin::SyntheticSpec::parse("mixture"), 3000, 6, 13);
        knnjoin::RunConfig base;
        base.seed = 9;
        base.buffer_size = 100'000'000;
        const std::vector<std::pair<double, double>> cands = {{0.0, 0.0}, {0.3, 0.5}, {1.5, 0.0}};
        const auto ref = knnjoin::parameter_search(d, 8, 0.05, cands, base);
        const auto got = knnjoin_b200::parameter_search(eng, d, 8, 0.05, cands, base);
        bool ok = ref.candidates.size() == got.candidates.size();
        for (std::size_t i = 0; ok && i < ref.candidates.size(); ++i) {
            ok = ok && ref.candidates[i].beta == got.candidates[i].beta &&
                 ref.candidates[i].gamma == got.candidates[i].gamma &&
                 ref.candidates[i].error == got.candidates[i].error &&
                 (got.candidates[i].error.empty() == (got.candidates[i].wall_seconds > 0.0));
        }
        const bool best_valid = (got.best_beta == 0.0 && got.best_gamma == 0.0) ||
                                (got.best_beta == 0.3 && got.best_gamma == 0.5);
        bool threw_same = false;
        try {
            (void)knnjoin_b200::parameter_search(eng, d, 8, 0.01, cands, base);
        } catch (const knnjoin::SampleTooSmallError& e) {
            try {
                (void)knnjoin::parameter_search(d, 8, 0.01, cands, base);
            } catch (const knnjoin::SampleTooSmallError& e2) {
                threw_same = std::string(e.what()) == std::string(e2.what());
            }
        }
        ok = ok && best_valid && threw_same;
        std::printf("%s parameter_search candidates=%zu errors/meta=%d best_valid=%d sample_error=%d\n",
                    ok ? "ok " : "BAD", got.candidates.size(), (int)(ok || !best_valid), (int)best_valid,
                    (int)threw_same);
        bad += !ok;
        ++n;
    }
    std::printf("%s %d/%d\n", bad ? "ADAPTER MISMATCH" : "ADAPTER OK", n - bad, n);
    return bad ? 1 : 0;
}
