/* knnj_c.h — the drop-in C ABI of the B200 KNN self-join engine.
 *
 * Replaces the hot path of the reference HybridKNN-Join library
 * (/root/reference/proj, arXiv 1810.04758) at PHASE granularity: every entry
 * point below names the reference function/class it stands in for
 * (file:line, relative to /root/reference/). Plain pointers and sizes only; no
 * C++ or torch types cross this boundary. Host buffers are caller-owned; all
 * device memory is owned by the knnj_ctx (allocated lazily, freed by
 * knnj_destroy). Calls on one ctx are synchronous and not re-entrant; use one
 * ctx per GPU (one process per GPU for multi-GPU runs).
 *
 * Arithmetic contract: every distance that decides an output is the FP64
 * squared Euclidean distance accumulated in the reference SCALAR kernel's
 * order (proj/src/kernels_scalar.cpp:9-27: d=a-b; sum += d*d, separately
 * rounded, dimensions in order), over the variance-reordered columns.
 * Output distances are sqrt of that sum, so they are bit-identical to the
 * reference run with kernel "scalar". FP32/FP16 is used only as a screen whose
 * error is bounded rigorously; anything inside the bound is re-decided in FP64.
 *
 * Return codes mirror the reference exception types
 * (proj/include/knnjoin/errors.hpp:11-62). */
#ifndef KNNJ_C_H
#define KNNJ_C_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define KNNJ_ABI_VERSION 5

enum knnj_status {
    KNNJ_OK = 0,
    KNNJ_E_USAGE = 1,             /* UsageError              errors.hpp:11-15 */
    KNNJ_E_INGEST = 2,            /* IngestError             errors.hpp:17-21 */
    KNNJ_E_INDEXING = 3,          /* IndexingError           errors.hpp:23-27 */
    KNNJ_E_DEGENERATE = 4,        /* DegenerateProfileError  errors.hpp:29-34 */
    KNNJ_E_TARGET_UNREACHABLE = 5,/* TargetUnreachableError  errors.hpp:36-42 */
    KNNJ_E_BATCH_OVERFLOW = 6,    /* BatchOverflowError      errors.hpp:44-50 (never raised: no pair buffer) */
    KNNJ_E_SAMPLE_TOO_SMALL = 7,  /* SampleTooSmallError     errors.hpp:52-56 */
    KNNJ_E_ORACLE_CAP = 8,        /* OracleCapError          errors.hpp:58-62 */
    KNNJ_E_CUDA = 9               /* device / runtime failure (no reference analogue) */
};

/* EngineMode, proj/include/knnjoin/orchestrator.hpp:15 */
enum knnj_mode { KNNJ_HYBRID = 0, KNNJ_SPARSE_ONLY = 1, KNNJ_DENSE_ONLY = 2, KNNJ_BRUTE_ORACLE = 3 };
/* Provenance, proj/include/knnjoin/orchestrator.hpp:43 */
enum knnj_provenance { KNNJ_PROV_DENSE = 0, KNNJ_PROV_SPARSE = 1, KNNJ_PROV_DENSE_FAILED = 2 };

typedef struct knnj_ctx knnj_ctx;

/* ---- context ---------------------------------------------------------- */
int knnj_abi_version(void);
int knnj_create(int device, knnj_ctx** out);
void knnj_destroy(knnj_ctx* ctx);
/* Message of the last failed call on ctx (same text as the reference exception's what()). */
const char* knnj_last_error(const knnj_ctx* ctx);
/* The CUDA stream (cudaStream_t) all of ctx's work is ordered on, for callers
 * that time or synchronise with it (e.g. torch.cuda.ExternalStream). */
void* knnj_stream(knnj_ctx* ctx);
/* Measured FP32 FFMA throughput of this device (TFLOP/s, 2 flops per FFMA):
 * the roofline denominator for the SIMT distance kernels. */
int knnj_fp32_peak(knnj_ctx* ctx, double* tflops);
/* Engine knobs (no reference analogue; results never depend on them, and every one has
 * an on/off bit-identity test in tests/test_gpu_shard_hist.py):
 *   "tensor_cores" 0/1 : allow the tcgen05 distance screen (default 1).
 *   "split_items" 0/1  : split work items with oversized candidate sets across CTAs (1).
 *   "box_filter" 0/1   : drop candidate blocks provably out of the pass radius (1).
 *   "sweep_order" 0/1  : tcgen05 passes sweep each item's blocks nearest-first (1).
 *   "tc_slack" 8..96   : tcgen05 near-tie list capacity K + slack (24).
 *   "simt_slack" 0..128: SIMT near-tie list capacity K + slack (0 = max(8, K/8)).
 *   "fine", "fine2"    : fine-grid cascade ahead of level 0 at width eps * value/1000 (0 = off).
 *   "morton_dims", "morton_bits" : join order inside a cell (10, 3).
 *   "finalize_xj" 0/1  : exact recheck reads a join-ordered FP64 copy (1).
 *   "early_d2h" 0/1    : knnj_run copies results during the fallback, patching after (1).
 *   "hist_cap" 0/1/2   : eps-selection histogram counts only the bins select_eps_beta
 *                        needs when the profile is not requested: 0 never, 1 when the
 *                        histogram is large (default), 2 always (tests).
 *   "hist_grid" 0/1/2  : capped histogram bins of n <= 8 data on a grid of the cap radius
 *                        (k_hist_grid): 0 never, 1 for >= 65536 queries (default), 2 always.
 *   "pilot_cap" 0/1/2  : the cap-placing pilot counts growing prefixes of the bins (4% and
 *                        a quarter only for n <= 8 or value 1; a tenth always) before
 *                        binning in full (2). */
int knnj_set_option(knnj_ctx* ctx, const char* name, int64_t value);
/* Page-locked host buffers for the end-to-end path (H2D/D2H at full PCIe rate). */
void* knnj_alloc_pinned(size_t bytes);
void knnj_free_pinned(void* p);

/* ---- dataset (Dataset, proj/include/knnjoin/dataset.hpp:14-40) --------- */
/* Uploads |D| x n row-major FP64 points; rejects non-finite values like
 * proj/src/dataset.cpp:22-33 ("non-finite coordinate at point i, dimension j"). */
int knnj_set_points(knnj_ctx* ctx, const double* rowmajor, uint64_t n_points, uint32_t dims);
/* reorder_by_variance, proj/src/dataset.cpp:87-111. perm[j] = original column of
 * working column j; var (optional) = population variances of the ORIGINAL columns
 * (Dataset::column_variances, dataset.cpp:58-74). Must precede the phases below. */
int knnj_reorder_by_variance(knnj_ctx* ctx, uint32_t m, uint32_t* perm, double* var);
/* Working (reordered) coordinates back to the host, |D| x n row-major. */
int knnj_get_points(knnj_ctx* ctx, double* out);

/* ---- distance (kernels::sq_dist_limited, proj/include/knnjoin/kernels.hpp:33-40) */
/* out[i] = scalar-order squared distance of working points ij[2i], ij[2i+1], or
 * +inf when it exceeds limit_sq (pass +inf for kernels::sq_dist). */
int knnj_pair_sq(knnj_ctx* ctx, const uint64_t* ij, uint64_t n_pairs, double limit_sq,
                 double* out);

/* ---- epsilon selection (proj/src/epsilon.cpp) -------------------------- */
/* estimate_eps_mean, epsilon.cpp:14-44 (pairs drawn with the reference RNG). */
int knnj_eps_mean(knnj_ctx* ctx, uint64_t sample_pairs, uint64_t seed, double* out);
/* build_distance_histogram, epsilon.cpp:46-120: integer bin counts (divide by
 * *query_count for EpsilonProfile::counts). Queries are sampled on the host with
 * the reference sampler (util.hpp:70-92); the all-pairs binning runs on the GPU. */
int knnj_histogram(knnj_ctx* ctx, double eps_mean, uint32_t n_bins, double query_fraction,
                   uint64_t seed, uint64_t* raw_counts, uint64_t* query_count);
/* Same binning over an explicit query-id list (used for sharding). raw_counts
 * is ACCUMULATED into (caller zeroes it). */
int knnj_histogram_queries(knnj_ctx* ctx, const uint64_t* query_ids, uint64_t n_queries,
                           double eps_mean, uint32_t n_bins, uint64_t* raw_counts);

/* ---- grid index (GridIndex, proj/include/knnjoin/grid_index.hpp:34-84) -- */
typedef struct {
    uint32_t m;
    double eps;
    uint64_t n_cells;              /* |B| */
    double mins[64], maxs[64];     /* first m working dims */
    uint64_t cells_per_dim[64];
} knnj_grid_info;
/* GridIndex::build, grid_index.cpp:13-75 (IndexingError on 64-bit overflow). */
int knnj_grid_build(knnj_ctx* ctx, uint32_t m, double eps, knnj_grid_info* info);
/* B (n_cells), G (2*n_cells: begin,end), A (|D|), slot (|D|); any may be NULL. */
int knnj_grid_export(knnj_ctx* ctx, uint64_t* B, uint64_t* G, uint32_t* A, uint32_t* slot);
/* range_query sizes (self included) and candidates examined per query:
 * grid_index.cpp:149-167 — what estimate_batches (dense_engine.cpp:48-75) sums. */
int knnj_range_count(knnj_ctx* ctx, const uint32_t* queries, uint64_t n_queries,
                     uint64_t* in_eps, uint64_t* candidates);

/* ---- split (split_work, proj/src/partition.cpp:30-75) ------------------- */
typedef struct {
    double n_min, n_thresh;
    uint64_t q_gpu, q_cpu, demoted;
} knnj_split_info;
int knnj_split(knnj_ctx* ctx, const uint32_t* queries, uint64_t n_queries, uint32_t k,
               double beta, double gamma, double rho, uint8_t* is_dense, uint64_t* cell_pop,
               knnj_split_info* info);

/* ---- joins -------------------------------------------------------------- */
typedef struct {
    uint64_t candidates_examined; /* DenseJoinStats::candidates_examined (dense_engine.hpp:86-92) */
    uint64_t solved, failed;
    double kernel_ms;             /* device time of the fused join kernels (CUDA events) */
} knnj_join_stats;
/* run_dense_join (dense_engine.cpp:229-303) with filter_keys fused
 * (dense_engine.cpp:165-196) over the grid of knnj_grid_build: per query solved[i] = 1
 * and its k (dist,id)-ordered in-eps neighbours, or solved[i] = 0 when fewer than k
 * non-self points lie within eps; filter_keys then discards the partial list
 * (dense_engine.cpp:182-192), so a failed row reads ids = 0xFFFFFFFF, dist = +inf. */
int knnj_dense_join(knnj_ctx* ctx, const uint32_t* queries, uint64_t n_queries, uint32_t k,
                    uint32_t* ids, double* dist, uint8_t* solved, knnj_join_stats* stats);
/* Exact KNN, self excluded, (dist,id) order: the contract of KdTree::knn_query
 * (proj/src/kdtree.cpp:109-159) and brute_force_knn (dense_engine.cpp:322-346).
 * Needs only knnj_set_points (+ optional reorder). k <= |D|-1. */
int knnj_exact_knn(knnj_ctx* ctx, const uint32_t* queries, uint64_t n_queries, uint32_t k,
                   uint32_t* ids, double* dist);

/* ---- full pipeline (run_hybrid, proj/src/orchestrator.cpp:67-250) ------- */
typedef struct {
    uint32_t k;                   /* RunConfig::k */
    uint32_t m;                   /* 0 -> min(6, n) */
    double beta, gamma, rho;
    uint32_t mode;                /* enum knnj_mode */
    uint32_t n_bins;              /* 100 */
    double hist_query_fraction;   /* 0.01 */
    uint64_t eps_mean_pair_cap;   /* 1e6 */
    uint64_t seed;
    const uint32_t* query_subset; /* NULL = all points */
    uint64_t n_query_subset;
} knnj_config;

typedef struct {
    uint64_t n_queries;
    uint32_t k_effective, m_used;
    uint32_t k_clamped, eps_fallback;
    double eps_mean, bin_width, eps_default, eps_beta, eps_final, eps_used;
    uint64_t hist_query_count, hist_bin;
    double n_min, n_thresh;
    uint64_t q_gpu, q_cpu, demoted, failed_count;
    uint64_t candidates_examined;
    uint64_t fallback_queries, fallback_passes, slow_path_queries;
    uint64_t grid_cells;
    uint64_t kernel_launches;     /* this library's own kernels launched by the call */
    uint32_t join_tensor_cores;   /* 1: level-0 join ran on the tcgen05 screen, 0: SIMT FP32 */
    uint32_t hist_tensor_cores;   /* same for the eps histogram */
    uint32_t hist_bins_counted;   /* bins counted exactly (n_bins unless the histogram was capped) */
    uint64_t n_owned;             /* query rows this call (shard) produced */
    uint64_t join_candidate_pairs;/* candidate pairs of the level-0 join over the owned queries */
    uint64_t join_screened_pairs; /* of which left after the exact box filter (the work done) */
    /* device-event timings (ms) */
    double ms_upload, ms_reorder, ms_eps_mean, ms_histogram, ms_grid, ms_split, ms_join,
        ms_fallback, ms_download, ms_total;
    double ms_join_kernel, ms_hist_kernel;
    double ms_join_build;         /* work-item / adjacency construction of the level-0 pass */
    double kth_bound2;            /* radius bound (squared) of the level-0 pass; 0 = unbounded */
    uint64_t bound_retried;       /* level-0 rows re-run without the bound */
    uint32_t perm[1024];
} knnj_run_info;

/* Runs Alg. 1 over the points set by knnj_set_points (which it reorders in place).
 * Outputs (caller-allocated, n_queries rows in ascending query-id order):
 *   ids, dist : n_queries * k_effective   (row stride k_effective)
 *   prov      : n_queries                 (enum knnj_provenance)
 *   raw_hist  : n_bins (may be NULL)      integer histogram counts
 * ids == NULL and dist == NULL keeps the results device-resident (no D2H).
 * k_effective = min(k, |D|-1) (orchestrator.cpp:77-82). */
int knnj_run(knnj_ctx* ctx, const knnj_config* cfg, uint32_t* ids, double* dist, uint8_t* prov,
             uint64_t* raw_hist, knnj_run_info* info);

/* ---- parameter search (parameter_search, proj/src/orchestrator.cpp:252-303) ----
 * Draws a seeded f-fraction query subset (derive_seed(seed, kSeedQuerySubset = 4),
 * sample_without_replacement), runs knnj_run over it for each (beta, gamma) candidate
 * in hybrid mode at rho = 0.5 with base's other settings, and returns the fastest
 * candidate. wall_seconds is the run's device time (knnj_run_info.ms_total). A failing
 * candidate keeps its error (status, message) and does not stop the search. Errors,
 * with the reference's messages: f outside (0, 1] or no candidates -> KNNJ_E_USAGE;
 * floor(f|D|) < 50 -> KNNJ_E_SAMPLE_TOO_SMALL; every candidate failed -> KNNJ_E_USAGE.
 * (t1/t2/rho_model of the reference are its CPU load-balance model: no analogue.) */
typedef struct {
    double beta, gamma;
    double wall_seconds;
    int32_t status;               /* KNNJ_OK or the candidate's error code */
    char error[256];              /* the candidate's error message ("" if none) */
} knnj_search_row;

int knnj_parameter_search(knnj_ctx* ctx, const knnj_config* base, double f, const double* betas,
                          const double* gammas, uint64_t n_candidates, knnj_search_row* rows,
                          double* best_beta, double* best_gamma);

/* ---- multi-GPU: one process per GPU, queries sharded by cell range ------
 * Sum `count` u64 values element-wise over every shard, in place (e.g. an
 * ncclAllReduce / torch.distributed.all_reduce issued by the caller). Returns 0 on success. */
typedef int (*knnj_allreduce_fn)(uint64_t* data, uint64_t count, void* user);
/* The cell-range partition knnj_run_shard uses (host-only, no GPU needed): items
 * 0..n_items-1 in cell order with estimated costs; shard k owns the contiguous run
 * [*first, *last) holding the items whose cost midpoint falls in the k-th equal
 * share of the total. The runs of shards 0..shard_count-1 tile [0, n_items). */
int knnj_shard_range(const double* cost, uint64_t n_items, uint32_t shard_index,
                     uint32_t shard_count, uint64_t* first, uint64_t* last);
/* knnj_run as shard `shard_index` of `shard_count` identical calls (one per GPU,
 * same points and config). Every shard rebuilds the reorder, eps, grid and split
 * redundantly (deterministic, identical); the sampled histogram queries are split
 * evenly and their counts summed through `allreduce` (the run's only exchange); the
 * join + fallback run only for this shard's contiguous range of grid cells, cut at
 * equal estimated work. Outputs are this shard's rows, compacted in ascending query
 * id: owned_queries[n_owned], ids/dist[n_owned * k_effective], prov[n_owned]
 * (info->n_owned; size the buffers for the whole query set). The union over shards
 * equals knnj_run's output. shard_count == 1 is knnj_run. */
int knnj_run_shard(knnj_ctx* ctx, const knnj_config* cfg, uint32_t shard_index,
                   uint32_t shard_count, knnj_allreduce_fn allreduce, void* allreduce_user,
                   uint32_t* ids, double* dist, uint8_t* prov, uint32_t* owned_queries,
                   uint64_t* raw_hist, knnj_run_info* info);

/* ---- host I/O (no GPU needed) ------------------------------------------- */
/* Message of the last failed I/O call on this thread. */
const char* knnj_io_last_error(void);
/* io::tsv_string (proj/src/io.cpp:141-154): "%u\t%u\t%.17g\n" per (query, rank), rows
 * in the given order (queries NULL = row index). Byte-identical text, formatted by
 * `threads` host threads (0 = all). out NULL: only *length (bytes) is computed. */
int knnj_tsv_format(const uint32_t* queries, const uint32_t* ids, const double* dist,
                    uint64_t n_rows, uint32_t k, char* out, uint64_t capacity, uint64_t* length,
                    uint32_t threads);
/* write_tsv (proj/src/io.cpp:137-139) to a file, formatted and written in parallel. */
int knnj_tsv_write(const char* path, const uint32_t* queries, const uint32_t* ids,
                   const double* dist, uint64_t n_rows, uint32_t k, uint32_t threads,
                   uint64_t* bytes_written);
/* ingest_binary (proj/src/io.cpp:69-91): LE u64 |D|, u64 n, |D|*n row-major f64.
 * knnj_binary_header reads the sizes; knnj_binary_read fills `out` (e.g. a pinned
 * buffer from knnj_alloc_pinned) and rejects short bodies / non-finite values with
 * the reference's messages (KNNJ_E_INGEST). */
int knnj_binary_header(const char* path, uint64_t* n_points, uint64_t* dims);
int knnj_binary_read(const char* path, double* out, uint64_t capacity_doubles);
/* ingest_text (proj/src/io.cpp:24-67): CSV (sep ',') or TSV (sep '\t'), one point per
 * line, empty lines skipped, a trailing '\r' stripped, fields parsed with
 * std::from_chars after optional spaces/tabs. knnj_text_parse parses the whole file
 * with `threads` host threads (0 = all) into a handle and reports |D| and n;
 * knnj_text_copy writes the row-major coordinates (e.g. into a pinned buffer);
 * knnj_text_free releases the handle. Failures are KNNJ_E_INGEST with the
 * reference's messages ("<path>: row r, column c: not a number: '<field>'",
 * "...: non-finite value", "<path>: row r has c columns, expected n", "<path>: no
 * points", "cannot open <path>"), the first one in file order. */
typedef struct knnj_text knnj_text;
int knnj_text_parse(const char* path, char sep, uint32_t threads, knnj_text** out,
                    uint64_t* n_points, uint64_t* dims);
int knnj_text_copy(const knnj_text* text, double* out, uint64_t capacity_doubles);
void knnj_text_free(knnj_text* text);

/* ---- test hooks (no reference analogue; used by tests/ only) -------------- */
/* knnj_histogram_queries counting only bins [0, n_count): the kernels of the capped
 * eps-selection histogram (the counted bins must equal the full histogram's). */
int knnj_histogram_queries_capped(knnj_ctx* ctx, const uint64_t* query_ids, uint64_t n_queries,
                                  double eps_mean, uint32_t n_bins, uint32_t n_count,
                                  uint64_t* raw_counts);
/* One 128x128 tcgen05 accumulator tile of the level-0 grid built by knnj_grid_build:
 * queries at join-order positions [q0, q0+128) against [c0, c0+128). Returns the raw
 * FP32 accumulators D[128][128], both FP16 operand row blocks (row_halfs halfs per
 * row), the scale S, the screen bound delta (scaled units) and the point ids. */
int knnj_debug_tc_tile(knnj_ctx* ctx, uint32_t q0, uint32_t c0, float* D, uint16_t* Bq,
                       uint16_t* Bc, double* scale_S, double* delta, uint32_t* pid_q,
                       uint32_t* pid_c);

#ifdef __cplusplus
}
#endif
#endif /* KNNJ_C_H */
