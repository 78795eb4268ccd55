/* TEST INFRASTRUCTURE ONLY — CPU oracle (checker) for the KNN self-join hot path.
 * See knnj_oracle.h for scope and pinning. Compiled with -ffp-contract=off so every
 * FP64 product and sum rounds separately, as in the reference scalar kernel.
 * Parity status: PINNED (tests/test_oracle_golden.py: reference known-answer
 * tests + fixtures produced by the unmodified reference in tests/golden/). */
#include "knnj_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

/* ---------------------------------------------------------------- distance */

/* proj/src/kernels_scalar.cpp:9-27: single accumulator, strict dimension order,
 * checkpoint every 8 terms. */
double orc_sq_dist_limited(const double* a, const double* b, size_t n, double limit_sq) {
    double sum = 0.0;
    size_t i = 0;
    while (i + 8 <= n) {
        for (size_t j = 0; j < 8; ++j) {
            double d = a[i + j] - b[i + j];
            sum += d * d;
        }
        i += 8;
        if (sum > limit_sq) return INFINITY;
    }
    for (; i < n; ++i) {
        double d = a[i] - b[i];
        sum += d * d;
    }
    if (sum > limit_sq) return INFINITY;
    return sum;
}

/* ---------------------------------------------------------------- RNG */

#define MT_N 312
#define MT_M 156
void orc_mt_seed(orc_mt64* s, uint64_t seed) {
    s->mt[0] = seed;
    for (int i = 1; i < MT_N; ++i)
        s->mt[i] = 6364136223846793005ULL * (s->mt[i - 1] ^ (s->mt[i - 1] >> 62)) + (uint64_t)i;
    s->mti = MT_N;
}

static void mt_twist(orc_mt64* s) {
    const uint64_t upper = ~0ULL << 31, lower = ~upper, a = 0xB5026F5AA96619E9ULL;
    int k;
    for (k = 0; k < MT_N - MT_M; ++k) {
        uint64_t y = (s->mt[k] & upper) | (s->mt[k + 1] & lower);
        s->mt[k] = s->mt[k + MT_M] ^ (y >> 1) ^ ((y & 1) ? a : 0);
    }
    for (; k < MT_N - 1; ++k) {
        uint64_t y = (s->mt[k] & upper) | (s->mt[k + 1] & lower);
        s->mt[k] = s->mt[k + (MT_M - MT_N)] ^ (y >> 1) ^ ((y & 1) ? a : 0);
    }
    uint64_t y = (s->mt[MT_N - 1] & upper) | (s->mt[0] & lower);
    s->mt[MT_N - 1] = s->mt[MT_M - 1] ^ (y >> 1) ^ ((y & 1) ? a : 0);
    s->mti = 0;
}

uint64_t orc_mt_next(orc_mt64* s) {
    if (s->mti >= MT_N) mt_twist(s);
    uint64_t z = s->mt[s->mti++];
    z ^= (z >> 29) & 0x5555555555555555ULL;
    z ^= (z << 17) & 0x71D67FFFEDA60000ULL;
    z ^= (z << 37) & 0xFFF7EEE000000000ULL;
    z ^= z >> 43;
    return z;
}

/* libstdc++ uniform_int_distribution<u64>::operator() with a 64-bit engine:
 * full range -> raw draw, else Lemire's nearly-divisionless downscale. */
uint64_t orc_uniform_u64(orc_mt64* s, uint64_t a, uint64_t b) {
    uint64_t urange = b - a;
    if (urange == ~0ULL) return orc_mt_next(s) + a;
    uint64_t range = urange + 1;
    unsigned __int128 product = (unsigned __int128)orc_mt_next(s) * range;
    uint64_t low = (uint64_t)product;
    if (low < range) {
        uint64_t threshold = (0 - range) % range;
        while (low < threshold) {
            product = (unsigned __int128)orc_mt_next(s) * range;
            low = (uint64_t)product;
        }
    }
    return (uint64_t)(product >> 64) + a;
}

static uint64_t splitmix64(uint64_t x) {
    x += 0x9e3779b97f4a7c15ULL;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
    return x ^ (x >> 31);
}
uint64_t orc_derive_seed(uint64_t master, uint64_t tag) {
    return splitmix64(master ^ splitmix64(tag));
}

/* open-addressing u64 -> u64 map (stands in for the reference's unordered_map;
 * only membership/lookup semantics matter) */
typedef struct {
    uint64_t* keys;
    uint64_t* vals;
    uint8_t* used;
    uint64_t cap;
} u64map;
static void map_init(u64map* m, uint64_t want) {
    uint64_t cap = 16;
    while (cap < 2 * want + 16) cap <<= 1;
    m->cap = cap;
    m->keys = malloc(cap * 8);
    m->vals = malloc(cap * 8);
    m->used = calloc(cap, 1);
}
static void map_free(u64map* m) {
    free(m->keys);
    free(m->vals);
    free(m->used);
}
static uint64_t* map_find(u64map* m, uint64_t key, int insert) {
    uint64_t h = splitmix64(key) & (m->cap - 1);
    while (m->used[h]) {
        if (m->keys[h] == key) return &m->vals[h];
        h = (h + 1) & (m->cap - 1);
    }
    if (!insert) return NULL;
    m->used[h] = 1;
    m->keys[h] = key;
    return &m->vals[h];
}
static int cmp_u64(const void* a, const void* b) {
    uint64_t x = *(const uint64_t*)a, y = *(const uint64_t*)b;
    return x < y ? -1 : x > y;
}

/* proj/include/knnjoin/util.hpp:70-92 (partial Fisher-Yates over an index map) */
uint64_t orc_sample_without_replacement(uint64_t n, uint64_t k, orc_mt64* rng, uint64_t* out) {
    if (k >= n) {
        for (uint64_t i = 0; i < n; ++i) out[i] = i;
        return n;
    }
    u64map m;
    map_init(&m, k);
    for (uint64_t i = 0; i < k; ++i) {
        uint64_t j = orc_uniform_u64(rng, i, n - 1);
        uint64_t* jp = map_find(&m, j, 0);
        uint64_t jv = jp ? *jp : j;
        uint64_t* ip = map_find(&m, i, 0);
        uint64_t iv = ip ? *ip : i;
        out[i] = jv;
        *map_find(&m, j, 1) = iv;
    }
    map_free(&m);
    qsort(out, k, 8, cmp_u64);
    return k;
}

/* ---------------------------------------------------------------- dataset */

/* proj/src/dataset.cpp:58-74 (two-pass population variance in point order) and
 * :87-111 (full descending sort, ties to the lower index). */
void orc_variance_order(const double* X, uint64_t N, uint32_t n, uint32_t* order, double* var) {
    double* mean = calloc(n, sizeof(double));
    double* v = calloc(n, sizeof(double));
    for (uint64_t i = 0; i < N; ++i)
        for (uint32_t j = 0; j < n; ++j) mean[j] += X[i * n + j];
    for (uint32_t j = 0; j < n; ++j) mean[j] /= (double)N;
    for (uint64_t i = 0; i < N; ++i)
        for (uint32_t j = 0; j < n; ++j) {
            double d = X[i * n + j] - mean[j];
            v[j] += d * d;
        }
    for (uint32_t j = 0; j < n; ++j) v[j] /= (double)N;
    for (uint32_t j = 0; j < n; ++j) order[j] = j;
    /* insertion sort: (var desc, index asc) */
    for (uint32_t a = 1; a < n; ++a) {
        uint32_t x = order[a];
        int b = (int)a - 1;
        while (b >= 0 && (v[order[b]] < v[x] || (v[order[b]] == v[x] && order[b] > x))) {
            order[b + 1] = order[b];
            --b;
        }
        order[b + 1] = x;
    }
    if (var) memcpy(var, v, n * sizeof(double));
    free(mean);
    free(v);
}

void orc_permute_columns(const double* X, uint64_t N, uint32_t n, const uint32_t* order,
                         double* out) {
    for (uint64_t i = 0; i < N; ++i)
        for (uint32_t j = 0; j < n; ++j) out[i * n + j] = X[i * n + order[j]];
}

/* ---------------------------------------------------------------- threads */

typedef void (*task_fn)(void* ctx, uint64_t i, uint32_t tid);
typedef struct {
    task_fn fn;
    void* ctx;
    uint64_t n;
    uint64_t next;
    pthread_mutex_t mu;
    uint32_t tid;
} pool_t;
typedef struct {
    pool_t* p;
    uint32_t tid;
} worker_arg;
static void* worker_main(void* arg) {
    worker_arg* w = arg;
    pool_t* p = w->p;
    for (;;) {
        pthread_mutex_lock(&p->mu);
        uint64_t i = p->next++;
        pthread_mutex_unlock(&p->mu);
        if (i >= p->n) return NULL;
        p->fn(p->ctx, i, w->tid);
    }
}
static void parallel_for(uint64_t n, uint32_t threads, task_fn fn, void* ctx) {
    if (threads <= 1 || n <= 1) {
        for (uint64_t i = 0; i < n; ++i) fn(ctx, i, 0);
        return;
    }
    pool_t p = {fn, ctx, n, 0, PTHREAD_MUTEX_INITIALIZER, 0};
    pthread_t* th = malloc(sizeof(pthread_t) * threads);
    worker_arg* wa = malloc(sizeof(worker_arg) * threads);
    for (uint32_t t = 0; t < threads; ++t) {
        wa[t].p = &p;
        wa[t].tid = t;
        pthread_create(&th[t], NULL, worker_main, &wa[t]);
    }
    for (uint32_t t = 0; t < threads; ++t) pthread_join(th[t], NULL);
    free(th);
    free(wa);
}

/* ---------------------------------------------------------------- epsilon */

/* proj/src/epsilon.cpp:14-44 */
int orc_eps_mean(const double* X, uint64_t N, uint32_t n, uint64_t pairs, uint64_t seed,
                 double* out) {
    if (N < 2 || pairs < 1) return 1;
    const uint64_t all = N * (N - 1);
    double sum = 0.0;
    uint64_t used;
    if (pairs >= all) {
        for (uint64_t i = 0; i < N; ++i)
            for (uint64_t j = 0; j < N; ++j) {
                if (i == j) continue;
                sum += sqrt(orc_sq_dist_limited(X + i * n, X + j * n, n, INFINITY));
            }
        used = all;
    } else {
        orc_mt64 rng;
        orc_mt_seed(&rng, seed);
        for (uint64_t s = 0; s < pairs; ++s) {
            uint64_t i = orc_uniform_u64(&rng, 0, N - 1);
            uint64_t j = orc_uniform_u64(&rng, 0, N - 1);
            while (j == i) j = orc_uniform_u64(&rng, 0, N - 1);
            sum += sqrt(orc_sq_dist_limited(X + i * n, X + j * n, n, INFINITY));
        }
        used = pairs;
    }
    *out = sum / (double)used;
    return 0;
}

typedef struct {
    const double* X;
    uint64_t N;
    uint32_t n, n_bins;
    const uint64_t* queries;
    double eps_mean, limit_sq, inv_width;
    uint64_t* local; /* threads * n_bins */
} hist_ctx;

static void hist_task(void* vc, uint64_t qi, uint32_t tid) {
    hist_ctx* c = vc;
    uint64_t* bins = c->local + (uint64_t)tid * c->n_bins;
    const uint64_t q = c->queries[qi];
    const double* qp = c->X + q * c->n;
    for (uint64_t t = 0; t < c->N; ++t) {
        if (t == q) continue;
        double sq = orc_sq_dist_limited(qp, c->X + t * c->n, c->n, c->limit_sq);
        if (isinf(sq)) continue;
        double dist = sqrt(sq);
        if (dist >= c->eps_mean) continue;
        uint64_t b = (uint64_t)(dist * c->inv_width);
        if (b >= c->n_bins) b = c->n_bins - 1;
        ++bins[b];
    }
}

/* proj/src/epsilon.cpp:46-120 */
int orc_histogram(const double* X, uint64_t N, uint32_t n, double eps_mean, uint32_t n_bins,
                  double frac, uint64_t seed, uint32_t threads, uint64_t* raw,
                  uint64_t* query_count) {
    if (!(eps_mean > 0.0)) return 4;
    if (n_bins < 2) return 1;
    if (!(frac > 0.0) || frac > 1.0) return 1;
    double bin_width = eps_mean / (double)n_bins;
    uint64_t want = (uint64_t)floor(frac * (double)N);
    if (want < 100) want = 100;
    if (want > N) want = N;
    uint64_t* queries = malloc(sizeof(uint64_t) * (want ? want : 1));
    orc_mt64 rng;
    orc_mt_seed(&rng, seed);
    uint64_t nq = orc_sample_without_replacement(N, want, &rng, queries);
    if (threads < 1) threads = 1;
    hist_ctx c = {X, N, n, n_bins, queries, eps_mean, eps_mean * eps_mean, 1.0 / bin_width,
                  calloc((size_t)threads * n_bins, 8)};
    parallel_for(nq, threads, hist_task, &c);
    for (uint32_t b = 0; b < n_bins; ++b) {
        raw[b] = 0;
        for (uint32_t t = 0; t < threads; ++t) raw[b] += c.local[(uint64_t)t * n_bins + b];
    }
    *query_count = nq;
    free(c.local);
    free(queries);
    return 0;
}

/* The per-query binning of build_distance_histogram (proj/src/epsilon.cpp:76-104) over
 * an explicit query-id list: checks the device histogram on a subset of the sampled
 * queries at sizes where the whole sample is out of the oracle's reach. */
int orc_histogram_queries(const double* X, uint64_t N, uint32_t n, double eps_mean,
                          uint32_t n_bins, const uint64_t* queries, uint64_t nq,
                          uint32_t threads, uint64_t* raw) {
    if (!(eps_mean > 0.0)) return 4;
    if (n_bins < 2) return 1;
    for (uint64_t i = 0; i < nq; ++i)
        if (queries[i] >= N) return 1;
    if (threads < 1) threads = 1;
    double bin_width = eps_mean / (double)n_bins;
    hist_ctx c = {X, N, n, n_bins, queries, eps_mean, eps_mean * eps_mean, 1.0 / bin_width,
                  calloc((size_t)threads * n_bins, 8)};
    parallel_for(nq, threads, hist_task, &c);
    for (uint32_t b = 0; b < n_bins; ++b) {
        raw[b] = 0;
        for (uint32_t t = 0; t < threads; ++t) raw[b] += c.local[(uint64_t)t * n_bins + b];
    }
    free(c.local);
    return 0;
}

/* proj/src/epsilon.cpp:122-141 + orchestrator.cpp:49-63 */
int orc_select_eps(const double* cum, uint32_t n_bins, double bin_width, uint32_t k, double beta,
                   int allow_fallback, double* eps_beta, double* eps_final, uint64_t* bin,
                   int* fell_back) {
    const double target = (double)k + (100.0 * (double)k - (double)k) * beta;
    uint32_t it = 0;
    while (it < n_bins && cum[it] < target) ++it; /* lower_bound */
    if (fell_back) *fell_back = 0;
    if (it == n_bins) {
        if (!allow_fallback) return 5;
        if (fell_back) *fell_back = 1;
        double top = cum[n_bins - 1];
        it = 0;
        while (it < n_bins && cum[it] < top) ++it;
    }
    uint64_t b = (uint64_t)it + 1;
    double start = (double)(b - 1) * bin_width;
    double end = (double)b * bin_width;
    *eps_beta = (start + end) / 2.0;
    *eps_final = 2.0 * *eps_beta;
    *bin = b;
    return 0;
}

/* ---------------------------------------------------------------- grid */

typedef struct {
    uint64_t key;
    uint32_t pid;
} keyed_t;

/* (key, pid) ascending, as the reference's std::sort of (linear_id, pid) pairs
 * (grid_index.cpp:56-61): the input is in pid order, so a stable LSD radix sort on the
 * key alone gives the same order (11-bit digits over the key's significant bits). */
static void sort_keyed(keyed_t* a, uint64_t N) {
    if (N < 2) return;
    uint64_t kmax = 0;
    for (uint64_t i = 0; i < N; ++i)
        if (a[i].key > kmax) kmax = a[i].key;
    int bits = 0;
    while (bits < 64 && (kmax >> bits)) ++bits;
    keyed_t* tmp = malloc(sizeof(keyed_t) * N);
    keyed_t *src = a, *dst = tmp;
    for (int sh = 0; sh < bits; sh += 11) {
        uint64_t cnt[2048] = {0};
        for (uint64_t i = 0; i < N; ++i) ++cnt[(src[i].key >> sh) & 2047u];
        uint64_t run = 0;
        for (int d = 0; d < 2048; ++d) {
            uint64_t c = cnt[d];
            cnt[d] = run;
            run += c;
        }
        for (uint64_t i = 0; i < N; ++i) dst[cnt[(src[i].key >> sh) & 2047u]++] = src[i];
        keyed_t* t = src;
        src = dst;
        dst = t;
    }
    if (src != a) memcpy(a, src, sizeof(keyed_t) * N);
    free(tmp);
}

/* proj/src/grid_index.cpp:77-94 */
static void cell_of(const orc_grid* g, const double* p, uint64_t* coords, uint64_t* linear) {
    uint64_t id = 0;
    for (uint32_t j = 0; j < g->m; ++j) {
        double rel = (p[j] - g->mins[j]) / g->eps;
        if (rel < 0.0) rel = 0.0;
        uint64_t idx = (uint64_t)floor(rel);
        if (idx > g->cpd[j] - 1) idx = g->cpd[j] - 1;
        coords[j] = idx;
        id += idx * g->strides[j];
    }
    *linear = id;
}

/* proj/src/grid_index.cpp:13-75 */
int orc_grid_build(const double* X, uint64_t N, uint32_t n, uint32_t m, double eps, orc_grid* g,
                   char* err, size_t errlen) {
    memset(g, 0, sizeof(*g));
    if (!(eps > 0.0) || m < 1 || m > n || m > 64) return 1;
    g->m = m;
    g->eps = eps;
    for (uint32_t j = 0; j < m; ++j) {
        g->mins[j] = INFINITY;
        g->maxs[j] = -INFINITY;
    }
    for (uint64_t i = 0; i < N; ++i)
        for (uint32_t j = 0; j < m; ++j) {
            double v = X[i * n + j];
            if (v < g->mins[j]) g->mins[j] = v;
            if (v > g->maxs[j]) g->maxs[j] = v;
        }
    unsigned __int128 total = 1;
    for (uint32_t j = 0; j < m; ++j) {
        double extent = (g->maxs[j] - g->mins[j]) / eps;
        if (!(extent < 9.2e18)) {
            if (err) snprintf(err, errlen, "grid extent overflows linear cell ids: dimension %u", j);
            return 3;
        }
        uint64_t c = (uint64_t)floor(extent) + 1;
        g->cpd[j] = c < 1 ? 1 : c;
        total *= g->cpd[j];
        if (total > (unsigned __int128)~0ULL) {
            if (err) snprintf(err, errlen, "grid extent overflows linear cell ids: required extent");
            return 3;
        }
    }
    g->strides[m - 1] = 1;
    for (int j = (int)m - 2; j >= 0; --j) g->strides[j] = g->strides[j + 1] * g->cpd[j + 1];

    keyed_t* keyed = malloc(sizeof(keyed_t) * (N ? N : 1));
    uint64_t coords[64];
    for (uint64_t i = 0; i < N; ++i) {
        cell_of(g, X + i * n, coords, &keyed[i].key);
        keyed[i].pid = (uint32_t)i;
    }
    sort_keyed(keyed, N);
    g->B = malloc(8 * (N ? N : 1));
    g->G = malloc(16 * (N ? N : 1));
    g->A = malloc(4 * (N ? N : 1));
    g->slot = malloc(4 * (N ? N : 1));
    uint64_t nc = 0;
    for (uint64_t i = 0; i < N; ++i) {
        if (i == 0 || keyed[i].key != keyed[i - 1].key) {
            g->B[nc] = keyed[i].key;
            g->G[2 * nc] = i;
            ++nc;
        }
        g->G[2 * (nc - 1) + 1] = i + 1;
        g->A[i] = keyed[i].pid;
        g->slot[keyed[i].pid] = (uint32_t)(nc - 1);
    }
    g->ncells = nc;
    free(keyed);
    return 0;
}

void orc_grid_free(orc_grid* g) {
    free(g->B);
    free(g->G);
    free(g->A);
    free(g->slot);
    memset(g, 0, sizeof(*g));
}

static uint64_t lower_bound_u64(const uint64_t* a, uint64_t n, uint64_t key) {
    uint64_t lo = 0, hi = n;
    while (lo < hi) {
        uint64_t mid = lo + (hi - lo) / 2;
        if (a[mid] < key) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

/* ---------------------------------------------------------------- partition */

/* proj/src/partition.cpp:12-23 */
double orc_n_min(uint32_t k, uint32_t m_eff) {
    double m = (double)m_eff;
    return (double)k * pow(2.0, m) * tgamma(m / 2.0 + 1.0) / pow(3.14159265358979323846, m / 2.0);
}
double orc_n_thresh(double n_min, double gamma) { return n_min + (10.0 * n_min - n_min) * gamma; }

/* ---------------------------------------------------------------- top-k */

/* canonical (sq, id) order: proj/src/kdtree.cpp:17-24, dense_engine.cpp:176-191 */
static inline int less_pair(double sa, uint32_t ia, double sb, uint32_t ib) {
    return sa < sb || (sa == sb && ia < ib);
}
static inline void topk_insert(double* sq, uint32_t* id, uint32_t* cnt, uint32_t k, double s,
                               uint32_t t) {
    uint32_t c = *cnt;
    if (c == k) {
        if (!less_pair(s, t, sq[k - 1], id[k - 1])) return;
        c = k - 1;
    }
    int p = (int)c - 1;
    while (p >= 0 && less_pair(s, t, sq[p], id[p])) {
        sq[p + 1] = sq[p];
        id[p + 1] = id[p];
        --p;
    }
    sq[p + 1] = s;
    id[p + 1] = t;
    if (*cnt < k) ++*cnt;
}

typedef struct {
    const double* X;
    uint64_t N;
    uint32_t n, k;
    const uint32_t* q;
    uint32_t* ids;
    double* dist;
} brute_ctx;
static void brute_task(void* vc, uint64_t qi, uint32_t tid) {
    (void)tid;
    brute_ctx* c = vc;
    uint32_t q = c->q[qi];
    double sq[1024];
    uint32_t id[1024], cnt = 0;
    for (uint64_t t = 0; t < c->N; ++t) {
        if (t == q) continue;
        double s = orc_sq_dist_limited(c->X + (uint64_t)q * c->n, c->X + t * c->n, c->n, INFINITY);
        topk_insert(sq, id, &cnt, c->k, s, (uint32_t)t);
    }
    for (uint32_t j = 0; j < cnt; ++j) {
        c->ids[qi * c->k + j] = id[j];
        c->dist[qi * c->k + j] = sqrt(sq[j]);
    }
}

/* proj/src/dense_engine.cpp:322-346 */
int orc_brute_knn(const double* X, uint64_t N, uint32_t n, const uint32_t* q, uint64_t nq,
                  uint32_t k, uint32_t threads, uint32_t* ids, double* dist) {
    if (k > 1024) return 1;
    uint32_t want = (uint64_t)k < N - 1 ? k : (uint32_t)(N - 1);
    brute_ctx c = {X, N, n, want, q, ids, dist};
    /* outputs use the caller's stride k */
    if (want != k) {
        uint32_t* tmp_i = malloc(sizeof(uint32_t) * nq * (want ? want : 1));
        double* tmp_d = malloc(sizeof(double) * nq * (want ? want : 1));
        c.ids = tmp_i;
        c.dist = tmp_d;
        parallel_for(nq, threads, brute_task, &c);
        for (uint64_t i = 0; i < nq; ++i)
            for (uint32_t j = 0; j < want; ++j) {
                ids[i * k + j] = tmp_i[i * want + j];
                dist[i * k + j] = tmp_d[i * want + j];
            }
        free(tmp_i);
        free(tmp_d);
        return 0;
    }
    parallel_for(nq, threads, brute_task, &c);
    return 0;
}

/* dense join for one query: proj/src/grid_index.cpp:114-147 (3^m odometer walk,
 * lower_bound in B) + dense_engine.cpp:86-196 (eps filter, drop self, keep k). */
typedef struct {
    const double* X;
    uint32_t n, k;
    const orc_grid* g;
    double eps;
    const uint32_t* q;
    uint8_t* solved;
    uint32_t* ids;
    double* dist;
    uint64_t* cand;
} dense_ctx;
static void dense_task(void* vc, uint64_t qi, uint32_t tid) {
    (void)tid;
    dense_ctx* c = vc;
    const orc_grid* g = c->g;
    const uint32_t q = c->q[qi];
    const double* qp = c->X + (uint64_t)q * c->n;
    const double limit_sq = c->eps * c->eps;
    uint64_t center[64], lo[64], hi[64], cur[64], lin;
    cell_of(g, qp, center, &lin);
    for (uint32_t j = 0; j < g->m; ++j) {
        lo[j] = center[j] > 0 ? center[j] - 1 : 0;
        hi[j] = center[j] + 1 < g->cpd[j] - 1 ? center[j] + 1 : g->cpd[j] - 1;
        cur[j] = lo[j];
    }
    double sq[1024];
    uint32_t id[1024], cnt = 0;
    uint64_t n_in = 0, cand = 0;
    for (;;) {
        uint64_t idl = 0;
        for (uint32_t j = 0; j < g->m; ++j) idl += cur[j] * g->strides[j];
        uint64_t s = lower_bound_u64(g->B, g->ncells, idl);
        if (s < g->ncells && g->B[s] == idl) {
            for (uint64_t a = g->G[2 * s]; a < g->G[2 * s + 1]; ++a) {
                uint32_t t = g->A[a];
                ++cand;
                double d2 = orc_sq_dist_limited(qp, c->X + (uint64_t)t * c->n, c->n, limit_sq);
                if (isinf(d2) || t == q) continue;
                ++n_in;
                topk_insert(sq, id, &cnt, c->k, d2, t);
            }
        }
        uint32_t j = g->m;
        int done = 0;
        for (;;) {
            if (j == 0) {
                done = 1;
                break;
            }
            --j;
            if (cur[j] < hi[j]) {
                ++cur[j];
                break;
            }
            cur[j] = lo[j];
        }
        if (done) break;
    }
    c->cand[qi] = cand;
    c->solved[qi] = n_in >= c->k;
    if (c->solved[qi])
        for (uint32_t j = 0; j < c->k; ++j) {
            c->ids[qi * c->k + j] = id[j];
            c->dist[qi * c->k + j] = sqrt(sq[j]);
        }
}

typedef struct {
    uint64_t pop, cell;
    uint32_t pid;
} demote_t;
static int cmp_demote(const void* a, const void* b) {
    const demote_t *x = a, *y = b;
    if (x->pop != y->pop) return x->pop < y->pop ? -1 : 1;
    if (x->cell != y->cell) return x->cell < y->cell ? -1 : 1;
    return x->pid < y->pid ? -1 : (x->pid > y->pid);
}

/* proj/src/orchestrator.cpp:67-250 */
int orc_run(const double* X, uint64_t N, uint32_t n, const orc_cfg* cfg, uint32_t* ids,
            double* dist, uint8_t* prov, uint64_t* raw_hist, orc_info* info, char* err,
            size_t errlen) {
    memset(info, 0, sizeof(*info));
    if (cfg->k < 1 || cfg->m > n || n > 1024 || N < 1) return 1;
    if (cfg->beta < 0 || cfg->beta > 1 || cfg->gamma < 0 || cfg->gamma > 1 || cfg->rho < 0 ||
        cfg->rho > 1)
        return 1;
    uint32_t k_eff = cfg->k;
    if ((uint64_t)k_eff >= N) k_eff = (uint32_t)(N - 1);
    info->k_eff = k_eff;
    const uint32_t m = cfg->m == 0 ? (n < 6 ? n : 6) : cfg->m;
    info->m_used = m;
    const uint32_t threads = cfg->threads ? cfg->threads : 1;

    uint32_t order[1024];
    orc_variance_order(X, N, n, order, NULL);
    memcpy(info->perm, order, n * sizeof(uint32_t));
    double* W = malloc(sizeof(double) * N * n);
    orc_permute_columns(X, N, n, order, W);
    if (k_eff == 0) {
        free(W);
        return 0;
    }
    uint32_t* all = malloc(sizeof(uint32_t) * N);
    for (uint64_t i = 0; i < N; ++i) all[i] = (uint32_t)i;

    if (cfg->mode == ORC_ORACLE || cfg->mode == ORC_SPARSE) {
        orc_brute_knn(W, N, n, all, N, k_eff, threads, ids, dist);
        /* output stride is k_eff when clamped */
        for (uint64_t i = 0; i < N; ++i) prov[i] = cfg->mode == ORC_ORACLE ? 0 : 1;
        free(all);
        free(W);
        return 0;
    }

    const uint64_t pair_budget = 10 * N < cfg->eps_mean_cap ? 10 * N : cfg->eps_mean_cap;
    double eps_mean;
    orc_eps_mean(W, N, n, pair_budget, orc_derive_seed(cfg->seed, 1), &eps_mean);
    info->eps_mean = eps_mean;
    uint64_t* raw = calloc(cfg->n_bins, 8);
    uint64_t qc = 0;
    int rc = orc_histogram(W, N, n, eps_mean, cfg->n_bins, cfg->hist_frac,
                           orc_derive_seed(cfg->seed, 2), threads, raw, &qc);
    if (rc) {
        if (err) snprintf(err, errlen, "mean pairwise distance is not positive");
        free(raw);
        free(all);
        free(W);
        return rc;
    }
    info->hist_query_count = qc;
    info->bin_width = eps_mean / (double)cfg->n_bins;
    double* cum = malloc(sizeof(double) * cfg->n_bins);
    uint64_t running = 0;
    for (uint32_t b = 0; b < cfg->n_bins; ++b) {
        running += raw[b];
        cum[b] = (double)running / (double)qc;
        if (raw_hist) raw_hist[b] = raw[b];
    }
    double eb, ef, eb0, ef0;
    uint64_t bin, bin0;
    int fb = 0, fb0 = 0;
    orc_select_eps(cum, cfg->n_bins, info->bin_width, k_eff, cfg->beta, 1, &eb, &ef, &bin, &fb);
    orc_select_eps(cum, cfg->n_bins, info->bin_width, k_eff, 0.0, 1, &eb0, &ef0, &bin0, &fb0);
    info->eps_default = eb0;
    info->eps_beta = eb;
    info->eps_used = ef;
    info->eps_fallback = (uint32_t)fb;
    free(cum);
    free(raw);

    orc_grid g;
    rc = orc_grid_build(W, N, n, m, ef, &g, err, errlen);
    if (rc) {
        free(all);
        free(W);
        return rc;
    }
    info->n_min = orc_n_min(k_eff, m);
    info->n_thresh = orc_n_thresh(info->n_min, cfg->gamma);
    uint8_t* dense = malloc(N);
    uint64_t n_cpu = 0;
    for (uint64_t i = 0; i < N; ++i) {
        uint64_t pop = g.G[2 * g.slot[i] + 1] - g.G[2 * g.slot[i]];
        dense[i] = cfg->mode == ORC_DENSE || (double)pop >= info->n_thresh;
        n_cpu += !dense[i];
    }
    if (cfg->mode != ORC_DENSE) {
        uint64_t floor_cpu = (uint64_t)ceil(cfg->rho * (double)N);
        if (n_cpu < floor_cpu) {
            uint64_t need = floor_cpu - n_cpu, nd = N - n_cpu, w = 0;
            demote_t* ord = malloc(sizeof(demote_t) * (nd ? nd : 1));
            for (uint64_t i = 0; i < N; ++i)
                if (dense[i]) {
                    uint32_t s = g.slot[i];
                    ord[w].pop = g.G[2 * s + 1] - g.G[2 * s];
                    ord[w].cell = g.B[s];
                    ord[w].pid = (uint32_t)i;
                    ++w;
                }
            qsort(ord, nd, sizeof(demote_t), cmp_demote);
            if (need > nd) need = nd;
            for (uint64_t i = 0; i < need; ++i) dense[ord[i].pid] = 0;
            info->demoted = need;
            n_cpu += need;
            free(ord);
        }
    }
    info->q_cpu = n_cpu;
    info->q_gpu = N - n_cpu;

    uint64_t nd = N - n_cpu, w = 0;
    uint32_t* qd = malloc(sizeof(uint32_t) * (nd ? nd : 1));
    for (uint64_t i = 0; i < N; ++i)
        if (dense[i]) qd[w++] = (uint32_t)i;
    uint8_t* solved = calloc(nd ? nd : 1, 1);
    uint32_t* dids = malloc(sizeof(uint32_t) * (nd ? nd : 1) * k_eff);
    double* ddist = malloc(sizeof(double) * (nd ? nd : 1) * k_eff);
    uint64_t* cand = calloc(nd ? nd : 1, 8);
    dense_ctx dc = {W, n, k_eff, &g, ef, qd, solved, dids, ddist, cand};
    parallel_for(nd, threads, dense_task, &dc);

    /* everything not solved by the dense engine gets the exact KNN */
    uint64_t nrest = 0;
    uint32_t* rest = malloc(sizeof(uint32_t) * N);
    for (uint64_t i = 0, d = 0; i < N; ++i) {
        if (dense[i]) {
            info->candidates_examined += cand[d];
            if (solved[d]) {
                memcpy(ids + i * k_eff, dids + d * k_eff, sizeof(uint32_t) * k_eff);
                memcpy(dist + i * k_eff, ddist + d * k_eff, sizeof(double) * k_eff);
                prov[i] = 0;
            } else {
                prov[i] = 2;
                info->failed_count++;
                rest[nrest++] = (uint32_t)i;
            }
            ++d;
        } else {
            prov[i] = 1;
            rest[nrest++] = (uint32_t)i;
        }
    }
    if (nrest) {
        uint32_t* rids = malloc(sizeof(uint32_t) * nrest * k_eff);
        double* rdist = malloc(sizeof(double) * nrest * k_eff);
        orc_brute_knn(W, N, n, rest, nrest, k_eff, threads, rids, rdist);
        for (uint64_t r = 0; r < nrest; ++r) {
            memcpy(ids + (uint64_t)rest[r] * k_eff, rids + r * k_eff, sizeof(uint32_t) * k_eff);
            memcpy(dist + (uint64_t)rest[r] * k_eff, rdist + r * k_eff, sizeof(double) * k_eff);
        }
        free(rids);
        free(rdist);
    }
    free(rest);
    free(cand);
    free(dids);
    free(ddist);
    free(solved);
    free(qd);
    free(dense);
    orc_grid_free(&g);
    free(all);
    free(W);
    return 0;
}
