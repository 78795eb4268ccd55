// Host I/O around the join: the reference's
// result TSV at multi-core speed and binary-f64 dataset ingest.
//
//   * TSV: "%u\t%u\t%.17g\n" per (query, rank), exactly io::tsv_string
//     (proj/src/io.cpp:141-154 with append_double :93-97). std::to_chars with
//     chars_format::general and precision 17 is specified as printf("%.17g") in
//     the C locale, so the bytes are identical; rows are formatted by a thread
//     pool in contiguous chunks and written with pwrite at their prefix offsets.
//   * binary-f64 ingest: ingest_binary (proj/src/io.cpp:69-91): LE u64 |D|, u64 n,
//     |D|*n row-major doubles, same validation and messages; the body can be
//     read straight into a pinned buffer (knnj_alloc_pinned) for the H2D.
#include <fcntl.h>
#include <unistd.h>

#include <algorithm>
#include <charconv>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "knnj_c.h"

namespace {

thread_local std::string g_io_err;

int fail(int code, const std::string& msg) {
    g_io_err = msg;
    return code;
}

// rows [r0, r1) of the result as TSV text
void format_rows(const uint32_t* queries, const uint32_t* ids, const double* dist, uint32_t k,
                 uint64_t r0, uint64_t r1, std::string& out) {
    out.clear();
    out.reserve((r1 - r0) * k * 32);
    char buf[64];
    for (uint64_t r = r0; r < r1; ++r) {
        char qb[16];
        const uint32_t q = queries ? queries[r] : (uint32_t)r;
        const auto qe = std::to_chars(qb, qb + sizeof qb, q).ptr;
        for (uint32_t j = 0; j < k; ++j) {
            char* p = buf;
            std::memcpy(p, qb, qe - qb);
            p += qe - qb;
            *p++ = '\t';
            p = std::to_chars(p, buf + sizeof buf, ids[r * k + j]).ptr;
            *p++ = '\t';
            p = std::to_chars(p, buf + sizeof buf, dist[r * k + j], std::chars_format::general, 17).ptr;
            *p++ = '\n';
            out.append(buf, p - buf);
        }
    }
}

unsigned pick_threads(unsigned threads, uint64_t rows) {
    unsigned t = threads ? threads : std::max(1u, std::thread::hardware_concurrency());
    return (unsigned)std::max<uint64_t>(1, std::min<uint64_t>(t, rows / 256 + 1));
}

}  // namespace

extern "C" {

const char* knnj_io_last_error(void) { return g_io_err.c_str(); }

int knnj_tsv_format(const uint32_t* queries, const uint32_t* ids, const double* dist,
                    uint64_t n_rows, uint32_t k, char* out, uint64_t capacity, uint64_t* length,
                    uint32_t threads) {
    if (!length || (n_rows && k && (!ids || !dist))) return fail(KNNJ_E_USAGE, "null argument");
    const unsigned nt = pick_threads(threads, n_rows);
    std::vector<std::string> parts(nt);
    std::vector<std::thread> pool;
    for (unsigned t = 0; t < nt; ++t)
        pool.emplace_back([&, t] {
            format_rows(queries, ids, dist, k, n_rows * t / nt, n_rows * (t + 1) / nt, parts[t]);
        });
    for (auto& th : pool) th.join();
    uint64_t total = 0;
    for (auto& p : parts) total += p.size();
    *length = total;
    if (!out) return KNNJ_OK;  // size query
    if (capacity < total) return fail(KNNJ_E_USAGE, "output buffer too small for the TSV text");
    uint64_t at = 0;
    for (auto& p : parts) {
        std::memcpy(out + at, p.data(), p.size());
        at += p.size();
    }
    return KNNJ_OK;
}

int knnj_tsv_write(const char* path, const uint32_t* queries, const uint32_t* ids,
                   const double* dist, uint64_t n_rows, uint32_t k, uint32_t threads,
                   uint64_t* bytes_written) {
    if (!path || (n_rows && k && (!ids || !dist))) return fail(KNNJ_E_USAGE, "null argument");
    const int fd = ::open(path, O_CREAT | O_TRUNC | O_WRONLY, 0644);
    if (fd < 0) return fail(KNNJ_E_INGEST, std::string("cannot write ") + path);
    // chunks of ~64k rows: formatted in parallel, written in order at prefix offsets
    const uint64_t chunk = 65536;
    const uint64_t nchunks = (n_rows + chunk - 1) / chunk;
    const unsigned nt = pick_threads(threads, n_rows);
    uint64_t total = 0;
    int rc = KNNJ_OK;
    for (uint64_t c0 = 0; c0 < nchunks && rc == KNNJ_OK; c0 += nt) {
        const unsigned nc = (unsigned)std::min<uint64_t>(nt, nchunks - c0);
        std::vector<std::string> parts(nc);
        std::vector<std::thread> pool;
        for (unsigned t = 0; t < nc; ++t)
            pool.emplace_back([&, t] {
                const uint64_t r0 = (c0 + t) * chunk, r1 = std::min(n_rows, r0 + chunk);
                format_rows(queries, ids, dist, k, r0, r1, parts[t]);
            });
        for (auto& th : pool) th.join();
        std::vector<uint64_t> off(nc + 1, total);
        for (unsigned t = 0; t < nc; ++t) off[t + 1] = off[t] + parts[t].size();
        pool.clear();
        std::vector<int> ok(nc, 1);
        for (unsigned t = 0; t < nc; ++t)
            pool.emplace_back([&, t] {
                const char* p = parts[t].data();
                uint64_t left = parts[t].size(), o = off[t];
                while (left) {
                    const ssize_t w = ::pwrite(fd, p, left, (off_t)o);
                    if (w <= 0) {
                        ok[t] = 0;
                        return;
                    }
                    p += w;
                    o += (uint64_t)w;
                    left -= (uint64_t)w;
                }
            });
        for (auto& th : pool) th.join();
        for (int v : ok)
            if (!v) rc = fail(KNNJ_E_INGEST, std::string("short write to ") + path);
        total = off[nc];
    }
    ::close(fd);
    if (bytes_written) *bytes_written = total;
    return rc;
}

int knnj_binary_header(const char* path, uint64_t* n_points, uint64_t* dims) {
    if (!path || !n_points || !dims) return fail(KNNJ_E_USAGE, "null argument");
    FILE* f = std::fopen(path, "rb");
    if (!f) return fail(KNNJ_E_INGEST, std::string("cannot open ") + path);
    uint64_t h[2] = {0, 0};
    const size_t got = std::fread(h, 8, 2, f);
    std::fclose(f);
    if (got != 2) return fail(KNNJ_E_INGEST, std::string(path) + ": truncated header");
    if (h[0] == 0 || h[1] == 0) return fail(KNNJ_E_INGEST, std::string(path) + ": empty dataset in header");
    *n_points = h[0];
    *dims = h[1];
    return KNNJ_OK;
}

int knnj_binary_read(const char* path, double* out, uint64_t capacity_doubles) {
    uint64_t size = 0, dims = 0;
    int rc = knnj_binary_header(path, &size, &dims);
    if (rc) return rc;
    if (!out) return fail(KNNJ_E_USAGE, "null output buffer");
    const uint64_t count = size * dims;
    if (capacity_doubles < count) return fail(KNNJ_E_USAGE, "output buffer smaller than the dataset");
    FILE* f = std::fopen(path, "rb");
    if (!f) return fail(KNNJ_E_INGEST, std::string("cannot open ") + path);
    std::fseek(f, 16, SEEK_SET);
    const size_t got = std::fread(out, 8, count, f);
    std::fclose(f);
    if (got != count)
        return fail(KNNJ_E_INGEST, std::string(path) + ": body shorter than header promises (" +
                                       std::to_string(size) + " x " + std::to_string(dims) + ")");
    for (uint64_t i = 0; i < count; ++i)
        if (!std::isfinite(out[i]))
            return fail(KNNJ_E_INGEST, std::string(path) + ": row " + std::to_string(i / dims + 1) +
                                           ", column " + std::to_string(i % dims + 1) +
                                           ": non-finite value");
    return KNNJ_OK;
}

}  // extern "C"
