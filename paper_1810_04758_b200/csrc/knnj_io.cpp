// Host I/O around the join: the reference's
// result TSV at multi-core speed and binary-f64 dataset ingest.
//
//   * TSV: "%u\t%u\t%.17g\n" per (query, rank), exactly io::tsv_string
//     (proj/src/io.cpp:141-154 with append_double :93-97). std::to_chars with
//     chars_format::general and precision 17 is specified as printf("%.17g") in
//     the C locale, so the bytes are identical; rows are formatted by a thread
//     pool in contiguous chunks and written with pwrite at their prefix offsets.
//   * binary-f64 ingest: ingest_binary (proj/src/io.cpp:69-91): LE u64 |D|, u64 n,
//     |D|*n row-major doubles, same validation and messages. The file is mmapped and
//     copied into the caller's buffer (a pinned one from knnj_alloc_pinned feeds the
//     H2D at full PCIe rate) by a thread pool that also checks finiteness; the first
//     non-finite value in file order is the one reported.
//   * CSV/TSV ingest: ingest_text (proj/src/io.cpp:24-67) over an mmapped file cut into
//     per-thread chunks at line boundaries; fields are parsed with std::from_chars (the
//     reference's parser, same libstdc++), and the first error in file order is reported
//     with the reference's row/column message.
#include <fcntl.h>
#include <sys/mman.h>
#include <sys/stat.h>
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

// read-only mapping of a whole file (size 0: no mapping)
struct Mapped {
    int fd = -1;
    const char* p = nullptr;
    uint64_t size = 0;
    bool open(const char* path) {
        fd = ::open(path, O_RDONLY);
        if (fd < 0) return false;
        struct stat st;
        if (::fstat(fd, &st) != 0) return false;
        size = (uint64_t)st.st_size;
        if (size) {
            void* m = ::mmap(nullptr, size, PROT_READ, MAP_PRIVATE, fd, 0);
            if (m == MAP_FAILED) return false;
            ::madvise(m, size, MADV_SEQUENTIAL);
            p = static_cast<const char*>(m);
        }
        return true;
    }
    ~Mapped() {
        if (p) ::munmap(const_cast<char*>(p), size);
        if (fd >= 0) ::close(fd);
    }
};

template <class F>
void parallel_chunks(unsigned nt, F&& f) {
    std::vector<std::thread> pool;
    for (unsigned t = 1; t < nt; ++t) pool.emplace_back(f, t);
    f(0u);
    for (auto& th : pool) th.join();
}

// ---- ingest_text (proj/src/io.cpp:24-67), one chunk of whole lines
struct TextChunk {
    std::vector<double> coords;
    uint64_t lines = 0;          // std::getline lines in the chunk (empty ones included)
    uint64_t first_row = 0;      // local 1-based row of the first non-empty line (0: none)
    uint64_t first_cols = 0;     // its column count (0 if it failed to parse)
    // first error in the chunk: kind 1 not a number, 2 non-finite, 3 column count
    int err = 0;
    uint64_t err_row = 0, err_col = 0;
    std::string err_field;
};

void parse_text_chunk(const char* b, const char* e, char sep, TextChunk& out) {
    uint64_t row = 0, dims = 0;
    const char* at_line = b;
    while (at_line < e) {
        const char* nl = static_cast<const char*>(std::memchr(at_line, '\n', e - at_line));
        const char* lend = nl ? nl : e;
        const char* next = nl ? nl + 1 : e;
        ++row;
        const char* ls = at_line;
        at_line = next;
        if (lend == ls) continue;            // line.empty(): skipped before the '\r' strip
        if (lend[-1] == '\r') --lend;
        const uint64_t len = (uint64_t)(lend - ls);
        uint64_t col = 0, at = 0;
        while (at <= len) {
            const char* sp = static_cast<const char*>(std::memchr(ls + at, sep, len - at));
            const uint64_t end = sp ? (uint64_t)(sp - ls) : len;
            ++col;
            const char* first = ls + at;
            const char* last = ls + end;
            while (first < last && (*first == ' ' || *first == '\t')) ++first;
            double v = 0;
            auto [p, ec] = std::from_chars(first, last, v);
            while (p < last && (*p == ' ' || *p == '\t')) ++p;
            if (ec != std::errc() || p != last) {
                out.err = 1;
                out.err_row = row;
                out.err_col = col;
                out.err_field.assign(ls + at, ls + end);
                out.lines = row;
                return;
            }
            if (!std::isfinite(v)) {
                out.err = 2;
                out.err_row = row;
                out.err_col = col;
                out.lines = row;
                return;
            }
            out.coords.push_back(v);
            if (end == len) break;
            at = end + 1;
        }
        if (dims == 0) {
            dims = col;
            out.first_row = row;
            out.first_cols = col;
        } else if (col != dims) {
            out.err = 3;
            out.err_row = row;
            out.err_col = col;
            out.lines = row;
            return;
        }
    }
    out.lines = row;
}

}  // namespace

struct knnj_text {
    std::vector<TextChunk> chunks;
    uint64_t n_points = 0, dims = 0;
};

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
    Mapped f;
    if (!f.open(path)) return fail(KNNJ_E_INGEST, std::string("cannot open ") + path);
    if (f.size < 16 || (f.size - 16) / 8 < count)
        return fail(KNNJ_E_INGEST, std::string(path) + ": body shorter than header promises (" +
                                       std::to_string(size) + " x " + std::to_string(dims) + ")");
    const char* body = f.p + 16;
    // chunks of >= 8 MiB: copy + finiteness check per thread; the smallest bad index wins
    const unsigned nt = (unsigned)std::max<uint64_t>(
        1, std::min<uint64_t>(std::max(1u, std::thread::hardware_concurrency()), count / (1u << 20) + 1));
    std::vector<uint64_t> bad(nt, UINT64_MAX);
    parallel_chunks(nt, [&](unsigned t) {
        const uint64_t b = count * t / nt, e = count * (t + 1) / nt;
        std::memcpy(out + b, body + 8 * b, 8 * (e - b));
        for (uint64_t i = b; i < e; ++i)
            if (!std::isfinite(out[i])) {
                bad[t] = i;
                break;
            }
    });
    for (uint64_t i : bad)
        if (i != UINT64_MAX)
            return fail(KNNJ_E_INGEST, std::string(path) + ": row " + std::to_string(i / dims + 1) +
                                           ", column " + std::to_string(i % dims + 1) +
                                           ": non-finite value");
    return KNNJ_OK;
}

int knnj_text_parse(const char* path, char sep, uint32_t threads, knnj_text** out,
                    uint64_t* n_points, uint64_t* dims) {
    if (!path || !out || !n_points || !dims) return fail(KNNJ_E_USAGE, "null argument");
    *out = nullptr;
    Mapped f;
    if (!f.open(path)) return fail(KNNJ_E_INGEST, std::string("cannot open ") + path);
    const std::string ps(path);
    unsigned nt = threads ? threads : std::max(1u, std::thread::hardware_concurrency());
    nt = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>(nt, f.size / (1u << 20) + 1));
    // chunk starts: just after the first '\n' at or past an even byte split
    std::vector<uint64_t> cut(nt + 1, f.size);
    cut[0] = 0;
    for (unsigned t = 1; t < nt; ++t) {
        uint64_t c = std::max(cut[t - 1], f.size * t / nt);
        if (c > 0 && c < f.size) {
            const void* nl = std::memchr(f.p + c - 1, '\n', f.size - (c - 1));
            c = nl ? (uint64_t)(static_cast<const char*>(nl) - f.p) + 1 : f.size;
        }
        cut[t] = c;
    }
    auto* T = new knnj_text;
    T->chunks.resize(nt);
    parallel_chunks(nt, [&](unsigned t) {
        if (cut[t] < cut[t + 1]) parse_text_chunk(f.p + cut[t], f.p + cut[t + 1], sep, T->chunks[t]);
    });
    // merge in file order: the first error the reference's sequential loop would meet
    uint64_t base = 0, gdims = 0, total = 0;
    for (const TextChunk& c : T->chunks) {
        std::string msg;
        if (c.first_row && gdims && c.first_cols != gdims &&
            !(c.err && c.err_row == c.first_row)) {
            msg = ps + ": row " + std::to_string(base + c.first_row) + " has " +
                  std::to_string(c.first_cols) + " columns, expected " + std::to_string(gdims);
        } else if (c.err == 1) {
            msg = ps + ": row " + std::to_string(base + c.err_row) + ", column " +
                  std::to_string(c.err_col) + ": not a number: '" + c.err_field + "'";
        } else if (c.err == 2) {
            msg = ps + ": row " + std::to_string(base + c.err_row) + ", column " +
                  std::to_string(c.err_col) + ": non-finite value";
        } else if (c.err == 3) {
            msg = ps + ": row " + std::to_string(base + c.err_row) + " has " +
                  std::to_string(c.err_col) + " columns, expected " +
                  std::to_string(gdims ? gdims : c.first_cols);
        }
        if (!msg.empty()) {
            delete T;
            return fail(KNNJ_E_INGEST, msg);
        }
        if (!gdims && c.first_row) gdims = c.first_cols;
        base += c.lines;
        total += c.coords.size();
    }
    if (!total) {
        delete T;
        return fail(KNNJ_E_INGEST, ps + ": no points");
    }
    T->dims = gdims;
    T->n_points = total / gdims;
    *n_points = T->n_points;
    *dims = T->dims;
    *out = T;
    return KNNJ_OK;
}

int knnj_text_copy(const knnj_text* t, double* out, uint64_t capacity_doubles) {
    if (!t || !out) return fail(KNNJ_E_USAGE, "null argument");
    if (capacity_doubles < t->n_points * t->dims)
        return fail(KNNJ_E_USAGE, "output buffer smaller than the dataset");
    std::vector<uint64_t> off(t->chunks.size() + 1, 0);
    for (size_t i = 0; i < t->chunks.size(); ++i) off[i + 1] = off[i] + t->chunks[i].coords.size();
    parallel_chunks((unsigned)t->chunks.size(), [&](unsigned i) {
        const auto& c = t->chunks[i].coords;
        if (!c.empty()) std::memcpy(out + off[i], c.data(), 8 * c.size());
    });
    return KNNJ_OK;
}

void knnj_text_free(knnj_text* t) { delete t; }

}  // extern "C"
