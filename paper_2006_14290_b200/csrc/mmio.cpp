// MatrixMarket coordinate ingestion / serialisation on the host (C++17,
// multi-threaded) — the data format that feeds the SpMV path
// (SURVEY.md §8(f) rank 3). Semantics of the reference reader/writer
// (warpkit/sparse.py:269-354):
//   * banner "%%MatrixMarket matrix coordinate <real|integer|pattern>
//     <general|symmetric>" (case-insensitive); other layouts, fields or
//     symmetries -> UnsupportedFormat, a malformed banner -> ParseError;
//   * blank lines and lines whose first non-blank character is '%' are
//     skipped anywhere after the banner; the first remaining line is
//     "nrows ncols nnz" (non-negative), then exactly nnz entry lines;
//   * an entry has exactly 2 (pattern) or 3 fields; 1-based indices inside
//     the declared shape; pattern entries get 1.0; values are parsed with
//     correct rounding (std::from_chars, as Python's float());
//   * symmetric files emit each off-diagonal entry followed by its mirror;
//   * duplicates are NOT summed here: the caller runs from_entries (host
//     lexsort or the device sort + segmented sum), exactly as the reference
//     parses into lists and then calls CooMatrix.from_entries.
// The entry lines are split into chunks at line boundaries and parsed by
// std::threads; the first error in file order is reported with its line
// number. Writer: "%%MatrixMarket matrix coordinate real general", the size
// line, then "r c v" with v printed as %.17g (round-trips every double).
#include <stdint.h>

#include <algorithm>
#include <charconv>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "../../include/wk_sparse.h"

namespace wk {
void set_error(const char* fmt, ...);
void clear_error();
}  // namespace wk

namespace {

// Python str.splitlines() terminators that are ASCII (\r\n counts once)
inline bool is_eol(char c) { return c == '\n' || c == '\r' || c == '\v' || c == '\f' || (c >= 0x1c && c <= 0x1e); }
// Python str.split() whitespace (ASCII)
inline bool is_ws(char c) { return c == ' ' || c == '\t' || is_eol(c) || c == 0x1f; }

struct Line {
    const char* b;
    const char* e;
};

// next line starting at p (< end); returns the position after its terminator
inline const char* next_line(const char* p, const char* end, Line& ln) {
    const char* q = p;
    while (q < end && !is_eol(*q)) ++q;
    ln.b = p;
    ln.e = q;
    if (q < end) {
        if (*q == '\r' && q + 1 < end && q[1] == '\n') return q + 2;
        return q + 1;
    }
    return q;
}

inline int split(const Line& ln, const char** tb, const char** te, int cap) {
    int n = 0;
    const char* p = ln.b;
    while (p < ln.e) {
        while (p < ln.e && is_ws(*p)) ++p;
        if (p >= ln.e) break;
        const char* s = p;
        while (p < ln.e && !is_ws(*p)) ++p;
        if (n < cap) {
            tb[n] = s;
            te[n] = p;
        }
        ++n;
    }
    return n;
}

inline bool blank_or_comment(const Line& ln) {
    const char* p = ln.b;
    while (p < ln.e && is_ws(*p)) ++p;
    return p >= ln.e || *p == '%';
}

inline bool parse_i64(const char* b, const char* e, int64_t& v) {
    if (b < e && *b == '+') ++b;
    if (b >= e || *b == '+' || (*b == '-' && (b + 1 >= e || b[1] == '+' || b[1] == '-'))) return false;
    auto r = std::from_chars(b, e, v);
    return r.ec == std::errc() && r.ptr == e;
}

inline bool parse_f64(const char* b, const char* e, double& v) {
    if (b < e && *b == '+') ++b;
    if (b >= e || *b == '+') return false;
    for (const char* p = b; p < e; ++p)
        if (*p == 'x' || *p == 'X') return false;  // no hex floats (Python float() rejects them)
    auto r = std::from_chars(b, e, v, std::chars_format::general);
    if (r.ec == std::errc::result_out_of_range) {
        // Python: overflow -> +-inf, underflow -> +-0.0 (correctly rounded); from_chars
        // reports the range error: fall back to strtod on a terminated copy
        std::string s(b, e);
        v = std::strtod(s.c_str(), nullptr);
        return true;
    }
    return r.ec == std::errc() && r.ptr == e;
}

inline std::string lower(const char* b, const char* e) {
    std::string s(b, e);
    for (auto& c : s) c = char(std::tolower(static_cast<unsigned char>(c)));
    return s;
}

struct ChunkOut {
    std::vector<int64_t> r, c;
    std::vector<double> v;
    int64_t entries = 0;   // entry lines seen
    int64_t lines = 0;     // physical lines in the chunk
    int64_t err_line = -1; // chunk-relative line of the first error
    int err_code = 0;
    std::string err;
};

void parse_chunk(const char* b, const char* e, const wk_mm_header* h, ChunkOut& out) {
    const bool pattern = h->field == WK_MM_PATTERN;
    const int want = pattern ? 2 : 3;
    const char* tb[4];
    const char* te[4];
    const char* p = b;
    out.r.reserve(size_t(std::max<int64_t>(0, (e - b) / 8)));
    while (p < e) {
        Line ln;
        p = next_line(p, e, ln);
        ++out.lines;
        if (blank_or_comment(ln)) continue;
        ++out.entries;
        if (out.err_code) continue;  // keep counting entries after the first error
        const int n = split(ln, tb, te, 4);
        auto fail = [&](const char* fmt, ...) {
            char buf[256];
            va_list ap;
            va_start(ap, fmt);
            vsnprintf(buf, sizeof buf, fmt, ap);
            va_end(ap);
            out.err = buf;
            out.err_code = WK_ERR_PARSE;
            out.err_line = out.lines;
        };
        if (n != want) {
            fail("expected %d fields, got %d", want, n);
            continue;
        }
        int64_t i, j;
        double v = 1.0;
        if (!parse_i64(tb[0], te[0], i) || !parse_i64(tb[1], te[1], j) || (!pattern && !parse_f64(tb[2], te[2], v))) {
            fail("invalid literal");
            continue;
        }
        if (!(1 <= i && i <= h->nrows && 1 <= j && j <= h->ncols)) {
            fail("entry (%lld, %lld) outside %lldx%lld", (long long)i, (long long)j, (long long)h->nrows,
                 (long long)h->ncols);
            continue;
        }
        out.r.push_back(i - 1);
        out.c.push_back(j - 1);
        out.v.push_back(v);
        if (h->symmetric && i != j) {
            out.r.push_back(j - 1);
            out.c.push_back(i - 1);
            out.v.push_back(v);
        }
    }
}

}  // namespace

extern "C" {

int wk_mm_read_header(const char* data, int64_t len, wk_mm_header* h) {
    wk::clear_error();
    std::memset(h, 0, sizeof(*h));
    for (int64_t k = 0; k < len; ++k)
        if (static_cast<unsigned char>(data[k]) > 0x7f) {
            wk::set_error("MatrixMarket files must be ASCII (byte 0x%02x at offset %lld)",
                          unsigned(static_cast<unsigned char>(data[k])), (long long)k);
            return WK_ERR_PARSE;
        }
    const char* p = data;
    const char* end = data + len;
    if (len == 0) {
        wk::set_error("empty MatrixMarket stream");
        return WK_ERR_PARSE;
    }
    Line ln;
    p = next_line(p, end, ln);
    const char* tb[8];
    const char* te[8];
    const int n = split(ln, tb, te, 8);
    if (n != 5 || lower(tb[0], te[0]) != "%%matrixmarket" || lower(tb[1], te[1]) != "matrix") {
        wk::set_error("malformed MatrixMarket banner: '%.*s'", int(std::min<ptrdiff_t>(ln.e - ln.b, 120)), ln.b);
        return WK_ERR_PARSE;
    }
    const std::string layout = lower(tb[2], te[2]), field = lower(tb[3], te[3]), sym = lower(tb[4], te[4]);
    if (layout != "coordinate") {
        wk::set_error("only coordinate layout is supported, got '%s'", layout.c_str());
        return WK_ERR_UNSUPPORTED;
    }
    if (field == "real")
        h->field = WK_MM_REAL;
    else if (field == "integer")
        h->field = WK_MM_INTEGER;
    else if (field == "pattern")
        h->field = WK_MM_PATTERN;
    else {
        wk::set_error("unsupported field '%s' (complex files are not supported)", field.c_str());
        return WK_ERR_UNSUPPORTED;
    }
    if (sym == "general")
        h->symmetric = 0;
    else if (sym == "symmetric")
        h->symmetric = 1;
    else {
        wk::set_error("unsupported symmetry '%s'", sym.c_str());
        return WK_ERR_UNSUPPORTED;
    }
    int64_t line_no = 1;
    while (p < end) {
        p = next_line(p, end, ln);
        ++line_no;
        if (blank_or_comment(ln)) continue;
        const int k = split(ln, tb, te, 8);
        if (k != 3) {
            wk::set_error("line %lld: size line must be 'nrows ncols nnz'", (long long)line_no);
            return WK_ERR_PARSE;
        }
        if (!parse_i64(tb[0], te[0], h->nrows) || !parse_i64(tb[1], te[1], h->ncols) ||
            !parse_i64(tb[2], te[2], h->nnz)) {
            wk::set_error("line %lld: invalid size literal", (long long)line_no);
            return WK_ERR_PARSE;
        }
        if (h->nrows < 0 || h->ncols < 0 || h->nnz < 0) {
            wk::set_error("line %lld: negative size", (long long)line_no);
            return WK_ERR_PARSE;
        }
        h->body_offset = p - data;
        h->body_line = line_no;
        return 0;
    }
    wk::set_error("missing size line");
    return WK_ERR_PARSE;
}

int wk_mm_parse_entries(const char* data, int64_t len, const wk_mm_header* h, int32_t nthreads, int64_t* rows,
                        int64_t* cols, double* vals, int64_t capacity, int64_t* count) {
    wk::clear_error();
    const char* b = data + h->body_offset;
    const char* e = data + len;
    int T = nthreads > 0 ? nthreads : int(std::thread::hardware_concurrency());
    if (T < 1) T = 1;
    const int64_t body = e - b;
    if (body < (int64_t(1) << 20)) T = 1;  // small files: one pass
    // chunk boundaries just after a line terminator (a \r\n pair is never split)
    std::vector<const char*> cut(size_t(T) + 1);
    cut[0] = b;
    cut[T] = e;
    for (int t = 1; t < T; ++t) {
        const char* q = b + body * t / T;
        if (q < cut[t - 1]) q = cut[t - 1];
        while (q < e && !is_eol(q[-1])) ++q;
        while (q < e && q[-1] == '\r' && *q == '\n') ++q;
        cut[t] = q;
    }
    std::vector<ChunkOut> out(static_cast<size_t>(T));
    std::vector<std::thread> th;
    for (int t = 1; t < T; ++t) th.emplace_back(parse_chunk, cut[t], cut[t + 1], h, std::ref(out[t]));
    parse_chunk(cut[0], cut[1], h, out[0]);
    for (auto& x : th) x.join();
    int64_t entries = 0, produced = 0;
    for (auto& o : out) {
        entries += o.entries;
        produced += int64_t(o.r.size());
    }
    if (entries != h->nnz) {
        wk::set_error("expected %lld entries, found %lld", (long long)h->nnz, (long long)entries);
        return WK_ERR_PARSE;
    }
    int64_t line_base = h->body_line;
    for (auto& o : out) {
        if (o.err_code) {
            wk::set_error("line %lld: %s", (long long)(line_base + o.err_line), o.err.c_str());
            return o.err_code;
        }
        line_base += o.lines;
    }
    if (produced > capacity) {
        wk::set_error("output capacity %lld < %lld entries", (long long)capacity, (long long)produced);
        return WK_ERR_INVALID;
    }
    int64_t off = 0;
    for (auto& o : out) {
        const size_t k = o.r.size();
        if (k) {
            std::memcpy(rows + off, o.r.data(), k * sizeof(int64_t));
            std::memcpy(cols + off, o.c.data(), k * sizeof(int64_t));
            std::memcpy(vals + off, o.v.data(), k * sizeof(double));
        }
        off += int64_t(k);
    }
    *count = off;
    return 0;
}

// Serialise as 'coordinate real general' with %.17g values (sparse.py:338-353).
// out == nullptr: *written = the exact byte count needed.
int wk_mm_write(int64_t nrows, int64_t ncols, int64_t nnz, const int64_t* rows, const int64_t* cols,
                const double* vals, char* out, int64_t capacity, int64_t* written) {
    wk::clear_error();
    char line[96];
    int64_t total = 0;
    auto put = [&](const char* s, int n) {
        if (out != nullptr && total + n <= capacity) std::memcpy(out + total, s, size_t(n));
        total += n;
    };
    int n = snprintf(line, sizeof line, "%%%%MatrixMarket matrix coordinate real general\n");
    put(line, n);
    n = snprintf(line, sizeof line, "%lld %lld %lld\n", (long long)nrows, (long long)ncols, (long long)nnz);
    put(line, n);
    for (int64_t k = 0; k < nnz; ++k) {
        n = snprintf(line, sizeof line, "%lld %lld %.17g\n", (long long)(rows[k] + 1), (long long)(cols[k] + 1),
                     vals[k]);
        put(line, n);
    }
    *written = total;
    if (out != nullptr && total > capacity) {
        wk::set_error("output capacity %lld < %lld bytes", (long long)capacity, (long long)total);
        return WK_ERR_INVALID;
    }
    return 0;
}

}  // extern "C"
