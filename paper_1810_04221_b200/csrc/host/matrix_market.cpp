// matrix_market.cpp — MatrixMarket coordinate I/O of the matchamg API
// (reference: proj/src/matrix_market.cpp). Same grammar, error texts and
// results; built for large inputs (the step before
// setup): the file is mapped, the body is cut at line boundaries and parsed
// on every host thread (std::from_chars: correctly rounded, the same double
// as the reference's istream extraction), and the CSR is assembled by a
// parallel row bucketing + per-row column sort. Duplicate (i, j) entries are
// summed by the reference's own from_triplets order (std::sort of the
// file-order triplets), so even their floating-point sums are identical.
#include "matchamg/matrix_market.hpp"

#include <fcntl.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <atomic>
#include <cctype>
#include <charconv>
#include <cstdio>
#include <cstring>
#include <sstream>
#include <stdexcept>
#include <thread>
#include <vector>

namespace matchamg {
namespace {

std::string lower(std::string s) {
    std::transform(s.begin(), s.end(), s.begin(), [](unsigned char c) { return std::tolower(c); });
    return s;
}

[[noreturn]] void fail(const std::string& path, long line, const std::string& what) {
    throw std::runtime_error(path + ":" + std::to_string(line) + ": " + what);
}

struct Mapped {
    const char* p = nullptr;
    size_t n = 0;
    int fd = -1;
    ~Mapped() {
        if (p && n) munmap(const_cast<char*>(p), n);
        if (fd >= 0) close(fd);
    }
};

int nthreads() { return static_cast<int>(std::max(1u, std::thread::hardware_concurrency())); }

inline bool is_space(char c) { return c == ' ' || c == '\t' || c == '\r' || c == '\v' || c == '\f'; }

// istream-compatible integer token: optional sign, digits
inline bool parse_int(const char*& s, const char* e, index_t& out) {
    while (s < e && is_space(*s)) ++s;
    if (s >= e) return false;
    const char* t = s;
    if (*t == '+') ++t;
    auto r = std::from_chars(t, e, out);
    if (r.ec != std::errc() || r.ptr == t) return false;
    s = r.ptr;
    return true;
}

// istream-compatible double token; 0 = ok, 1 = malformed, 2 = unusual form
// (inf/nan/hex: the caller re-parses the line with std::istringstream)
inline int parse_double(const char*& s, const char* e, double& out) {
    while (s < e && is_space(*s)) ++s;
    if (s >= e) return 1;
    const char* t = s;
    if (*t == '+') ++t;
    if (t < e && (*t == 'i' || *t == 'I' || *t == 'n' || *t == 'N')) return 2;
    if (t + 1 < e && t[0] == '0' && (t[1] == 'x' || t[1] == 'X')) return 2;
    auto r = std::from_chars(t, e, out);
    if (r.ec != std::errc() || r.ptr == t) return 1;
    s = r.ptr;
    return 0;
}

struct Entry {
    index_t i, j;
    double v;
};

struct Chunk {
    std::vector<Entry> ent; // file order (1-based indices as read)
    long lines = 0;         // lines in this chunk
    long err_line = -1;     // first bad line (chunk-local, 1-based)
    std::string err;
};

// pattern symmetry on the host (csr.cpp:106-112 semantics) — I/O must not
// need the device
bool host_symmetric_pattern(const CsrMatrix& A) {
    if (A.nrows != A.ncols) return false;
    const int T = static_cast<int>(std::min<index_t>(nthreads(), std::max<index_t>(1, A.nrows / 4096)));
    std::atomic<bool> ok{true};
    auto chk = [&](int t) {
        for (index_t i = A.nrows * t / T; i < A.nrows * (t + 1) / T && ok; ++i)
            for (index_t k = A.row_begin(i); k < A.row_end(i); ++k) {
                const index_t j = A.col_idx[k];
                const auto b = A.col_idx.begin() + A.row_begin(j), e = A.col_idx.begin() + A.row_end(j);
                if (!std::binary_search(b, e, i)) {
                    ok = false;
                    return;
                }
            }
    };
    std::vector<std::thread> th;
    for (int t = 1; t < T; ++t) th.emplace_back(chk, t);
    chk(0);
    for (auto& x : th) x.join();
    return ok;
}

} // namespace

CsrMatrix read_matrix_market(const std::string& path) {
    Mapped m;
    m.fd = open(path.c_str(), O_RDONLY);
    if (m.fd < 0) throw std::runtime_error("cannot open matrix file: " + path);
    struct stat st;
    if (fstat(m.fd, &st) != 0) throw std::runtime_error("cannot open matrix file: " + path);
    m.n = static_cast<size_t>(st.st_size);
    if (m.n == 0) fail(path, 1, "empty file");
    void* addr = mmap(nullptr, m.n, PROT_READ, MAP_PRIVATE, m.fd, 0);
    if (addr == MAP_FAILED) throw std::runtime_error("cannot open matrix file: " + path);
    m.p = static_cast<const char*>(addr);
    madvise(addr, m.n, MADV_SEQUENTIAL);
    const char* const end = m.p + m.n;

    auto next_line = [&](const char*& at, std::string& line) -> bool {
        if (at >= end) return false;
        const char* nl = static_cast<const char*>(std::memchr(at, '\n', static_cast<size_t>(end - at)));
        const char* le = nl ? nl : end;
        line.assign(at, le);
        at = nl ? nl + 1 : end;
        return true;
    };

    // banner and size line, sequentially (reference matrix_market.cpp:27-66)
    const char* at = m.p;
    long line_no = 0;
    std::string line;
    if (!next_line(at, line)) fail(path, 1, "empty file");
    ++line_no;
    std::istringstream banner(line);
    std::string tag, object, format, field, qualifier;
    banner >> tag >> object >> format >> field >> qualifier;
    if (lower(tag) != "%%matrixmarket") fail(path, line_no, "missing %%MatrixMarket banner");
    if (lower(object) != "matrix" || lower(format) != "coordinate")
        fail(path, line_no, "only `matrix coordinate` files are supported");
    if (lower(field) != "real") fail(path, line_no, "unsupported field `" + field + "` (want real)");
    const std::string sym = lower(qualifier);
    if (sym != "general" && sym != "symmetric")
        fail(path, line_no, "unsupported qualifier `" + qualifier + "` (want general or symmetric)");
    const bool symmetric = sym == "symmetric";

    index_t nrows = 0, ncols = 0;
    long declared_nnz = -1;
    while (next_line(at, line)) {
        ++line_no;
        if (line.empty() || line[0] == '%') continue;
        std::istringstream sizes(line);
        if (!(sizes >> nrows >> ncols >> declared_nnz)) fail(path, line_no, "malformed size line");
        break;
    }
    if (declared_nnz < 0) fail(path, line_no, "missing size line");
    if (nrows < 0 || ncols < 0) fail(path, line_no, "negative matrix dimension");

    // body: T chunks cut at line starts, parsed in parallel
    const size_t body = static_cast<size_t>(at - m.p);
    const int T = static_cast<int>(std::min<size_t>(nthreads(), std::max<size_t>(1, (m.n - body) >> 20)));
    std::vector<const char*> cut(T + 1);
    cut[0] = at;
    cut[T] = end;
    for (int t = 1; t < T; ++t) {
        const char* c = m.p + body + (m.n - body) * t / T;
        if (c < cut[t - 1]) c = cut[t - 1];
        const char* nl = static_cast<const char*>(std::memchr(c, '\n', static_cast<size_t>(end - c)));
        cut[t] = nl ? nl + 1 : end;
    }
    std::vector<Chunk> ch(T);
    auto parse = [&](int t) {
        Chunk& C = ch[t];
        C.ent.reserve(static_cast<size_t>(cut[t + 1] - cut[t]) / 24 + 16);
        const char* s = cut[t];
        const char* e = cut[t + 1];
        while (s < e) {
            const char* nl = static_cast<const char*>(std::memchr(s, '\n', static_cast<size_t>(e - s)));
            const char* le = nl ? nl : e;
            ++C.lines;
            if (le > s && *s != '%') {
                Entry x{};
                const char* q = s;
                int dk = 1;
                const bool ok = parse_int(q, le, x.i) && parse_int(q, le, x.j) &&
                                (dk = parse_double(q, le, x.v)) == 0;
                if (!ok && dk == 2) { // unusual number form: the reference's own extraction
                    std::istringstream entry(std::string(s, le));
                    if (!(entry >> x.i >> x.j >> x.v)) dk = 1;
                    else dk = 0;
                }
                if (!ok && dk != 0) {
                    C.err_line = C.lines;
                    C.err = "malformed entry line";
                    return;
                }
                if (x.i < 1 || x.i > nrows || x.j < 1 || x.j > ncols) {
                    C.err_line = C.lines;
                    C.err = "index (" + std::to_string(x.i) + ", " + std::to_string(x.j) +
                            ") outside " + std::to_string(nrows) + "x" + std::to_string(ncols);
                    return;
                }
                C.ent.push_back(x);
            }
            s = nl ? nl + 1 : e;
        }
    };
    {
        std::vector<std::thread> th;
        for (int t = 1; t < T; ++t) th.emplace_back(parse, t);
        parse(0);
        for (auto& x : th) x.join();
    }
    long seen = 0;
    for (int t = 0; t < T; ++t) {
        if (ch[t].err_line >= 0) fail(path, line_no + ch[t].err_line, ch[t].err);
        line_no += ch[t].lines;
        seen += static_cast<long>(ch[t].ent.size());
    }
    if (seen != declared_nnz)
        fail(path, line_no,
             "entry count " + std::to_string(seen) + " does not match header (" +
                 std::to_string(declared_nnz) + ")");

    // CSR: count per row, bucket, sort each row by column
    std::vector<std::atomic<index_t>> cnt(static_cast<size_t>(nrows) + 1);
    for (auto& c : cnt) c.store(0, std::memory_order_relaxed);
    auto count = [&](int t) {
        for (const Entry& x : ch[t].ent) {
            cnt[x.i].fetch_add(1, std::memory_order_relaxed);
            if (symmetric && x.i != x.j) cnt[x.j].fetch_add(1, std::memory_order_relaxed);
        }
    };
    auto run = [&](auto&& f, int n) {
        std::vector<std::thread> th;
        for (int t = 1; t < n; ++t) th.emplace_back(f, t);
        f(0);
        for (auto& x : th) x.join();
    };
    run(count, T);
    CsrMatrix A;
    A.nrows = nrows;
    A.ncols = ncols;
    A.row_ptr.assign(static_cast<size_t>(nrows) + 1, 0);
    for (index_t r = 0; r < nrows; ++r) A.row_ptr[r + 1] = A.row_ptr[r] + cnt[r + 1].load();
    const index_t total = A.row_ptr[nrows];
    A.col_idx.resize(static_cast<size_t>(total));
    A.values.resize(static_cast<size_t>(total));
    std::vector<std::atomic<index_t>> pos(static_cast<size_t>(nrows));
    for (index_t r = 0; r < nrows; ++r) pos[r].store(A.row_ptr[r], std::memory_order_relaxed);
    auto scatter = [&](int t) {
        for (const Entry& x : ch[t].ent) {
            index_t k = pos[x.i - 1].fetch_add(1, std::memory_order_relaxed);
            A.col_idx[k] = x.j - 1;
            A.values[k] = x.v;
            if (symmetric && x.i != x.j) {
                k = pos[x.j - 1].fetch_add(1, std::memory_order_relaxed);
                A.col_idx[k] = x.i - 1;
                A.values[k] = x.v;
            }
        }
    };
    run(scatter, T);
    const int TR = static_cast<int>(std::min<index_t>(nthreads(), std::max<index_t>(1, nrows / 4096)));
    std::atomic<bool> dup{false};
    auto sort_rows = [&](int t) {
        std::vector<std::pair<index_t, double>> row;
        for (index_t r = nrows * t / TR; r < nrows * (t + 1) / TR; ++r) {
            const index_t lo = A.row_ptr[r], hi = A.row_ptr[r + 1];
            row.resize(static_cast<size_t>(hi - lo));
            for (index_t k = lo; k < hi; ++k) row[k - lo] = {A.col_idx[k], A.values[k]};
            std::sort(row.begin(), row.end(),
                      [](const auto& a, const auto& b) { return a.first < b.first; });
            for (index_t k = lo; k < hi; ++k) {
                A.col_idx[k] = row[k - lo].first;
                A.values[k] = row[k - lo].second;
                if (k > lo && A.col_idx[k] == A.col_idx[k - 1]) dup = true;
            }
        }
    };
    run(sort_rows, TR);
    if (!dup) return A;
    // duplicates: the reference's summation order (from_triplets over the
    // file-order triplets, matrix_market.cpp:79-81 + csr.cpp from_triplets)
    std::vector<Triplet> trip;
    trip.reserve(static_cast<size_t>(total));
    for (int t = 0; t < T; ++t)
        for (const Entry& x : ch[t].ent) {
            trip.push_back({x.i - 1, x.j - 1, x.v});
            if (symmetric && x.i != x.j) trip.push_back({x.j - 1, x.i - 1, x.v});
        }
    return CsrMatrix::from_triplets(nrows, ncols, std::move(trip));
}

void write_matrix_market(const CsrMatrix& A, const std::string& path, bool symmetric) {
    if (symmetric && !host_symmetric_pattern(A))
        throw std::invalid_argument(
            "write_matrix_market: symmetric output of a matrix with an asymmetric pattern");
    std::FILE* f = std::fopen(path.c_str(), "w");
    if (!f) throw std::runtime_error("cannot open file for writing: " + path);
    const int T = static_cast<int>(std::min<index_t>(nthreads(), std::max<index_t>(1, A.nrows / 4096)));
    std::vector<std::string> buf(T);
    std::vector<index_t> count(T, 0);
    auto fmt = [&](int t) {
        std::string& b = buf[t];
        char tmp[96];
        for (index_t i = A.nrows * t / T; i < A.nrows * (t + 1) / T; ++i)
            for (index_t k = A.row_begin(i); k < A.row_end(i); ++k) {
                const index_t j = A.col_idx[k];
                if (symmetric && j > i) continue;
                const int len = std::snprintf(tmp, sizeof(tmp), "%lld %lld %.16e\n",
                                              static_cast<long long>(i + 1),
                                              static_cast<long long>(j + 1), A.values[k]);
                b.append(tmp, static_cast<size_t>(len));
                ++count[t];
            }
    };
    {
        std::vector<std::thread> th;
        for (int t = 1; t < T; ++t) th.emplace_back(fmt, t);
        fmt(0);
        for (auto& x : th) x.join();
    }
    index_t total = 0;
    for (index_t c : count) total += c;
    std::fprintf(f, "%%%%MatrixMarket matrix coordinate real %s\n", symmetric ? "symmetric" : "general");
    std::fprintf(f, "%lld %lld %lld\n", static_cast<long long>(A.nrows),
                 static_cast<long long>(A.ncols), static_cast<long long>(total));
    for (const std::string& b : buf) std::fwrite(b.data(), 1, b.size(), f);
    std::fclose(f);
}

} // namespace matchamg
