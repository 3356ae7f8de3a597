// Instance I/O of the algebraic import path: the reference's
// text formats, parsed and written by all host threads.
//
//   element block file   read_block_operator / write_block_operator (src/block_io.cpp:15-94)
//   Matrix Market        read_matrix_market / write_matrix_market   (src/matrix_market.cpp:36-122)
//   vector files         read_vector_lines / write_vector_lines     (src/matrix_market.cpp:124-146)
//
// The reference reads line by line through istringstream and writes through one
// ofstream; at BASELINE sizes (config 5: 15 GB of blocks) that is the bottleneck
// of an import.  Here a file is read into memory once, its lines indexed by a
// parallel newline scan, the records located by a sequential walk over the
// headers only (block dof counts / the size line) and every record parsed in
// parallel with std::from_chars, which rounds exactly like the reference's
// stream extraction, so the values are bit-identical.  Writers format with the
// reference's "%.17g" in parallel chunks and write the bytes once: the files are
// byte-identical to the reference's.  Matrix Market triplets are summed into CSR
// like CsrMatrix::from_triplets (src/csr.cpp:43-75: sorted by (row, col),
// duplicates summed in file order — deterministic; the reference's unstable sort
// leaves the order of equal keys unspecified).  Errors: HDR_FORMAT_ERROR with
// the reference's message and physical line number (FormatError), or
// HDR_DIMENSION_MISMATCH for the checks of ElementBlockOperator::validate
// (src/block_operator.cpp:10-27).
#include <algorithm>
#include <charconv>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <memory>
#include <numeric>
#include <string>
#include <thread>
#include <vector>

#include "../../include/hdivred_b200.h"

namespace hdr {
std::string& last_error_ref();  // capi.cu
}

struct hdr_blocks_s {
  int64_t nblocks = 0, broken_dim = 0, global_dim = 0;
  std::vector<int64_t> sizes, entry_off, dof_global;
  std::vector<double> dof_sign, entries;
};

struct hdr_csr_host_s {
  int64_t nrows = 0, ncols = 0;
  std::vector<int64_t> row_offsets, col_indices;
  std::vector<double> values;
};

namespace {

hdr_status fail(hdr_status s, const std::string& msg) {
  hdr::last_error_ref() = msg;
  return s;
}

template <class F>
hdr_status catch_all(F&& fn) {  // host-only entry points: no CUDA here
  try {
    return fn();
  } catch (const std::bad_alloc&) {
    return fail(HDR_INVALID_ARGUMENT, "host allocation failed");
  } catch (const std::exception& e) {
    return fail(HDR_INVALID_ARGUMENT, e.what());
  }
}

struct FormatErr {
  std::string msg;
  long line;
};

int nthreads(int requested) {
  if (requested > 0) return requested;
  const unsigned hc = std::thread::hardware_concurrency();
  return hc ? static_cast<int>(hc) : 4;
}

template <class F>
void parallel_for(int64_t n, int threads, F&& fn) {  // fn(lo, hi, thread)
  const int t = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(threads, n)));
  if (t == 1) {
    fn(int64_t(0), n, 0);
    return;
  }
  std::vector<std::thread> pool;
  for (int i = 0; i < t; ++i) {
    const int64_t lo = n * i / t, hi = n * (i + 1) / t;
    pool.emplace_back([&fn, lo, hi, i] { fn(lo, hi, i); });
  }
  for (auto& th : pool) th.join();
}

bool read_file(const char* path, std::string& buf) {
  FILE* f = std::fopen(path, "rb");
  if (!f) return false;
  std::fseek(f, 0, SEEK_END);
  const long sz = std::ftell(f);
  std::fseek(f, 0, SEEK_SET);
  buf.resize(sz > 0 ? static_cast<size_t>(sz) : 0);
  const size_t got = sz > 0 ? std::fread(&buf[0], 1, buf.size(), f) : 0;
  std::fclose(f);
  return got == buf.size();
}

// line starts (and the implied ends) of the whole buffer, found in parallel
struct Lines {
  const char* base = nullptr;
  std::vector<int64_t> start;  // start offset of line i; line i ends at start[i+1] - 1 (the '\n') or the buffer end
  int64_t size = 0;
  int64_t count() const { return static_cast<int64_t>(start.size()); }
  const char* b(int64_t i) const { return base + start[i]; }
  const char* e(int64_t i) const {
    int64_t end = i + 1 < count() ? start[i + 1] - 1 : size;
    if (end > start[i] && base[end - 1] == '\n') --end;  // the last line's own newline
    while (end > start[i] && base[end - 1] == '\r') --end;
    return base + end;
  }
};

Lines index_lines(const std::string& buf, int threads) {
  Lines L;
  L.base = buf.data();
  L.size = static_cast<int64_t>(buf.size());
  const int64_t n = L.size;
  const int t = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(threads, n / (1 << 16) + 1)));
  std::vector<int64_t> cnt(t + 1, 0);
  parallel_for(t, t, [&](int64_t lo, int64_t hi, int) {
    for (int64_t c = lo; c < hi; ++c) {
      const int64_t a = n * c / t, z = n * (c + 1) / t;
      int64_t k = 0;
      for (const char* p = L.base + a; (p = static_cast<const char*>(std::memchr(p, '\n', L.base + z - p))); ++p) ++k;
      cnt[c + 1] = k;
    }
  });
  for (int c = 0; c < t; ++c) cnt[c + 1] += cnt[c];
  const bool tail = n > 0 && L.base[n - 1] != '\n';
  L.start.assign(static_cast<size_t>(cnt[t] + (tail ? 1 : 0)), 0);
  parallel_for(t, t, [&](int64_t lo, int64_t hi, int) {
    for (int64_t c = lo; c < hi; ++c) {
      const int64_t a = n * c / t, z = n * (c + 1) / t;
      int64_t k = cnt[c];
      for (const char* p = L.base + a; (p = static_cast<const char*>(std::memchr(p, '\n', L.base + z - p))); ++p)
        if (k + 1 < L.count()) L.start[static_cast<size_t>(++k)] = (p - L.base) + 1;
        else ++k;
    }
  });
  return L;
}

inline const char* skip_ws(const char* p, const char* e) {
  while (p < e && (*p == ' ' || *p == '\t' || *p == '\r' || *p == '\v' || *p == '\f')) ++p;
  return p;
}

// one token of the stream-extraction grammar: optional '+', then from_chars
template <class T>
bool next_num(const char*& p, const char* e, T& v) {
  p = skip_ws(p, e);
  if (p >= e) return false;
  const char* q = p;
  if (*q == '+' && q + 1 < e && *(q + 1) != '-') ++q;
  auto r = std::from_chars(q, e, v);
  if (r.ec != std::errc()) return false;
  if (r.ptr < e && !(*r.ptr == ' ' || *r.ptr == '\t' || *r.ptr == '\r' || *r.ptr == '\v' || *r.ptr == '\f'))
    return false;  // the stream would stop inside the token: a malformed number
  p = r.ptr;
  return true;
}

bool content(const Lines& L, int64_t i) {  // block / Matrix Market content line: not empty, not a comment
  return L.e(i) > L.b(i) && *L.b(i) != '%';
}

std::string banner(const Lines& L) {
  if (L.count() == 0) return std::string();
  std::string s(L.b(0), L.e(0));
  while (!s.empty() && (s.back() == ' ' || s.back() == '\r' || s.back() == '\t' || s.back() == '\n')) s.pop_back();
  return s;
}

hdr_status format_error(const std::string& msg, long line) {
  return fail(HDR_FORMAT_ERROR, msg + " (line " + std::to_string(line) + ")");
}

std::string fmt17(double v) {
  char buf[40];
  const int k = std::snprintf(buf, sizeof buf, "%.17g", v);
  return std::string(buf, static_cast<size_t>(k));
}

// writes the chunks produced in parallel: chunk(i) formats records [lo, hi)
template <class F>
hdr_status write_chunks(const char* path, const std::string& head, int64_t nrec, int threads, F&& chunk) {
  const int t = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(threads, nrec)));
  std::vector<std::string> out(static_cast<size_t>(t));
  parallel_for(t, t, [&](int64_t lo, int64_t hi, int) {
    for (int64_t c = lo; c < hi; ++c) chunk(nrec * c / t, nrec * (c + 1) / t, out[static_cast<size_t>(c)]);
  });
  FILE* f = std::fopen(path, "wb");
  if (!f) return format_error("cannot open '" + std::string(path) + "' for writing", 0);
  bool ok = std::fwrite(head.data(), 1, head.size(), f) == head.size();
  for (const auto& s : out) ok = ok && std::fwrite(s.data(), 1, s.size(), f) == s.size();
  ok = std::fclose(f) == 0 && ok;
  if (!ok) return format_error("write failed on '" + std::string(path) + "'", 0);
  return HDR_OK;
}

}  // namespace

extern "C" {

hdr_status hdr_io_read_block_operator(const char* path, int threads, hdr_blocks_t* out) {
  if (!path || !out) return fail(HDR_INVALID_ARGUMENT, "null argument");
  *out = nullptr;
  return catch_all([&]() -> hdr_status {
    std::string buf;
    if (!read_file(path, buf)) return format_error("cannot open '" + std::string(path) + "' for reading", 0);
    const int T = nthreads(threads);
    const Lines L = index_lines(buf, T);
    if (L.count() == 0 || buf.empty()) return format_error("empty block file", 1);
    if (banner(L) != "%%ElementBlockOperator") return format_error("bad block file header: '" + banner(L) + "'", 1);
    // content lines after the banner (next_line skips empty and '%' lines)
    std::vector<int64_t> cl;
    cl.reserve(static_cast<size_t>(L.count()));
    for (int64_t i = 1; i < L.count(); ++i)
      if (content(L, i)) cl.push_back(i);
    auto ln = [&](size_t c) { return static_cast<long>(cl[c] + 1); };
    if (cl.empty()) return format_error("unexpected end of block file", static_cast<long>(L.count()));
    auto op = std::make_unique<hdr_blocks_s>();
    {
      const char* p = L.b(cl[0]);
      const char* e = L.e(cl[0]);
      long long nb = 0, bd = 0, gd = 0;
      if (!next_num(p, e, nb) || !next_num(p, e, bd) || !next_num(p, e, gd) || nb < 0)
        return format_error("bad block file size line", ln(0));
      op->nblocks = nb;
      op->broken_dim = bd;
      op->global_dim = gd;
    }
    // headers walk: the first content line of each block (its dof count)
    std::vector<size_t> first(static_cast<size_t>(op->nblocks));
    op->sizes.resize(static_cast<size_t>(op->nblocks));
    op->entry_off.assign(static_cast<size_t>(op->nblocks) + 1, 0);
    size_t c = 1;
    for (int64_t b = 0; b < op->nblocks; ++b) {
      if (c >= cl.size()) return format_error("unexpected end of block file", static_cast<long>(L.count()));
      const char* p = L.b(cl[c]);
      long long n = 0;
      if (!next_num(p, L.e(cl[c]), n) || n < 0) return format_error("bad block dof count", ln(c));
      first[static_cast<size_t>(b)] = c;
      op->sizes[static_cast<size_t>(b)] = n;
      op->entry_off[static_cast<size_t>(b) + 1] = op->entry_off[static_cast<size_t>(b)] + n * n;
      c += 1 + (n > 0 ? 1 : 0) + static_cast<size_t>(n);
    }
    if (c > cl.size()) return format_error("unexpected end of block file", static_cast<long>(L.count()));
    std::vector<int64_t> doff(static_cast<size_t>(op->nblocks) + 1, 0);
    for (int64_t b = 0; b < op->nblocks; ++b) doff[static_cast<size_t>(b) + 1] = doff[static_cast<size_t>(b)] + op->sizes[static_cast<size_t>(b)];
    op->dof_global.resize(static_cast<size_t>(doff.back()));
    op->dof_sign.resize(static_cast<size_t>(doff.back()));
    op->entries.resize(static_cast<size_t>(op->entry_off.back()));
    // parallel record parse; the first error (by line) wins
    std::vector<FormatErr> errs(static_cast<size_t>(T));
    std::vector<long> err_line(static_cast<size_t>(T), -1);
    parallel_for(op->nblocks, T, [&](int64_t lo, int64_t hi, int t) {
      for (int64_t b = lo; b < hi && err_line[static_cast<size_t>(t)] < 0; ++b) {
        const int64_t n = op->sizes[static_cast<size_t>(b)];
        size_t q = first[static_cast<size_t>(b)] + 1;
        if (n > 0) {
          const char* p = L.b(cl[q]);
          const char* e = L.e(cl[q]);
          for (int64_t l = 0; l < n; ++l) {
            long long id = 0;
            if (!next_num(p, e, id) || id == 0) {
              errs[static_cast<size_t>(t)] = {"bad signed dof id", ln(q)};
              err_line[static_cast<size_t>(t)] = ln(q);
              break;
            }
            const int64_t g = std::llabs(id) - 1;
            if (g >= op->global_dim) {
              errs[static_cast<size_t>(t)] = {"dof id exceeds global dimension", ln(q)};
              err_line[static_cast<size_t>(t)] = ln(q);
              break;
            }
            op->dof_global[static_cast<size_t>(doff[static_cast<size_t>(b)] + l)] = g;
            op->dof_sign[static_cast<size_t>(doff[static_cast<size_t>(b)] + l)] = id < 0 ? -1.0 : 1.0;
          }
          ++q;
        }
        double* a = op->entries.data() + op->entry_off[static_cast<size_t>(b)];
        for (int64_t i = 0; i < n && err_line[static_cast<size_t>(t)] < 0; ++i, ++q) {
          const char* p = L.b(cl[q]);
          const char* e = L.e(cl[q]);
          for (int64_t j = 0; j < n; ++j)
            if (!next_num(p, e, a[i * n + j])) {
              errs[static_cast<size_t>(t)] = {"bad matrix entry", ln(q)};
              err_line[static_cast<size_t>(t)] = ln(q);
              break;
            }
        }
      }
    });
    long best = -1;
    size_t bi = 0;
    for (size_t t = 0; t < errs.size(); ++t)
      if (err_line[t] >= 0 && (best < 0 || err_line[t] < best)) best = err_line[t], bi = t;
    if (best >= 0) return format_error(errs[bi].msg, errs[bi].line);
    // ElementBlockOperator::validate (src/block_operator.cpp:10-27)
    for (double v : op->entries)
      if (!std::isfinite(v)) return fail(HDR_DIMENSION_MISMATCH, "ElementBlockOperator: non-finite entry");
    if (doff.back() != op->broken_dim)
      return fail(HDR_DIMENSION_MISMATCH, "ElementBlockOperator: broken_dim != sum of block sizes");
    *out = op.release();
    return HDR_OK;
  });
}

hdr_status hdr_io_blocks_info(hdr_blocks_t b, int64_t* info) {
  if (!b || !info) return fail(HDR_INVALID_ARGUMENT, "null argument");
  info[0] = b->nblocks;
  info[1] = b->broken_dim;
  info[2] = b->global_dim;
  info[3] = static_cast<int64_t>(b->entries.size());
  return HDR_OK;
}

hdr_status hdr_io_blocks_get(hdr_blocks_t b, int64_t* block_sizes, int64_t* dof_global, double* dof_sign,
                             double* entries) {
  if (!b) return fail(HDR_INVALID_ARGUMENT, "null argument");
  if (block_sizes) std::copy(b->sizes.begin(), b->sizes.end(), block_sizes);
  if (dof_global) std::copy(b->dof_global.begin(), b->dof_global.end(), dof_global);
  if (dof_sign) std::copy(b->dof_sign.begin(), b->dof_sign.end(), dof_sign);
  if (entries) std::copy(b->entries.begin(), b->entries.end(), entries);
  return HDR_OK;
}

void hdr_io_blocks_destroy(hdr_blocks_t b) { delete b; }

hdr_status hdr_io_write_block_operator(const char* path, int64_t nblocks, int64_t broken_dim, int64_t global_dim,
                                       const int64_t* block_sizes, const int64_t* dof_global, const double* dof_sign,
                                       const double* entries, int threads) {
  if (!path || nblocks < 0 || (nblocks > 0 && (!block_sizes || !dof_global || !dof_sign || !entries)))
    return fail(HDR_INVALID_ARGUMENT, "null argument");
  return catch_all([&]() -> hdr_status {
    std::vector<int64_t> doff(static_cast<size_t>(nblocks) + 1, 0), eoff(static_cast<size_t>(nblocks) + 1, 0);
    for (int64_t b = 0; b < nblocks; ++b) {
      doff[static_cast<size_t>(b) + 1] = doff[static_cast<size_t>(b)] + block_sizes[b];
      eoff[static_cast<size_t>(b) + 1] = eoff[static_cast<size_t>(b)] + block_sizes[b] * block_sizes[b];
    }
    const std::string head = "%%ElementBlockOperator\n" + std::to_string(nblocks) + " " + std::to_string(broken_dim) +
                             " " + std::to_string(global_dim) + "\n";
    return write_chunks(path, head, nblocks, nthreads(threads), [&](int64_t lo, int64_t hi, std::string& s) {
      for (int64_t b = lo; b < hi; ++b) {
        const int64_t n = block_sizes[b];
        s += std::to_string(n);
        s += '\n';
        for (int64_t l = 0; l < n; ++l) {  // signed 1-based ids (block_io.cpp:23-27)
          const int64_t d = doff[static_cast<size_t>(b)] + l;
          const long long id = static_cast<long long>(dof_global[d] + 1) * (dof_sign[d] < 0.0 ? -1 : 1);
          s += std::to_string(id);
          s += (l + 1 == n) ? '\n' : ' ';
        }
        const double* a = entries + eoff[static_cast<size_t>(b)];
        for (int64_t i = 0; i < n; ++i)
          for (int64_t j = 0; j < n; ++j) {
            s += fmt17(a[i * n + j]);
            s += (j + 1 == n) ? '\n' : ' ';
          }
      }
    });
  });
}

hdr_status hdr_io_read_matrix_market(const char* path, int threads, hdr_csr_host_t* out) {
  if (!path || !out) return fail(HDR_INVALID_ARGUMENT, "null argument");
  *out = nullptr;
  return catch_all([&]() -> hdr_status {
    std::string buf;
    if (!read_file(path, buf)) return format_error("cannot open '" + std::string(path) + "' for reading", 0);
    const int T = nthreads(threads);
    const Lines L = index_lines(buf, T);
    if (L.count() == 0 || buf.empty()) return format_error("empty file", 1);
    if (banner(L) != "%%MatrixMarket matrix coordinate real general")
      return format_error("bad MatrixMarket header: '" + std::string(L.b(0), L.e(0)) + "'", 1);
    int64_t i0 = 1;
    while (i0 < L.count() && L.e(i0) > L.b(i0) && *L.b(i0) == '%') ++i0;  // comments before the size line
    long long nr = -1, nc = -1, nz = -1;
    if (i0 >= L.count()) return format_error("missing size line", static_cast<long>(L.count()));
    {
      const char* p = L.b(i0);
      if (!next_num(p, L.e(i0), nr) || !next_num(p, L.e(i0), nc) || !next_num(p, L.e(i0), nz))
        return format_error("bad size line", static_cast<long>(i0 + 1));
    }
    if (nr < 0 || nc < 0 || nz < 0) return format_error("missing size line", static_cast<long>(i0 + 1));
    std::vector<int64_t> el;  // entry lines
    el.reserve(static_cast<size_t>(nz));
    for (int64_t i = i0 + 1; i < L.count() && static_cast<long long>(el.size()) < nz; ++i)
      if (content(L, i)) el.push_back(i);
    if (static_cast<long long>(el.size()) < nz)
      return format_error("unexpected end of file: expected " + std::to_string(nz) + " entries",
                          static_cast<long>(L.count()));
    std::vector<int64_t> rows(static_cast<size_t>(nz)), cols(static_cast<size_t>(nz));
    std::vector<double> vals(static_cast<size_t>(nz));
    std::vector<long> err_line(static_cast<size_t>(T), -1);
    std::vector<std::string> err_msg(static_cast<size_t>(T));
    parallel_for(nz, T, [&](int64_t lo, int64_t hi, int t) {
      for (int64_t k = lo; k < hi; ++k) {
        const char* p = L.b(el[static_cast<size_t>(k)]);
        const char* e = L.e(el[static_cast<size_t>(k)]);
        long long i = 0, j = 0;
        double v = 0.0;
        const long line = static_cast<long>(el[static_cast<size_t>(k)] + 1);
        if (!next_num(p, e, i) || !next_num(p, e, j) || !next_num(p, e, v)) {
          err_line[static_cast<size_t>(t)] = line;
          err_msg[static_cast<size_t>(t)] = "bad entry line";
          return;
        }
        if (i < 1 || i > nr || j < 1 || j > nc) {
          err_line[static_cast<size_t>(t)] = line;
          err_msg[static_cast<size_t>(t)] = "entry index out of range";
          return;
        }
        rows[static_cast<size_t>(k)] = i - 1;
        cols[static_cast<size_t>(k)] = j - 1;
        vals[static_cast<size_t>(k)] = v;
      }
    });
    long best = -1;
    size_t bi = 0;
    for (size_t t = 0; t < err_line.size(); ++t)
      if (err_line[t] >= 0 && (best < 0 || err_line[t] < best)) best = err_line[t], bi = t;
    if (best >= 0) return format_error(err_msg[bi], best);
    // from_triplets: counting sort by row, stable sort by column inside each row,
    // duplicates summed in file order (csr.cpp:43-75)
    auto csr = std::make_unique<hdr_csr_host_s>();
    csr->nrows = nr;
    csr->ncols = nc;
    std::vector<int64_t> cnt(static_cast<size_t>(nr) + 1, 0);
    for (int64_t r : rows) ++cnt[static_cast<size_t>(r) + 1];
    for (int64_t r = 0; r < nr; ++r) cnt[static_cast<size_t>(r) + 1] += cnt[static_cast<size_t>(r)];
    std::vector<int64_t> ord(static_cast<size_t>(nz)), fill(cnt.begin(), cnt.end() - 1);
    for (int64_t k = 0; k < nz; ++k) ord[static_cast<size_t>(fill[static_cast<size_t>(rows[static_cast<size_t>(k)])]++)] = k;
    std::vector<int64_t> rnnz(static_cast<size_t>(nr), 0);
    parallel_for(nr, T, [&](int64_t lo, int64_t hi, int) {
      for (int64_t r = lo; r < hi; ++r) {
        auto b = ord.begin() + cnt[static_cast<size_t>(r)], e = ord.begin() + cnt[static_cast<size_t>(r) + 1];
        std::stable_sort(b, e, [&](int64_t x, int64_t y) { return cols[static_cast<size_t>(x)] < cols[static_cast<size_t>(y)]; });
        int64_t u = 0;
        for (auto it = b; it != e; ++it)
          if (it == b || cols[static_cast<size_t>(*it)] != cols[static_cast<size_t>(*(it - 1))]) ++u;
        rnnz[static_cast<size_t>(r)] = u;
      }
    });
    csr->row_offsets.assign(static_cast<size_t>(nr) + 1, 0);
    for (int64_t r = 0; r < nr; ++r) csr->row_offsets[static_cast<size_t>(r) + 1] = csr->row_offsets[static_cast<size_t>(r)] + rnnz[static_cast<size_t>(r)];
    csr->col_indices.resize(static_cast<size_t>(csr->row_offsets.back()));
    csr->values.resize(static_cast<size_t>(csr->row_offsets.back()));
    parallel_for(nr, T, [&](int64_t lo, int64_t hi, int) {
      for (int64_t r = lo; r < hi; ++r) {
        int64_t o = csr->row_offsets[static_cast<size_t>(r)] - 1;
        for (int64_t q = cnt[static_cast<size_t>(r)]; q < cnt[static_cast<size_t>(r) + 1]; ++q) {
          const int64_t k = ord[static_cast<size_t>(q)];
          if (q == cnt[static_cast<size_t>(r)] || cols[static_cast<size_t>(k)] != cols[static_cast<size_t>(ord[static_cast<size_t>(q - 1)])]) {
            ++o;
            csr->col_indices[static_cast<size_t>(o)] = cols[static_cast<size_t>(k)];
            csr->values[static_cast<size_t>(o)] = vals[static_cast<size_t>(k)];
          } else {
            csr->values[static_cast<size_t>(o)] += vals[static_cast<size_t>(k)];
          }
        }
      }
    });
    *out = csr.release();
    return HDR_OK;
  });
}

hdr_status hdr_io_read_vector_lines(const char* path, int threads, hdr_csr_host_t* out) {
  if (!path || !out) return fail(HDR_INVALID_ARGUMENT, "null argument");
  *out = nullptr;
  return catch_all([&]() -> hdr_status {
    std::string buf;
    if (!read_file(path, buf)) return format_error("cannot open '" + std::string(path) + "' for reading", 0);
    const int T = nthreads(threads);
    const Lines L = index_lines(buf, T);
    std::vector<int64_t> vl;
    for (int64_t i = 0; i < L.count(); ++i)
      if (L.e(i) > L.b(i)) vl.push_back(i);  // read_vector_lines skips empty lines only
    auto v = std::make_unique<hdr_csr_host_s>();
    const int64_t n = static_cast<int64_t>(vl.size());
    v->nrows = n;
    v->ncols = 1;
    v->values.resize(static_cast<size_t>(n));
    std::vector<long> bad(static_cast<size_t>(T), -1);
    parallel_for(n, T, [&](int64_t lo, int64_t hi, int t) {
      for (int64_t k = lo; k < hi; ++k) {
        const char* p = L.b(vl[static_cast<size_t>(k)]);
        if (!next_num(p, L.e(vl[static_cast<size_t>(k)]), v->values[static_cast<size_t>(k)])) {
          bad[static_cast<size_t>(t)] = static_cast<long>(vl[static_cast<size_t>(k)] + 1);
          return;
        }
      }
    });
    for (long b : bad)
      if (b >= 0) return format_error("bad vector line", *std::min_element(bad.begin(), bad.end(), [](long x, long y) {
                                        return x >= 0 && (y < 0 || x < y);
                                      }));
    v->row_offsets.resize(static_cast<size_t>(n) + 1);
    std::iota(v->row_offsets.begin(), v->row_offsets.end(), int64_t(0));
    v->col_indices.assign(static_cast<size_t>(n), 0);
    *out = v.release();
    return HDR_OK;
  });
}

hdr_status hdr_io_csr_info(hdr_csr_host_t a, int64_t* info) {
  if (!a || !info) return fail(HDR_INVALID_ARGUMENT, "null argument");
  info[0] = a->nrows;
  info[1] = a->ncols;
  info[2] = static_cast<int64_t>(a->values.size());
  return HDR_OK;
}

hdr_status hdr_io_csr_get(hdr_csr_host_t a, int64_t* row_offsets, int64_t* col_indices, double* values) {
  if (!a) return fail(HDR_INVALID_ARGUMENT, "null argument");
  if (row_offsets) std::copy(a->row_offsets.begin(), a->row_offsets.end(), row_offsets);
  if (col_indices) std::copy(a->col_indices.begin(), a->col_indices.end(), col_indices);
  if (values) std::copy(a->values.begin(), a->values.end(), values);
  return HDR_OK;
}

void hdr_io_csr_destroy(hdr_csr_host_t a) { delete a; }

hdr_status hdr_io_write_matrix_market(const char* path, int64_t nrows, int64_t ncols, const int64_t* row_offsets,
                                      const int64_t* col_indices, const double* values, int threads) {
  if (!path || nrows < 0 || ncols < 0 || !row_offsets) return fail(HDR_INVALID_ARGUMENT, "null argument");
  return catch_all([&]() -> hdr_status {
    const int64_t nnz = row_offsets[nrows];
    const std::string head = "%%MatrixMarket matrix coordinate real general\n" + std::to_string(nrows) + " " +
                             std::to_string(ncols) + " " + std::to_string(nnz) + "\n";
    return write_chunks(path, head, nrows, nthreads(threads), [&](int64_t lo, int64_t hi, std::string& s) {
      for (int64_t i = lo; i < hi; ++i)
        for (int64_t k = row_offsets[i]; k < row_offsets[i + 1]; ++k) {
          s += std::to_string(i + 1);
          s += ' ';
          s += std::to_string(col_indices[k] + 1);
          s += ' ';
          s += fmt17(values[k]);
          s += '\n';
        }
    });
  });
}

hdr_status hdr_io_write_vector_lines(const char* path, int64_t n, const double* v, int threads) {
  if (!path || n < 0 || (n > 0 && !v)) return fail(HDR_INVALID_ARGUMENT, "null argument");
  return catch_all([&]() -> hdr_status {
    return write_chunks(path, std::string(), n, nthreads(threads), [&](int64_t lo, int64_t hi, std::string& s) {
      for (int64_t i = lo; i < hi; ++i) {
        s += fmt17(v[i]);
        s += '\n';
      }
    });
  });
}

}  // extern "C"
