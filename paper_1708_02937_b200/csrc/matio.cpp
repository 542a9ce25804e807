// Matrix Market exchange for the device matrices ("real general"; coordinate
// files become a device CSR, array files a device dense matrix).
//
// Semantics follow the reference reader/writer (proj/include/semikern/matio.hpp,
// proj/src/matio.cpp: accepted header forms, std::from_chars number rules, the
// 1-based line numbers and texts of every ParseError, "%.9g" output); the
// implementation is built for large files feeding the GPU:
//
//  * the text is indexed once (line spans, '\r' stripped) and the entry lines
//    are tokenised and converted by several host threads, each over a
//    contiguous block of lines.  Pass 1 counts the non-blank lines of every
//    block, so pass 2 knows each line's entry ordinal and every block stops at
//    its own first error; the error with the smallest line number is the one a
//    sequential reader would meet first, so messages are independent of the
//    thread count.
//  * coordinate entries go to the device triple builder (stable radix sort by
//    (row, col), duplicate check, zero elision, CSR).  Its stable order
//    reports the later line of a duplicate pair, as the reference does.
//  * the writer formats blocks of rows (columns for arrays) in parallel and
//    concatenates them in order.
#include <algorithm>
#include <charconv>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <iterator>
#include <string>
#include <string_view>
#include <thread>
#include <vector>

#include "sk_common.cuh"

namespace sk {
namespace {

constexpr char kMagic[] = "%%MatrixMarket";

// ---- text index -------------------------------------------------------------------

struct Span {
  uint32_t b, e;  // [b, e) into the text, '\r' stripped
};

// Lines as std::getline yields them: '\n'-separated, a last line without a
// newline counts, nothing after a final newline.
std::vector<Span> index_lines(std::string_view t) {
  std::vector<Span> out;
  out.reserve(t.size() / 16 + 1);
  size_t p = 0;
  while (p < t.size()) {
    const void* nl = std::memchr(t.data() + p, '\n', t.size() - p);
    size_t e = nl ? size_t(static_cast<const char*>(nl) - t.data()) : t.size();
    const size_t next = nl ? e + 1 : t.size();
    if (e > p && t[e - 1] == '\r') --e;
    out.push_back({uint32_t(p), uint32_t(e)});
    p = next;
  }
  return out;
}

// Whitespace (' ', '\t') separated tokens of one line: stores up to kCap,
// returns how many there are.
constexpr int kCap = 6;
int tokens(std::string_view s, std::string_view* tok) {
  int n = 0;
  const char* p = s.data();
  const char* const end = p + s.size();
  for (;;) {
    while (p != end && (*p == ' ' || *p == '\t')) ++p;
    if (p == end) return n;
    const char* q = p;
    while (q != end && *q != ' ' && *q != '\t') ++q;
    if (n < kCap) tok[n] = std::string_view(p, size_t(q - p));
    ++n;
    p = q;
  }
}

bool blank(std::string_view s) {
  for (char c : s)
    if (c != ' ' && c != '\t') return false;
  return true;
}

bool same_nocase(std::string_view a, const char* b) {
  const size_t n = std::strlen(b);
  if (a.size() != n) return false;
  for (size_t i = 0; i < n; ++i) {
    char c = a[i];
    if (c >= 'A' && c <= 'Z') c = char(c - 'A' + 'a');
    if (c != b[i]) return false;
  }
  return true;
}

std::string lower_copy(std::string_view a) {
  std::string s(a);
  for (char& c : s)
    if (c >= 'A' && c <= 'Z') c = char(c - 'A' + 'a');
  return s;
}

// ---- errors -----------------------------------------------------------------------

struct LineError {
  size_t line = SIZE_MAX;  // SIZE_MAX: none
  std::string msg;
  void set(size_t l, std::string m) {
    if (l < line) {
      line = l;
      msg = std::move(m);
    }
  }
  explicit operator bool() const { return line != SIZE_MAX; }
};

[[noreturn]] void raise(size_t line, const std::string& msg) {
  fail(SK_ERR_PARSE, "line " + std::to_string(line) + ": " + msg);
}

// std::from_chars with a leading '+' allowed; false (and the reference's text in
// *why) when the whole token is not one number of type T.
template <typename T>
bool number(std::string_view tok, const char* what, T& v, std::string* why) {
  const char* p = tok.data();
  const char* const e = p + tok.size();
  if (p != e && *p == '+') ++p;
  std::from_chars_result r;
  if constexpr (std::is_floating_point_v<T>)
    r = std::from_chars(p, e, v, std::chars_format::general);
  else
    r = std::from_chars(p, e, v);
  if (r.ec == std::errc{} && r.ptr == e) return true;
  *why = std::string("malformed ") + what + " '" + std::string(tok) + "'";
  return false;
}

template <typename T>
T number_or_raise(std::string_view tok, const char* what, size_t line) {
  T v{};
  std::string why;
  if (!number(tok, what, v, &why)) raise(line, why);
  return v;
}

// ---- header -----------------------------------------------------------------------

struct Head {
  bool coordinate = true;
  size_t size_line = 0;           // 1-based
  std::vector<std::string_view> size_tok;
  size_t body = 0;                // index of the first line after the size line
};

Head parse_head(std::string_view text, const std::vector<Span>& L) {
  if (L.empty()) raise(1, "empty file, expected Matrix Market header");
  std::string_view t[kCap];
  const auto at = [&](size_t i) { return text.substr(L[i].b, L[i].e - L[i].b); };
  const int n = tokens(at(0), t);
  if (n == 0 || t[0] != kMagic) raise(1, "header must begin '%%MatrixMarket matrix'");
  if (n != 5 || !same_nocase(t[1], "matrix"))
    raise(1, "header must be '%%MatrixMarket matrix <coordinate|array> real general'");
  Head h;
  if (same_nocase(t[2], "coordinate"))
    h.coordinate = true;
  else if (same_nocase(t[2], "array"))
    h.coordinate = false;
  else
    raise(1, "unsupported format '" + lower_copy(t[2]) + "' (expected coordinate or array)");
  if (!same_nocase(t[3], "real") || !same_nocase(t[4], "general"))
    raise(1, "only 'real general' matrices are supported");
  // comment lines ('%' first) and blank lines may precede the size line
  size_t i = 1;
  while (i < L.size()) {
    const std::string_view s = at(i);
    if ((s.empty() || s[0] != '%') && !blank(s)) break;
    ++i;
  }
  if (i == L.size()) raise(L.size() + 1, "unexpected end of file before size line");
  const int k = tokens(at(i), t);
  h.size_tok.assign(t, t + std::min(k, kCap));
  if (k > kCap) h.size_tok.resize(kCap + 1);  // only the count matters then
  h.size_line = i + 1;
  h.body = i + 1;
  return h;
}

// ---- parallel body pass -----------------------------------------------------------

int host_threads(size_t lines) {
  const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
  return int(std::max<size_t>(1, std::min<size_t>(std::min(hw, 32u), lines / 8192)));
}

template <typename F>
void parallel_blocks(int nb, F&& f) {
  if (nb == 1) {
    f(0);
    return;
  }
  std::vector<std::thread> th;
  th.reserve(size_t(nb));
  for (int b = 0; b < nb; ++b) th.emplace_back([&f, b] { f(b); });
  for (auto& x : th) x.join();
}

// Entries of the body: `want` non-blank lines of `fields` tokens each, then
// only blank lines.  parse(tokens, line, ordinal, why) converts one entry
// (false + *why on a bad entry); `noun` names entries in the messages.
template <typename Block, typename Parse>
std::vector<Block> parse_body(std::string_view text, const std::vector<Span>& L, size_t first,
                              size_t want, int fields, const char* field_msg, const char* noun,
                              Parse&& parse) {
  const size_t nlines = L.size() - first;
  const int nb = host_threads(nlines);
  std::vector<size_t> lo(static_cast<size_t>(nb) + 1), nonblank(static_cast<size_t>(nb), 0);
  for (int b = 0; b <= nb; ++b) lo[size_t(b)] = first + nlines * size_t(b) / size_t(nb);
  const auto at = [&](size_t i) { return text.substr(L[i].b, L[i].e - L[i].b); };
  parallel_blocks(nb, [&](int b) {
    size_t c = 0;
    for (size_t i = lo[size_t(b)]; i < lo[size_t(b) + 1]; ++i) c += !blank(at(i));
    nonblank[size_t(b)] = c;
  });
  const size_t nblk = size_t(nb);
  std::vector<Block> blocks(nblk);
  std::vector<LineError> errs(nblk);
  size_t total = 0;
  std::vector<size_t> base(nblk);
  for (int b = 0; b < nb; ++b) {
    base[size_t(b)] = total;
    total += nonblank[size_t(b)];
  }
  parallel_blocks(nb, [&](int b) {
    Block& out = blocks[size_t(b)];
    LineError& err = errs[size_t(b)];
    size_t ord = base[size_t(b)];
    std::string_view t[kCap];
    std::string why;
    for (size_t i = lo[size_t(b)]; i < lo[size_t(b) + 1]; ++i) {
      const int n = tokens(at(i), t);
      if (n == 0) continue;
      if (ord >= want) {  // the first non-blank line past the last entry
        err.set(i + 1, std::string("unexpected content after ") + std::to_string(want) + " " +
                           noun);
        return;
      }
      if (n != fields) {
        err.set(i + 1, std::string(field_msg) + std::to_string(n));
        return;
      }
      if (!parse(out, t, i + 1, ord, &why)) {
        err.set(i + 1, why);
        return;
      }
      ++ord;
    }
  });
  LineError first_err;
  for (auto& e : errs)
    if (e) first_err.set(e.line, e.msg);
  if (first_err) raise(first_err.line, first_err.msg);
  if (total < want)
    raise(L.size() + 1, "unexpected end of file: expected " + std::to_string(want) + " " + noun +
                            ", found " + std::to_string(total));
  return blocks;
}

struct NoBlock {};  // array values go straight into the dense host image

struct Triples {
  std::vector<uint32_t> r, c, line;
  std::vector<float> v;
};

void read_coordinate(sk_ctx* ctx, std::string_view text, const std::vector<Span>& L,
                     const Head& h, sk_csr** out) {
  if (h.size_tok.size() != 3) raise(h.size_line, "coordinate size line must be 'rows cols nnz'");
  const auto rows = number_or_raise<uint32_t>(h.size_tok[0], "row count", h.size_line);
  const auto cols = number_or_raise<uint32_t>(h.size_tok[1], "column count", h.size_line);
  const auto want = number_or_raise<size_t>(h.size_tok[2], "nnz count", h.size_line);
  auto blocks = parse_body<Triples>(
      text, L, h.body, want, 3, "entry must have 3 fields 'row col value', found ", "entries",
      [&](Triples& o, const std::string_view* t, size_t line, size_t, std::string* why) {
        uint64_t r = 0, c = 0;
        float v = 0.0f;
        if (!number(t[0], "row index", r, why) || !number(t[1], "column index", c, why) ||
            !number(t[2], "value", v, why))
          return false;
        if (r < 1 || r > rows) {
          *why = "row index " + std::to_string(r) + " out of range [1, " + std::to_string(rows) +
                 "]";
          return false;
        }
        if (c < 1 || c > cols) {
          *why = "column index " + std::to_string(c) + " out of range [1, " +
                 std::to_string(cols) + "]";
          return false;
        }
        o.r.push_back(uint32_t(r - 1));
        o.c.push_back(uint32_t(c - 1));
        o.v.push_back(v);
        o.line.push_back(uint32_t(line));
        return true;
      });
  // blocks in line order = the file's entry order (the builder's stable sort
  // keeps it among equal coordinates)
  Triples all;
  all.r.reserve(want);
  all.c.reserve(want);
  all.line.reserve(want);
  all.v.reserve(want);
  for (auto& b : blocks) {
    all.r.insert(all.r.end(), b.r.begin(), b.r.end());
    all.c.insert(all.c.end(), b.c.begin(), b.c.end());
    all.v.insert(all.v.end(), b.v.begin(), b.v.end());
    all.line.insert(all.line.end(), b.line.begin(), b.line.end());
  }
  const size_t n = all.r.size();
  uint32_t* d = dalloc<uint32_t>(ctx, 3 * std::max<size_t>(n, 1));
  if (n) {
    SK_CUDA(cudaMemcpyAsync(d, all.r.data(), n * 4, cudaMemcpyHostToDevice, ctx->stream));
    SK_CUDA(cudaMemcpyAsync(d + n, all.c.data(), n * 4, cudaMemcpyHostToDevice, ctx->stream));
    SK_CUDA(cudaMemcpyAsync(d + 2 * n, all.v.data(), n * 4, cudaMemcpyHostToDevice, ctx->stream));
  }
  uint64_t dup = ~0ull;
  sk_csr* a = nullptr;
  try {
    a = csr_from_device_triples(ctx, rows, cols, d, d + n, reinterpret_cast<const float*>(d + 2 * n),
                                n, all.r.data(), all.c.data(), &dup);
  } catch (...) {
    dfree(ctx, d);
    throw;
  }
  dfree(ctx, d);
  if (!a)
    raise(all.line[dup], "duplicate entry for (" + std::to_string(all.r[dup] + 1) + ", " +
                             std::to_string(all.c[dup] + 1) + ")");
  *out = a;
}

void read_array(sk_ctx* ctx, std::string_view text, const std::vector<Span>& L, const Head& h,
                sk_dense** out) {
  if (h.size_tok.size() != 2) raise(h.size_line, "array size line must be 'rows cols'");
  const auto rows = number_or_raise<uint32_t>(h.size_tok[0], "row count", h.size_line);
  const auto cols = number_or_raise<uint32_t>(h.size_tok[1], "column count", h.size_line);
  const size_t want = size_t(rows) * cols;
  std::vector<float> host(want, 0.0f);  // row-major; the file lists values down each column
  parse_body<NoBlock>(text, L, h.body, want, 1, "array lines carry one value each, found ", "values",
                   [&](NoBlock&, const std::string_view* t, size_t, size_t ord, std::string* why) {
                     float v = 0.0f;
                     if (!number(t[0], "value", v, why)) return false;
                     host[size_t(ord % rows) * cols + ord / rows] = v;
                     return true;
                   });
  sk_dense* d = new_dense(ctx, rows, cols);
  if (want)
    SK_CUDA(cudaMemcpyAsync(d->d, host.data(), want * 4, cudaMemcpyHostToDevice, ctx->stream));
  sync(ctx);
  *out = d;
}

void read_text(sk_ctx* ctx, std::string_view text, int* kind, sk_csr** csr, sk_dense** dense) {
  if (text.size() >= (size_t(1) << 32)) fail(SK_ERR_PARSE, "file larger than 4 GiB");
  const std::vector<Span> L = index_lines(text);
  const Head h = parse_head(text, L);
  *csr = nullptr;
  *dense = nullptr;
  *kind = h.coordinate ? 0 : 1;
  if (h.coordinate)
    read_coordinate(ctx, text, L, h, csr);
  else
    read_array(ctx, text, L, h, dense);
}

// ---- writer -----------------------------------------------------------------------

// "%.9g": nine significant digits round-trip every binary32 value.
inline void put_value(std::string& s, float v) {
  char buf[48];
  const int k = std::snprintf(buf, sizeof buf, "%.9g", double(v));
  s.append(buf, size_t(k));
}

inline void put_index(std::string& s, uint64_t x) {
  char buf[24];
  const auto r = std::to_chars(buf, buf + sizeof buf, x);
  s.append(buf, size_t(r.ptr - buf));
}

// Concatenation of f(b, out) over nb contiguous blocks of [0, n), in order.
template <typename F>
std::string formatted_blocks(size_t n, F&& f) {
  const int nb = int(std::max<size_t>(1, std::min<size_t>(std::max(1u, std::thread::hardware_concurrency()),
                                                          n / 4096)));
  std::vector<std::string> part(static_cast<size_t>(nb));
  parallel_blocks(nb, [&](int b) {
    f(n * size_t(b) / size_t(nb), n * size_t(b + 1) / size_t(nb), part[size_t(b)]);
  });
  std::string o;
  size_t tot = 0;
  for (auto& p : part) tot += p.size();
  o.reserve(tot);
  for (auto& p : part) o += p;
  return o;
}

std::string format_csr(sk_ctx* ctx, const sk_csr* a) {
  std::vector<uint32_t> rp(size_t(a->rows) + 1), ci(a->nnz);
  std::vector<float> v(a->nnz);
  SK_CUDA(cudaMemcpyAsync(rp.data(), a->rp, rp.size() * 4, cudaMemcpyDeviceToHost, ctx->stream));
  if (a->nnz) {
    SK_CUDA(cudaMemcpyAsync(ci.data(), a->ci, a->nnz * 4, cudaMemcpyDeviceToHost, ctx->stream));
    SK_CUDA(cudaMemcpyAsync(v.data(), a->v, a->nnz * 4, cudaMemcpyDeviceToHost, ctx->stream));
  }
  sync(ctx);
  std::string o = std::string(kMagic) + " matrix coordinate real general\n";
  put_index(o, a->rows);
  o += ' ';
  put_index(o, a->cols);
  o += ' ';
  put_index(o, a->nnz);
  o += '\n';
  o += formatted_blocks(a->rows, [&](size_t r0, size_t r1, std::string& s) {
    s.reserve((rp[r1] - rp[r0]) * 24);
    for (size_t i = r0; i < r1; ++i)
      for (uint32_t e = rp[i]; e < rp[i + 1]; ++e) {
        put_index(s, i + 1);
        s += ' ';
        put_index(s, uint64_t(ci[e]) + 1);
        s += ' ';
        put_value(s, v[e]);
        s += '\n';
      }
  });
  return o;
}

std::string format_dense(sk_ctx* ctx, const sk_dense* d) {
  std::vector<float> h(d->elems());
  if (!h.empty())
    SK_CUDA(cudaMemcpyAsync(h.data(), d->d, h.size() * 4, cudaMemcpyDeviceToHost, ctx->stream));
  sync(ctx);
  std::string o = std::string(kMagic) + " matrix array real general\n";
  put_index(o, d->rows);
  o += ' ';
  put_index(o, d->cols);
  o += '\n';
  o += formatted_blocks(d->cols, [&](size_t j0, size_t j1, std::string& s) {
    for (size_t j = j0; j < j1; ++j)  // values down each column
      for (uint32_t i = 0; i < d->rows; ++i) {
        put_value(s, h[size_t(i) * d->cols + j]);
        s += '\n';
      }
  });
  return o;
}

std::string format_matrix(sk_ctx* ctx, const sk_csr* a, const sk_dense* d) {
  return a ? format_csr(ctx, a) : format_dense(ctx, d);
}

}  // namespace
}  // namespace sk

using namespace sk;

extern "C" sk_status sk_read_matrix_text(sk_ctx* ctx, const char* text, size_t len, int* kind,
                                         sk_csr** csr, sk_dense** dense) {
  return guarded([&] {
    SK_CUDA(cudaSetDevice(ctx->device));
    read_text(ctx, std::string_view(text, len), kind, csr, dense);
  });
}

extern "C" sk_status sk_read_matrix(sk_ctx* ctx, const char* path, int* kind, sk_csr** csr,
                                    sk_dense** dense) {
  return guarded([&] {
    SK_CUDA(cudaSetDevice(ctx->device));
    std::ifstream in(path, std::ios::binary);
    if (!in) fail(SK_ERR, std::string("cannot open '") + path + "' for reading");
    const std::string text((std::istreambuf_iterator<char>(in)), std::istreambuf_iterator<char>());
    read_text(ctx, text, kind, csr, dense);
  });
}

extern "C" sk_status sk_format_matrix(sk_ctx* ctx, const sk_csr* csr, const sk_dense* dense,
                                      char* buf, size_t cap, size_t* len) {
  return guarded([&] {
    csr_ready(ctx, csr);
    if (!csr == !dense) fail(SK_ERR_INVALID_ARGUMENT, "pass exactly one of csr / dense");
    const std::string t = format_matrix(ctx, csr, dense);
    *len = t.size();
    if (buf && cap) {
      const size_t k = std::min(cap - 1, t.size());
      std::memcpy(buf, t.data(), k);
      buf[k] = 0;
    }
  });
}

extern "C" sk_status sk_write_matrix(sk_ctx* ctx, const sk_csr* csr, const sk_dense* dense,
                                     const char* path) {
  return guarded([&] {
    csr_ready(ctx, csr);
    if (!csr == !dense) fail(SK_ERR_INVALID_ARGUMENT, "pass exactly one of csr / dense");
    std::ofstream out(path, std::ios::binary);
    if (!out) fail(SK_ERR, std::string("cannot open '") + path + "' for writing");
    const std::string t = format_matrix(ctx, csr, dense);
    out.write(t.data(), std::streamsize(t.size()));
    out.flush();
    if (!out) fail(SK_ERR, std::string("write to '") + path + "' failed");
  });
}
