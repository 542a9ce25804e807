// Matrix Market exchange ("real general", coordinate -> CSR, array -> dense):
// the reference's matio (proj/include/semikern/matio.hpp, proj/src/matio.cpp)
// with the matrix built on the device.  The text is parsed on the host with
// the same rules and messages (std::from_chars, the same field splitting,
// header / size-line / entry checks, 1-based line numbers in ParseError); the
// coordinate entries then go through the device triple builder (stable radix
// sort by (row, col) -> duplicate check -> zero elision -> CSR), whose stable
// order makes "the later of two duplicate lines" the reported one, exactly as
// the reference's sort by (row, col, line) does.
#include <algorithm>
#include <cctype>
#include <charconv>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <sstream>
#include <string>
#include <string_view>
#include <vector>

#include "sk_common.cuh"

namespace sk {
namespace {

constexpr std::string_view kBanner = "%%MatrixMarket";

[[noreturn]] void parse_fail(size_t line, const std::string& msg) {
  fail(SK_ERR_PARSE, "line " + std::to_string(line) + ": " + msg);
}

std::vector<std::string_view> split_fields(std::string_view line) {
  std::vector<std::string_view> f;
  size_t pos = 0;
  while (pos < line.size()) {
    while (pos < line.size() && (line[pos] == ' ' || line[pos] == '\t')) ++pos;
    const size_t b = pos;
    while (pos < line.size() && line[pos] != ' ' && line[pos] != '\t') ++pos;
    if (pos > b) f.push_back(line.substr(b, pos - b));
  }
  return f;
}

std::string lowered(std::string_view s) {
  std::string o(s);
  std::transform(o.begin(), o.end(), o.begin(), [](unsigned char c) { return std::tolower(c); });
  return o;
}

template <typename T>
T parse_number(std::string_view tok, size_t line, const char* what) {
  const char* b = tok.data();
  const char* e = b + tok.size();
  if (b != e && *b == '+') ++b;  // from_chars rejects a leading '+'
  T v{};
  std::from_chars_result r{};
  if constexpr (std::is_floating_point_v<T>)
    r = std::from_chars(b, e, v, std::chars_format::general);
  else
    r = std::from_chars(b, e, v);
  if (r.ec != std::errc{} || r.ptr != e)
    parse_fail(line, std::string("malformed ") + what + " '" + std::string(tok) + "'");
  return v;
}

// std::getline over an in-memory text: '\n'-separated, a final line without a
// newline counts, a trailing '\r' is stripped.
class LineReader {
 public:
  explicit LineReader(std::string_view t) : t_(t) {}
  bool next(std::string_view& line) {
    if (pos_ >= t_.size()) return false;
    const size_t nl = t_.find('\n', pos_);
    const size_t end = nl == std::string_view::npos ? t_.size() : nl;
    line = t_.substr(pos_, end - pos_);
    pos_ = nl == std::string_view::npos ? t_.size() : nl + 1;
    ++lineno_;
    if (!line.empty() && line.back() == '\r') line.remove_suffix(1);
    return true;
  }
  size_t lineno() const { return lineno_; }

 private:
  std::string_view t_;
  size_t pos_ = 0, lineno_ = 0;
};

struct Header {
  bool coordinate;
  size_t size_line;
  std::vector<std::string_view> size_fields;
};

Header read_header(LineReader& rd) {
  std::string_view line;
  if (!rd.next(line)) parse_fail(1, "empty file, expected Matrix Market header");
  const auto f = split_fields(line);
  if (f.empty() || f[0] != kBanner) parse_fail(rd.lineno(), "header must begin '%%MatrixMarket matrix'");
  if (f.size() != 5 || lowered(f[1]) != "matrix")
    parse_fail(rd.lineno(),
               "header must be '%%MatrixMarket matrix <coordinate|array> real general'");
  const std::string format = lowered(f[2]), type = lowered(f[3]), sym = lowered(f[4]);
  if (format != "coordinate" && format != "array")
    parse_fail(rd.lineno(), "unsupported format '" + format + "' (expected coordinate or array)");
  if (type != "real" || sym != "general")
    parse_fail(rd.lineno(), "only 'real general' matrices are supported");
  Header h;
  h.coordinate = format == "coordinate";
  while (true) {  // comments ('%') and blank lines before the size line
    if (!rd.next(line)) parse_fail(rd.lineno() + 1, "unexpected end of file before size line");
    if (!line.empty() && line[0] == '%') continue;
    if (split_fields(line).empty()) continue;
    break;
  }
  h.size_fields = split_fields(line);
  h.size_line = rd.lineno();
  return h;
}

void read_coordinate(sk_ctx* ctx, LineReader& rd, const Header& h, sk_csr** out) {
  if (h.size_fields.size() != 3)
    parse_fail(h.size_line, "coordinate size line must be 'rows cols nnz'");
  const auto rows = parse_number<uint32_t>(h.size_fields[0], h.size_line, "row count");
  const auto cols = parse_number<uint32_t>(h.size_fields[1], h.size_line, "column count");
  const auto count = parse_number<size_t>(h.size_fields[2], h.size_line, "nnz count");
  std::vector<uint32_t> r, c;
  std::vector<float> v;
  std::vector<size_t> lines;
  const size_t res = std::min(count, size_t(1) << 20);
  r.reserve(res);
  c.reserve(res);
  v.reserve(res);
  lines.reserve(res);
  std::string_view line;
  while (r.size() < count) {
    if (!rd.next(line))
      parse_fail(rd.lineno() + 1, "unexpected end of file: expected " + std::to_string(count) +
                                      " entries, found " + std::to_string(r.size()));
    const auto f = split_fields(line);
    if (f.empty()) continue;
    if (f.size() != 3)
      parse_fail(rd.lineno(),
                 "entry must have 3 fields 'row col value', found " + std::to_string(f.size()));
    const auto ri = parse_number<uint64_t>(f[0], rd.lineno(), "row index");
    const auto ci = parse_number<uint64_t>(f[1], rd.lineno(), "column index");
    const auto vi = parse_number<float>(f[2], rd.lineno(), "value");
    if (ri < 1 || ri > rows)
      parse_fail(rd.lineno(), "row index " + std::to_string(ri) + " out of range [1, " +
                                  std::to_string(rows) + "]");
    if (ci < 1 || ci > cols)
      parse_fail(rd.lineno(), "column index " + std::to_string(ci) + " out of range [1, " +
                                  std::to_string(cols) + "]");
    r.push_back(uint32_t(ri - 1));
    c.push_back(uint32_t(ci - 1));
    v.push_back(vi);
    lines.push_back(rd.lineno());
  }
  while (rd.next(line))
    if (!split_fields(line).empty())
      parse_fail(rd.lineno(), "unexpected content after " + std::to_string(count) + " entries");

  const size_t n = r.size();
  uint32_t* dr = dalloc<uint32_t>(ctx, std::max<size_t>(n, 1));
  uint32_t* dc = dalloc<uint32_t>(ctx, std::max<size_t>(n, 1));
  float* dv = dalloc<float>(ctx, std::max<size_t>(n, 1));
  if (n) {
    SK_CUDA(cudaMemcpyAsync(dr, r.data(), n * 4, cudaMemcpyHostToDevice, ctx->stream));
    SK_CUDA(cudaMemcpyAsync(dc, c.data(), n * 4, cudaMemcpyHostToDevice, ctx->stream));
    SK_CUDA(cudaMemcpyAsync(dv, v.data(), n * 4, cudaMemcpyHostToDevice, ctx->stream));
  }
  uint64_t dup = ~0ull;
  sk_csr* a = nullptr;
  try {
    a = csr_from_device_triples(ctx, rows, cols, dr, dc, dv, n, r.data(), c.data(), &dup);
  } catch (...) {
    dfree(ctx, dr);
    dfree(ctx, dc);
    dfree(ctx, dv);
    throw;
  }
  dfree(ctx, dr);
  dfree(ctx, dc);
  dfree(ctx, dv);
  if (!a)
    parse_fail(lines[dup], "duplicate entry for (" + std::to_string(r[dup] + 1) + ", " +
                               std::to_string(c[dup] + 1) + ")");
  *out = a;
}

void read_array(sk_ctx* ctx, LineReader& rd, const Header& h, sk_dense** out) {
  if (h.size_fields.size() != 2) parse_fail(h.size_line, "array size line must be 'rows cols'");
  const auto rows = parse_number<uint32_t>(h.size_fields[0], h.size_line, "row count");
  const auto cols = parse_number<uint32_t>(h.size_fields[1], h.size_line, "column count");
  const size_t count = size_t(rows) * cols;
  std::vector<float> host(count, 0.0f);
  std::string_view line;
  size_t filled = 0;
  while (filled < count) {
    if (!rd.next(line))
      parse_fail(rd.lineno() + 1, "unexpected end of file: expected " + std::to_string(count) +
                                      " values, found " + std::to_string(filled));
    const auto f = split_fields(line);
    if (f.empty()) continue;
    if (f.size() != 1)
      parse_fail(rd.lineno(), "array lines carry one value each, found " + std::to_string(f.size()));
    const auto v = parse_number<float>(f[0], rd.lineno(), "value");
    const uint32_t i = uint32_t(filled % rows), j = uint32_t(filled / rows);  // column-major
    host[size_t(i) * cols + j] = v;
    ++filled;
  }
  while (rd.next(line))
    if (!split_fields(line).empty())
      parse_fail(rd.lineno(), "unexpected content after " + std::to_string(count) + " values");
  sk_dense* d = new_dense(ctx, rows, cols);
  if (count)
    SK_CUDA(cudaMemcpyAsync(d->d, host.data(), count * 4, cudaMemcpyHostToDevice, ctx->stream));
  sync(ctx);
  *out = d;
}

void read_text(sk_ctx* ctx, std::string_view text, int* kind, sk_csr** csr, sk_dense** dense) {
  LineReader rd(text);
  const Header h = read_header(rd);
  *csr = nullptr;
  *dense = nullptr;
  if (h.coordinate) {
    *kind = 0;
    read_coordinate(ctx, rd, h, csr);
  } else {
    *kind = 1;
    read_array(ctx, rd, h, dense);
  }
}

void append_value(std::string& s, float v) {
  char buf[48];
  std::snprintf(buf, sizeof buf, "%.9g", double(v));
  s += buf;
}

std::string format_matrix(sk_ctx* ctx, const sk_csr* a, const sk_dense* d) {
  std::string o;
  if (a) {
    std::vector<uint32_t> rp(size_t(a->rows) + 1), ci(a->nnz);
    std::vector<float> v(a->nnz);
    SK_CUDA(cudaMemcpyAsync(rp.data(), a->rp, rp.size() * 4, cudaMemcpyDeviceToHost, ctx->stream));
    if (a->nnz) {
      SK_CUDA(cudaMemcpyAsync(ci.data(), a->ci, a->nnz * 4, cudaMemcpyDeviceToHost, ctx->stream));
      SK_CUDA(cudaMemcpyAsync(v.data(), a->v, a->nnz * 4, cudaMemcpyDeviceToHost, ctx->stream));
    }
    sync(ctx);
    o += std::string(kBanner) + " matrix coordinate real general\n";
    o += std::to_string(a->rows) + ' ' + std::to_string(a->cols) + ' ' + std::to_string(a->nnz) + '\n';
    o.reserve(o.size() + a->nnz * 24);
    for (uint32_t i = 0; i < a->rows; ++i)
      for (uint32_t e = rp[i]; e < rp[i + 1]; ++e) {
        o += std::to_string(i + 1);
        o += ' ';
        o += std::to_string(ci[e] + 1);
        o += ' ';
        append_value(o, v[e]);
        o += '\n';
      }
  } else {
    std::vector<float> h(d->elems());
    if (!h.empty())
      SK_CUDA(cudaMemcpyAsync(h.data(), d->d, h.size() * 4, cudaMemcpyDeviceToHost, ctx->stream));
    sync(ctx);
    o += std::string(kBanner) + " matrix array real general\n";
    o += std::to_string(d->rows) + ' ' + std::to_string(d->cols) + '\n';
    for (uint32_t j = 0; j < d->cols; ++j)  // values down each column
      for (uint32_t i = 0; i < d->rows; ++i) {
        append_value(o, h[size_t(i) * d->cols + j]);
        o += '\n';
      }
  }
  return o;
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
    std::stringstream ss;
    ss << in.rdbuf();
    const std::string text = ss.str();
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
    out << format_matrix(ctx, csr, dense);
    out.flush();
    if (!out) fail(SK_ERR, std::string("write to '") + path + "' failed");
  });
}
