// semikern/matio.hpp (B200 shim) -- Matrix Market exchange
// (proj/include/semikern/matio.hpp:23-55).  Parsing and formatting run in the
// library's host C++ (csrc/matio.cpp, the reference's rules and messages); a
// coordinate file becomes a device CSR, an array file a device dense matrix.
#pragma once

#include <cstddef>
#include <filesystem>
#include <iterator>
#include <ostream>
#include <istream>
#include <string>

#include "matrix.hpp"

namespace semikern {

enum class MatrixFileKind { coordinate, array };

struct MatrixFileInfo {
  std::filesystem::path path;
  MatrixFileKind kind;
  index_t rows = 0;
  index_t cols = 0;
  std::size_t entries = 0;  // nnz for coordinate, rows*cols for array
};

namespace detail {
inline MatrixFileInfo file_info(const Matrix& a, std::filesystem::path path) {
  MatrixFileInfo info{std::move(path), a.is_sparse() ? MatrixFileKind::coordinate
                                                     : MatrixFileKind::array,
                      a.rows(), a.cols(), 0};
  info.entries = a.is_sparse() ? a.csr().nnz()
                               : static_cast<std::size_t>(a.rows()) * a.cols();
  return info;
}
inline Matrix adopt_read(int kind, sk_csr* csr, sk_dense* dense) {
  if (kind == 0) return Matrix(CsrMatrix::from_handle(csr));
  return Matrix(DenseMatrix::from_handle(dense));
}
}  // namespace detail

inline MatrixFileInfo write_matrix(const Matrix& a, const std::filesystem::path& path) {
  detail::check(sk_write_matrix(detail::ctx(), a.is_sparse() ? a.csr().handle() : nullptr,
                                a.is_sparse() ? nullptr : a.dense().handle(),
                                path.string().c_str()));
  return detail::file_info(a, path);
}
inline MatrixFileInfo write_matrix(const Matrix& a, std::ostream& out) {
  const sk_csr* c = a.is_sparse() ? a.csr().handle() : nullptr;
  const sk_dense* d = a.is_sparse() ? nullptr : a.dense().handle();
  std::size_t len = 0;
  detail::check(sk_format_matrix(detail::ctx(), c, d, nullptr, 0, &len));
  std::string text(len + 1, '\0');
  detail::check(sk_format_matrix(detail::ctx(), c, d, text.data(), text.size(), &len));
  out.write(text.data(), static_cast<std::streamsize>(len));
  if (!out) throw Error("write failed");
  return detail::file_info(a, {});
}

inline Matrix read_matrix(const std::filesystem::path& path) {
  int kind = 0;
  sk_csr* c = nullptr;
  sk_dense* d = nullptr;
  detail::check(sk_read_matrix(detail::ctx(), path.string().c_str(), &kind, &c, &d));
  return detail::adopt_read(kind, c, d);
}
inline Matrix read_matrix(std::istream& in) {
  const std::string text((std::istreambuf_iterator<char>(in)), std::istreambuf_iterator<char>());
  int kind = 0;
  sk_csr* c = nullptr;
  sk_dense* d = nullptr;
  detail::check(sk_read_matrix_text(detail::ctx(), text.data(), text.size(), &kind, &c, &d));
  return detail::adopt_read(kind, c, d);
}

}  // namespace semikern
