// semikern/error.hpp (B200 shim) -- the reference's exception hierarchy
// (proj/include/semikern/error.hpp:24-58).  A program built against the
// reference compiles against this directory instead (-I include/semikern_b200);
// every call below the headers runs on the B200 through include/sk_api.h.
#pragma once

#include <cstddef>
#include <stdexcept>
#include <string>

namespace semikern {

class Error : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};
class DimensionError : public Error {
 public:
  using Error::Error;
};
class DomainError : public Error {
 public:
  using Error::Error;
};
class InvalidArgument : public Error {
 public:
  using Error::Error;
};
class ParseError : public Error {
 public:
  ParseError(std::size_t line, const std::string& message)
      : Error("line " + std::to_string(line) + ": " + message), line_(line) {}
  std::size_t line() const noexcept { return line_; }

 private:
  std::size_t line_;
};
/// Device allocation failed (extension; the sweep reports it as a SkippedRun,
/// where the reference catches std::bad_alloc).
class OutOfMemory : public Error {
 public:
  using Error::Error;
};

}  // namespace semikern
