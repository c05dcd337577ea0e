// Shared error type and status codes.  Mirrors the reference's error categories
// (proj/include/ffit/errors.hpp:9-24) so the C ABI can keep its status-code
// contract (proj/include/ffit.h:20-25, proj/src/capi.cpp:40-50).
#pragma once

#include <stdexcept>
#include <string>

namespace ffb {

enum class ErrorCode { Usage = 1, Data = 2, Numeric = 3 };

class Error : public std::runtime_error {
 public:
  Error(ErrorCode code, const std::string& message)
      : std::runtime_error(message), code_(code) {}
  ErrorCode code() const { return code_; }

 private:
  ErrorCode code_;
};

[[noreturn]] inline void usage_error(const std::string& m) { throw Error(ErrorCode::Usage, m); }
[[noreturn]] inline void data_error(const std::string& m) { throw Error(ErrorCode::Data, m); }
[[noreturn]] inline void numeric_error(const std::string& m) { throw Error(ErrorCode::Numeric, m); }

}  // namespace ffb
