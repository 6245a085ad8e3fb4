// Error type shared by the host-side C++ of libfmmlu.
#pragma once
#include <stdexcept>
#include <string>

namespace fmmlu {
struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};
}  // namespace fmmlu
