// Error taxonomy of the host API. Mirrors the reference's exception classes
// one-for-one (R:proj/include/pipeshard/errors.hpp:26-59) so callers can keep
// their catch sites, and adds CudaError for the device layer. Across the
// C-ABI (include/mgg.h) each class maps to a status code: InputError 1,
// ParseError 2, ConfigError 3, IntegrityError 4, CudaError 5.
#pragma once

#include <cstddef>
#include <stdexcept>
#include <string>

namespace mgg {

class InputError : public std::runtime_error {
 public:
  explicit InputError(const std::string& what) : std::runtime_error(what) {}
};

/// Carries the 1-based line number for line-oriented sources, 0 otherwise
/// (R:proj/include/pipeshard/errors.hpp:33-46).
class ParseError : public InputError {
 public:
  ParseError(const std::string& what, std::size_t line)
      : InputError(line ? what + " (line " + std::to_string(line) + ")" : what),
        line_(line) {}
  std::size_t line() const { return line_; }

 private:
  std::size_t line_;
};

class ConfigError : public std::runtime_error {
 public:
  explicit ConfigError(const std::string& what) : std::runtime_error(what) {}
};

class IntegrityError : public std::runtime_error {
 public:
  explicit IntegrityError(const std::string& what) : std::runtime_error(what) {}
};

/// A CUDA runtime/driver call failed (no reference counterpart: the
/// reference never touches a device).
class CudaError : public std::runtime_error {
 public:
  explicit CudaError(const std::string& what) : std::runtime_error(what) {}
};

}  // namespace mgg
