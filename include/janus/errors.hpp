// janus/errors.hpp — exception vocabulary of the janus schedule API.
//
// Drop-in for the reference's proj/include/janus/errors.hpp:8-33: the same five
// exception types, the same std:: base classes, and parse_error's 1-based line
// number.  Additionally defines the integer status codes that the C ABI
// (include/janus_cuda.h) returns instead of throwing, plus the mapping between
// the two, so C++ callers of the ABI get the familiar exception types back.
#pragma once

#include <stdexcept>
#include <string>

namespace janus {

/// Argument value outside its domain (stage index, k, pipeline degree ...).
struct domain_error : std::invalid_argument {
  explicit domain_error(const std::string& msg) : std::invalid_argument(msg) {}
};

/// An operation was applied to an object that is in the wrong state.
struct state_error : std::logic_error {
  explicit state_error(const std::string& msg) : std::logic_error(msg) {}
};

/// Malformed schedule text.  `line` is 1-based; 0 means "unknown".
struct parse_error : std::runtime_error {
  parse_error(const std::string& msg, int line_no = 0)
      : std::runtime_error(line_no > 0 ? ("line " + std::to_string(line_no) + ": " + msg) : msg),
        line(line_no) {}
  int line = 0;
};

/// A replay / executor found work remaining but nothing runnable.
struct deadlock_error : std::runtime_error {
  explicit deadlock_error(const std::string& msg) : std::runtime_error(msg) {}
};

/// Inconsistent configuration (odd P for 1F1B-2nd, bad model shape ...).
struct config_error : std::invalid_argument {
  explicit config_error(const std::string& msg) : std::invalid_argument(msg) {}
};

/// Status codes used across the C ABI.  0 is success; each error kind above has
/// its own code, plus the device-side failures that have no C++ analogue.
enum Status : int {
  kOk = 0,
  kDomainError = 1,
  kStateError = 2,
  kParseError = 3,
  kDeadlockError = 4,
  kConfigError = 5,
  kCudaError = 6,
  kNcclError = 7,
  kOutOfMemory = 8,
  kInternalError = 9,
};

/// Re-raise an ABI status as the matching exception type (no-op for kOk).
[[noreturn]] inline void throw_status(int status, const std::string& msg) {
  switch (status) {
    case kDomainError: throw domain_error(msg);
    case kStateError: throw state_error(msg);
    case kParseError: throw parse_error(msg);
    case kDeadlockError: throw deadlock_error(msg);
    case kConfigError: throw config_error(msg);
    default: throw std::runtime_error(msg);
  }
}

inline void check_status(int status, const char* msg) {
  if (status != kOk) throw_status(status, msg ? msg : "janus: unknown error");
}

}  // namespace janus
