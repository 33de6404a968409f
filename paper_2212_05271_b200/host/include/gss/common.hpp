// gss/common.hpp (B200 build) -- the reference's error classes (common.hpp:17-79) and the device
// context the operators of this build run on. Drop-in for the reference header of the same name on the
// enhance_batch path: same namespace, class names and semantics; the arithmetic behind every operator
// lives in libgss_b200.so (include/gss_b200.h), there is no host implementation.
#pragma once

#include <complex>
#include <cstdint>
#include <stdexcept>
#include <string>

#include "gss_b200.h"

namespace gss {

using cfloat = std::complex<float>;
using cdouble = std::complex<double>;

class Error : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};
class ShapeError : public Error { public: using Error::Error; };
class ConfigError : public Error { public: using Error::Error; };
class ParseError : public Error { public: using Error::Error; };
class IoError : public Error { public: using Error::Error; };
class SingularMatrixError : public Error {
 public:
  explicit SingularMatrixError(const std::string& msg, long frequency = -1) : Error(msg), frequency_(frequency) {}
  long frequency() const { return frequency_; }

 private:
  long frequency_ = -1;
};
class InputTooShortError : public Error { public: using Error::Error; };
class EmptyTargetError : public Error { public: using Error::Error; };
class DegenerateStatsError : public Error { public: using Error::Error; };
class SpecError : public Error { public: using Error::Error; };
/// Not in the reference: device / driver failures and shapes outside the compiled kernel range.
class DeviceError : public Error { public: using Error::Error; };

namespace b200 {

/// Re-raises a C-ABI status as the exception class the reference would throw.
[[noreturn]] inline void raise(int status, const std::string& msg, long frequency = -1) {
  switch (status) {
    case GSS_SHAPE_ERROR: throw ShapeError(msg);
    case GSS_CONFIG_ERROR: throw ConfigError(msg);
    case GSS_PARSE_ERROR: throw ParseError(msg);
    case GSS_IO_ERROR: throw IoError(msg);
    case GSS_SINGULAR_MATRIX_ERROR: throw SingularMatrixError(msg, frequency);
    case GSS_INPUT_TOO_SHORT_ERROR: throw InputTooShortError(msg);
    case GSS_EMPTY_TARGET_ERROR: throw EmptyTargetError(msg);
    case GSS_DEGENERATE_STATS_ERROR: throw DegenerateStatsError(msg);
    case GSS_SPEC_ERROR: throw SpecError(msg);
    default: throw DeviceError(msg);
  }
}

/// One gss_b200_ctx (a device, a stream, its workspaces). One per host thread and device.
class Device {
 public:
  explicit Device(int index = 0) {
    const gss_status st = gss_b200_create(index, &ctx_);
    if (st != GSS_OK) raise(st, gss_b200_last_error(nullptr));
  }
  ~Device() { gss_b200_destroy(ctx_); }
  Device(const Device&) = delete;
  Device& operator=(const Device&) = delete;
  gss_b200_ctx* get() const { return ctx_; }
  void check(gss_status st) const {
    if (st != GSS_OK) raise(st, gss_b200_last_error(ctx_), static_cast<long>(gss_b200_last_error_frequency(ctx_)));
  }
  /// The calling thread's default device (GSS_B200_DEVICE, else 0), created on first use.
  static Device& current() {
    static thread_local Device dev(default_index());
    return dev;
  }

 private:
  static int default_index() {
    const char* s = std::getenv("GSS_B200_DEVICE");
    return s ? std::atoi(s) : 0;
  }
  gss_b200_ctx* ctx_ = nullptr;
};

inline void check_host(gss_status st) {
  if (st != GSS_OK) raise(st, gss_b200_last_error(nullptr));
}

}  // namespace b200
}  // namespace gss
