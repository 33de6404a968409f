// gss_oracle.hpp -- CPU ORACLE (test infrastructure, NOT the product).
//
// An Eigen-free restatement of the reference's guided-source-separation hot
// path (`scheduler::enhance_batch` and the stage functions it calls). Only
// tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
// reference legs may build, link or call this file. The product
// (paper_2212_05271_b200/csrc) never includes it.
//
// Why a restatement: the reference (/root/reference/proj, header-only C++20)
// needs Eigen >= 3.3 (proj/CMakeLists.txt:17-22), which is not vendored and is
// absent from this image, so the reference itself cannot be compiled here.
// The arithmetic Eigen supplies (LLT, SelfAdjointEigenSolver, cfloat GEMM,
// FFT<double>) is replaced by the plain-loop equivalents below; precision
// choices (double factorizations, float Gram chunks of 2048 rows summed in
// double, float log q, double log-sum-exp, ...) follow the reference.
//
// Parity is PINNED: tests/test_oracle_golden.py checks this file against every
// frozen known-answer value in the reference's own test-suite.
//
// Each function cites the reference file:line it follows
// (paths relative to /root/reference/proj/include/gss/).
#pragma once

#include <algorithm>
#include <cmath>
#include <complex>
#include <cstdint>
#include <cstdlib>
#include <functional>
#include <limits>
#include <set>
#include <stdexcept>
#include <string>
#include <thread>
#include <utility>
#include <vector>

namespace gss_oracle {

using cf = std::complex<float>;
using cd = std::complex<double>;

// ---------------------------------------------------------------------------
// Errors -- one exception type carrying the reference's class as a code
// (common.hpp:17-79). Codes are shared with include/gss_b200.h.
// ---------------------------------------------------------------------------
enum ErrCode {
  kOk = 0,
  kShapeError = 1,
  kConfigError = 2,
  kParseError = 3,
  kIoError = 4,
  kSingularMatrixError = 5,
  kInputTooShortError = 6,
  kEmptyTargetError = 7,
  kDegenerateStatsError = 8,
  kSpecError = 9,
};

struct OracleError : std::runtime_error {
  int code;
  long frequency;
  OracleError(int c, const std::string& m, long f = -1)
      : std::runtime_error(m), code(c), frequency(f) {}
};

// ---------------------------------------------------------------------------
// parallel_for (parallel.hpp:14-51): contiguous blocks, fresh threads per call
// ---------------------------------------------------------------------------
inline int& thread_override() {
  static int n = 0;
  return n;
}

inline int hardware_threads() {
  if (thread_override() > 0) return thread_override();
  if (const char* env = std::getenv("GSS_THREADS")) {
    int v = std::atoi(env);
    if (v > 0) return v;
  }
  unsigned hc = std::thread::hardware_concurrency();
  return hc > 0 ? static_cast<int>(hc) : 1;
}

template <typename Body>
inline void parallel_for(int64_t n, Body&& body) {
  int threads = static_cast<int>(std::min<int64_t>(hardware_threads(), n));
  if (threads <= 1) {
    for (int64_t i = 0; i < n; ++i) body(i);
    return;
  }
  const int64_t chunk = (n + threads - 1) / threads;
  std::vector<std::thread> pool;
  std::vector<std::exception_ptr> errs(threads);
  auto run = [&](int tid, int64_t b, int64_t e) {
    try {
      for (int64_t i = b; i < e; ++i) body(i);
    } catch (...) {
      errs[tid] = std::current_exception();
    }
  };
  for (int t = 1; t < threads; ++t) {
    int64_t b = t * chunk, e = std::min<int64_t>(n, b + chunk);
    if (b >= e) break;
    pool.emplace_back(run, t, b, e);
  }
  run(0, 0, std::min<int64_t>(n, chunk));
  for (auto& th : pool) th.join();
  for (auto& e : errs)
    if (e) std::rethrow_exception(e);
}

// ---------------------------------------------------------------------------
// Dense complex-double matrix, column-major (stands in for Eigen::MatrixXcd)
// ---------------------------------------------------------------------------
struct CMat {
  int r = 0, c = 0;
  std::vector<cd> v;
  CMat() = default;
  CMat(int rows, int cols) : r(rows), c(cols), v(static_cast<size_t>(rows) * cols) {}
  cd& operator()(int i, int j) { return v[static_cast<size_t>(j) * r + i]; }
  const cd& operator()(int i, int j) const { return v[static_cast<size_t>(j) * r + i]; }
  static CMat identity(int n) {
    CMat m(n, n);
    for (int i = 0; i < n; ++i) m(i, i) = 1.0;
    return m;
  }
};

constexpr double kDefaultRegEps = 1e-10;         // numerics.hpp:28
constexpr double kEigenvalueFloorRatio = 1e-10;  // numerics.hpp:29

/// (A + A^H)/2 -- numerics.hpp:32-38
inline CMat hermitize(const CMat& a) {
  if (a.r != a.c) throw OracleError(kShapeError, "hermitize: matrix is not square");
  CMat o(a.r, a.c);
  for (int j = 0; j < a.c; ++j)
    for (int i = 0; i < a.r; ++i) o(i, j) = 0.5 * (a(i, j) + std::conj(a(j, i)));
  return o;
}

/// A + eps*(tr(A)/M)*I, scale -> 1 when the trace is not positive -- numerics.hpp:41-49
inline CMat regularize(const CMat& a, double eps = kDefaultRegEps) {
  double tr = 0;
  for (int i = 0; i < a.r; ++i) tr += a(i, i).real();
  double scale = tr / static_cast<double>(a.r);
  if (!(scale > 0.0)) scale = 1.0;
  CMat o = a;
  for (int i = 0; i < a.r; ++i) o(i, i) += eps * scale;
  return o;
}

/// In-place lower Cholesky reading only the lower triangle (what
/// Eigen::LLT<MatrixXcd, Lower> does, numerics.hpp:88,105). Fails iff a pivot
/// x = Re(a_kk) - |row|^2 satisfies x <= 0 (Eigen's llt_inplace criterion).
inline bool cholesky_lower(CMat& a) {
  const int n = a.r;
  for (int k = 0; k < n; ++k) {
    double x = a(k, k).real();
    for (int j = 0; j < k; ++j) x -= std::norm(a(k, j));
    if (x <= 0.0) return false;
    x = std::sqrt(x);
    a(k, k) = x;
    for (int i = k + 1; i < n; ++i) {
      cd s = a(i, k);
      for (int j = 0; j < k; ++j) s -= a(i, j) * std::conj(a(k, j));
      a(i, k) = s / x;
    }
  }
  return true;
}

/// Solve L L^H X = B given the factor in the lower triangle of l.
inline CMat cholesky_solve(const CMat& l, const CMat& b) {
  const int n = l.r;
  CMat x = b;
  for (int col = 0; col < b.c; ++col) {
    for (int i = 0; i < n; ++i) {
      cd s = x(i, col);
      for (int j = 0; j < i; ++j) s -= l(i, j) * x(j, col);
      x(i, col) = s / l(i, i).real();
    }
    for (int i = n - 1; i >= 0; --i) {
      cd s = x(i, col);
      for (int j = i + 1; j < n; ++j) s -= std::conj(l(j, i)) * x(j, col);
      x(i, col) = s / l(i, i).real();
    }
  }
  return x;
}

/// Hermitian eigendecomposition by cyclic two-sided Jacobi (stands in for
/// Eigen::SelfAdjointEigenSolver, numerics.hpp:59). Uses the lower triangle.
/// Returns false if the iteration produced non-finite values.
inline bool hermitian_eig(const CMat& a_in, CMat& vecs, std::vector<double>& vals) {
  const int n = a_in.r;
  CMat a(n, n);
  for (int j = 0; j < n; ++j)
    for (int i = j; i < n; ++i) {
      a(i, j) = a_in(i, j);
      a(j, i) = std::conj(a_in(i, j));
    }
  for (int i = 0; i < n; ++i) a(i, i) = a(i, i).real();
  vecs = CMat::identity(n);
  for (int sweep = 0; sweep < 60; ++sweep) {
    double off = 0, diag = 0;
    for (int j = 0; j < n; ++j)
      for (int i = 0; i < n; ++i) (i == j ? diag : off) += std::norm(a(i, j));
    if (!std::isfinite(off + diag)) return false;
    if (off <= 1e-30 * diag || off == 0.0) break;
    for (int p = 0; p < n - 1; ++p) {
      for (int q = p + 1; q < n; ++q) {
        const cd apq = a(p, q);
        const double mag = std::abs(apq);
        if (mag == 0.0) continue;
        const double app = a(p, p).real(), aqq = a(q, q).real();
        const cd phase = apq / mag;  // e^{i phi}
        const double tau = (aqq - app) / (2.0 * mag);
        const double t = (tau >= 0 ? 1.0 : -1.0) / (std::abs(tau) + std::sqrt(1.0 + tau * tau));
        const double c = 1.0 / std::sqrt(1.0 + t * t);
        const double s = t * c;
        // J columns: p -> [c ; -s e^{-i phi}], q -> [s ; c e^{-i phi}]
        const cd jpp = c, jqp = -s * std::conj(phase), jpq = s, jqq = c * std::conj(phase);
        for (int i = 0; i < n; ++i) {  // A <- A J (columns p,q)
          const cd aip = a(i, p), aiq = a(i, q);
          a(i, p) = aip * jpp + aiq * jqp;
          a(i, q) = aip * jpq + aiq * jqq;
        }
        for (int j = 0; j < n; ++j) {  // A <- J^H A (rows p,q)
          const cd apj = a(p, j), aqj = a(q, j);
          a(p, j) = std::conj(jpp) * apj + std::conj(jqp) * aqj;
          a(q, j) = std::conj(jpq) * apj + std::conj(jqq) * aqj;
        }
        a(p, q) = 0.0;
        a(q, p) = 0.0;
        a(p, p) = a(p, p).real();
        a(q, q) = a(q, q).real();
        for (int i = 0; i < n; ++i) {  // V <- V J
          const cd vip = vecs(i, p), viq = vecs(i, q);
          vecs(i, p) = vip * jpp + viq * jqp;
          vecs(i, q) = vip * jpq + viq * jqq;
        }
      }
    }
  }
  vals.resize(n);
  for (int i = 0; i < n; ++i) {
    vals[i] = a(i, i).real();
    if (!std::isfinite(vals[i])) return false;
  }
  return true;
}

struct EigenFloored {
  CMat vectors;
  std::vector<double> values;
};

/// numerics.hpp:58-73
inline EigenFloored eigen_floor(const CMat& a, long frequency) {
  EigenFloored ef;
  if (!hermitian_eig(a, ef.vectors, ef.values))
    throw OracleError(kSingularMatrixError, "eigendecomposition failed", frequency);
  double emax = -std::numeric_limits<double>::infinity();
  for (double v : ef.values) emax = std::max(emax, v);
  if (!(emax > 0.0) || !std::isfinite(emax))
    throw OracleError(kSingularMatrixError, "matrix has no positive eigenvalue", frequency);
  const double floor = kEigenvalueFloorRatio * emax;
  for (double& v : ef.values) v = std::max(v, floor);
  return ef;
}

/// V diag(1/lambda) V^H B
inline CMat eig_apply_inverse(const EigenFloored& ef, const CMat& b) {
  const int n = ef.vectors.r;
  CMat tmp(n, b.c), out(n, b.c);
  for (int col = 0; col < b.c; ++col)
    for (int i = 0; i < n; ++i) {
      cd s = 0;
      for (int j = 0; j < n; ++j) s += std::conj(ef.vectors(j, i)) * b(j, col);
      tmp(i, col) = s / ef.values[i];
    }
  for (int col = 0; col < b.c; ++col)
    for (int i = 0; i < n; ++i) {
      cd s = 0;
      for (int j = 0; j < n; ++j) s += ef.vectors(i, j) * tmp(j, col);
      out(i, col) = s;
    }
  return out;
}

/// numerics.hpp:81-94
inline CMat hermitian_solve(const CMat& a, const CMat& b, long frequency = -1) {
  if (a.r != a.c || a.r != b.r)
    throw OracleError(kShapeError, "hermitian_solve: shape mismatch");
  CMat l = a;
  if (cholesky_lower(l)) return cholesky_solve(l, b);
  return eig_apply_inverse(eigen_floor(a, frequency), b);
}

struct InverseLogDet {
  CMat inverse;
  double log_det = 0.0;
};

/// numerics.hpp:103-122
inline InverseLogDet hermitian_inverse_logdet(const CMat& a, long frequency = -1) {
  InverseLogDet out;
  CMat l = a;
  if (cholesky_lower(l)) {
    double ld = 0;
    for (int i = 0; i < a.r; ++i) ld += std::log(l(i, i).real());
    out.log_det = 2.0 * ld;
    out.inverse = cholesky_solve(l, CMat::identity(a.r));
    return out;
  }
  EigenFloored ef = eigen_floor(a, frequency);
  for (double v : ef.values) out.log_det += std::log(v);
  out.inverse = eig_apply_inverse(ef, CMat::identity(a.r));
  return out;
}

/// Sum_t w[t] y_t y_t^H over rows of a (rows x cols row-major cfloat):
/// sqrt(w) row scaling in float, float Gram per 2048-row chunk, double across
/// chunks; entry (m,n) = Sum w y_m conj(y_n) -- numerics.hpp:128-152.
/// (Eigen forms the full square with a cfloat GEMM; this port forms the lower
/// triangle with planar float dot products and mirrors it.)
#ifdef GSS_ORACLE_VECTOR_GRAM
// TIMING-ONLY variant (bench.py's CPU arm; never the parity checker): the same chunked float Gram with
// double cross-chunk accumulation, but each dot product runs on kLanes independent partial sums that the
// compiler maps to SIMD registers (no -ffast-math needed), two rows of the triangle per pass over a column.
// This is what Eigen's cfloat GEMM buys the reference; the summation order inside a chunk differs from the
// scalar port below (tests/test_oracle_golden.py::test_vector_gram_variant_agrees bounds the difference).
inline CMat weighted_gram(const cf* a, int64_t rows, int cols, const float* w,
                          int64_t chunk = 2048) {
  constexpr int kLanes = 16;
  CMat acc(cols, cols);
  const int64_t pitch = (chunk + kLanes - 1) / kLanes * kLanes;
  std::vector<float> re(static_cast<size_t>(cols) * pitch), im(static_cast<size_t>(cols) * pitch);
  for (int64_t t0 = 0; t0 < rows; t0 += chunk) {
    const int64_t n = std::min<int64_t>(chunk, rows - t0);
    const int64_t np = (n + kLanes - 1) / kLanes * kLanes;
    for (int64_t t = 0; t < n; ++t) {
      const float s = w ? std::sqrt(std::max(0.0f, w[t0 + t])) : 1.0f;
      const cf* row = a + (t0 + t) * cols;
      for (int c = 0; c < cols; ++c) {
        re[static_cast<size_t>(c) * pitch + t] = row[c].real() * s;
        im[static_cast<size_t>(c) * pitch + t] = row[c].imag() * s;
      }
    }
    for (int c = 0; c < cols; ++c)
      for (int64_t t = n; t < np; ++t) re[static_cast<size_t>(c) * pitch + t] = im[static_cast<size_t>(c) * pitch + t] = 0.0f;
    for (int i = 0; i < cols; i += 2) {
      const bool two = i + 1 < cols;
      const float* r0 = &re[static_cast<size_t>(i) * pitch];
      const float* i0 = &im[static_cast<size_t>(i) * pitch];
      const float* r1 = two ? r0 + pitch : r0;
      const float* i1 = two ? i0 + pitch : i0;
      for (int j = 0; j <= (two ? i + 1 : i); ++j) {
        const float* rj = &re[static_cast<size_t>(j) * pitch];
        const float* ij = &im[static_cast<size_t>(j) * pitch];
        float ar0[kLanes] = {0}, ai0[kLanes] = {0}, ar1[kLanes] = {0}, ai1[kLanes] = {0};
        for (int64_t t = 0; t < np; t += kLanes) {
          for (int l = 0; l < kLanes; ++l) {
            const float a_r = rj[t + l], a_i = ij[t + l];
            ar0[l] += r0[t + l] * a_r + i0[t + l] * a_i;
            ai0[l] += i0[t + l] * a_r - r0[t + l] * a_i;
            ar1[l] += r1[t + l] * a_r + i1[t + l] * a_i;
            ai1[l] += i1[t + l] * a_r - r1[t + l] * a_i;
          }
        }
        float sr0 = 0, si0 = 0, sr1 = 0, si1 = 0;
        for (int l = 0; l < kLanes; ++l) {
          sr0 += ar0[l];
          si0 += ai0[l];
          sr1 += ar1[l];
          si1 += ai1[l];
        }
        if (j <= i) {
          acc(i, j) += cd(sr0, si0);
          if (j != i) acc(j, i) += cd(sr0, -si0);
        }
        if (two) {
          acc(i + 1, j) += cd(sr1, si1);
          if (j != i + 1) acc(j, i + 1) += cd(sr1, -si1);
        }
      }
    }
  }
  return acc;
}
#else
inline CMat weighted_gram(const cf* a, int64_t rows, int cols, const float* w,
                          int64_t chunk = 2048) {
  CMat acc(cols, cols);
  std::vector<float> re(static_cast<size_t>(cols) * chunk), im(static_cast<size_t>(cols) * chunk);
  for (int64_t t0 = 0; t0 < rows; t0 += chunk) {
    const int64_t n = std::min<int64_t>(chunk, rows - t0);
    for (int64_t t = 0; t < n; ++t) {
      const float s = w ? std::sqrt(std::max(0.0f, w[t0 + t])) : 1.0f;
      const cf* row = a + (t0 + t) * cols;
      for (int c = 0; c < cols; ++c) {
        re[static_cast<size_t>(c) * chunk + t] = row[c].real() * s;
        im[static_cast<size_t>(c) * chunk + t] = row[c].imag() * s;
      }
    }
    for (int i = 0; i < cols; ++i) {
      const float* ri = &re[static_cast<size_t>(i) * chunk];
      const float* ii = &im[static_cast<size_t>(i) * chunk];
      for (int j = 0; j <= i; ++j) {
        const float* rj = &re[static_cast<size_t>(j) * chunk];
        const float* ij = &im[static_cast<size_t>(j) * chunk];
        float sr = 0.0f, si = 0.0f;
        for (int64_t t = 0; t < n; ++t) {
          sr += ri[t] * rj[t] + ii[t] * ij[t];
          si += ii[t] * rj[t] - ri[t] * ij[t];
        }
        acc(i, j) += cd(sr, si);
        if (j != i) acc(j, i) += cd(sr, -si);
      }
    }
  }
  return acc;
}

#endif  // GSS_ORACLE_VECTOR_GRAM

// ---------------------------------------------------------------------------
// FFT (stands in for Eigen::FFT<double>, kissfft backend; power-of-two sizes)
// ---------------------------------------------------------------------------
struct FftPlan {
  int n = 0;
  std::vector<cd> tw;      // e^{-2 pi i k/n}
  std::vector<int> rev;
  explicit FftPlan(int size) : n(size), tw(size / 2), rev(size) {
    if (size < 1 || (size & (size - 1)))
      throw OracleError(kConfigError, "oracle fft: size must be a power of two");
    for (int k = 0; k < size / 2; ++k) {
      const double ang = -2.0 * M_PI * k / size;
      tw[k] = cd(std::cos(ang), std::sin(ang));
    }
    int bits = 0;
    while ((1 << bits) < size) ++bits;
    for (int i = 0; i < size; ++i) {
      int r = 0;
      for (int b = 0; b < bits; ++b)
        if (i & (1 << b)) r |= 1 << (bits - 1 - b);
      rev[i] = r;
    }
  }
  // in-place complex transform; inverse is unscaled
  void run(cd* x, bool inverse) const {
    for (int i = 0; i < n; ++i)
      if (rev[i] > i) std::swap(x[i], x[rev[i]]);
    for (int len = 2; len <= n; len <<= 1) {
      const int half = len / 2, step = n / len;
      for (int base = 0; base < n; base += len) {
        for (int k = 0; k < half; ++k) {
          cd w = tw[k * step];
          if (inverse) w = std::conj(w);
          const cd u = x[base + k], v = x[base + k + half] * w;
          x[base + k] = u + v;
          x[base + k + half] = u - v;
        }
      }
    }
  }
  /// real -> one-sided spectrum (n/2+1 bins), unscaled (Eigen fwd, HalfSpectrum)
  void forward_real(const double* in, cd* out, std::vector<cd>& scratch) const {
    scratch.resize(n);
    for (int i = 0; i < n; ++i) scratch[i] = in[i];
    run(scratch.data(), false);
    for (int k = 0; k <= n / 2; ++k) out[k] = scratch[k];
  }
  /// one-sided spectrum -> real, scaled by 1/n (Eigen inv default). As in the
  /// kissfft real inverse, imaginary parts of DC and Nyquist are ignored.
  void inverse_real(const cd* in, double* out, std::vector<cd>& scratch) const {
    scratch.resize(n);
    scratch[0] = in[0].real();
    scratch[n / 2] = in[n / 2].real();
    for (int k = 1; k < n / 2; ++k) {
      scratch[k] = in[k];
      scratch[n - k] = std::conj(in[k]);
    }
    run(scratch.data(), true);
    const double inv = 1.0 / n;
    for (int i = 0; i < n; ++i) out[i] = scratch[i].real() * inv;
  }
};

// ---------------------------------------------------------------------------
// STFT (stft.hpp)
// ---------------------------------------------------------------------------
struct StftConfig {  // stft.hpp:16-36
  int fft_size = 1024;
  int shift = 256;
  int window = 0;  // 0 = hann, 1 = sqrt-hann
  int sample_rate = 16000;
  int num_bins() const { return fft_size / 2 + 1; }
  void validate() const {
    if (fft_size <= 0 || shift <= 0)
      throw OracleError(kConfigError, "stft: fft_size and shift must be positive");
    if (fft_size % shift != 0)
      throw OracleError(kConfigError, "stft: shift must divide fft_size for overlap-add");
    if (sample_rate <= 0) throw OracleError(kConfigError, "stft: sample_rate must be positive");
  }
};

struct Signal {  // stft.hpp:39-47
  std::vector<std::vector<float>> channels;
  int sample_rate = 0;
  int num_channels() const { return static_cast<int>(channels.size()); }
  int64_t num_samples() const { return channels.empty() ? 0 : (int64_t)channels[0].size(); }
};

struct Spec {  // stft.hpp:52-80, (F,T,M) row-major cfloat
  std::vector<cf> data;
  StftConfig config;
  int64_t origin_samples = 0, num_samples = 0, num_frames = 0;
  int num_bins = 0, num_channels = 0;
  int64_t index(int f, int64_t t, int m) const {
    return (static_cast<int64_t>(f) * num_frames + t) * num_channels + m;
  }
  cf& at(int f, int64_t t, int m) { return data[index(f, t, m)]; }
  const cf& at(int f, int64_t t, int m) const { return data[index(f, t, m)]; }
  static Spec zeros(const StftConfig& cfg, int64_t frames, int channels) {
    Spec s;
    s.config = cfg;
    s.num_bins = cfg.num_bins();
    s.num_frames = frames;
    s.num_channels = channels;
    s.origin_samples = -cfg.fft_size / 2;
    s.data.assign(static_cast<size_t>(s.num_bins) * frames * channels, cf{});
    return s;
  }
};

/// periodic hann / sqrt-hann -- stft.hpp:89-97
inline std::vector<double> make_window(const StftConfig& cfg) {
  std::vector<double> w(cfg.fft_size);
  for (int n = 0; n < cfg.fft_size; ++n) {
    const double h = 0.5 * (1.0 - std::cos(2.0 * M_PI * n / cfg.fft_size));
    w[n] = cfg.window == 0 ? h : std::sqrt(h);
  }
  return w;
}

/// reflect padding without repeating the edge sample -- stft.hpp:100-116
inline std::vector<double> pad_reflect(const std::vector<float>& x, int64_t pl, int64_t pr) {
  const int64_t n = static_cast<int64_t>(x.size());
  std::vector<double> out(n + pl + pr);
  for (int64_t i = 0; i < pl; ++i) out[i] = x[pl - i];
  for (int64_t i = 0; i < n; ++i) out[pl + i] = x[i];
  for (int64_t i = 0; i < pr; ++i) {
    int64_t src = n - 2 - i;
    while (src < 0 || src >= n) {
      if (src < 0) src = -src;
      if (src >= n) src = 2 * (n - 1) - src;
    }
    out[pl + n + i] = x[src];
  }
  return out;
}

/// stft.hpp:120-124
inline int64_t frame_count(int64_t num_samples, const StftConfig& cfg) {
  const int64_t padded = num_samples + cfg.fft_size;
  return (padded - cfg.fft_size) / cfg.shift + 1;
}

/// stft.hpp:131-175 (single-threaded double FFT, cast to cfloat)
inline Spec analyze(const Signal& sig, const StftConfig& cfg) {
  cfg.validate();
  const int m_count = sig.num_channels();
  const int64_t n = sig.num_samples();
  if (m_count < 1) throw OracleError(kShapeError, "stft.analyze: no channels");
  for (const auto& ch : sig.channels)
    if (static_cast<int64_t>(ch.size()) != n)
      throw OracleError(kShapeError, "stft.analyze: channels differ in length");
  if (n < cfg.fft_size)
    throw OracleError(kInputTooShortError, "stft.analyze: fewer samples than fft_size");
  const int pad = cfg.fft_size / 2;
  const int64_t t_count = frame_count(n, cfg);
  Spec out = Spec::zeros(cfg, t_count, m_count);
  out.num_samples = n;
  if (sig.sample_rate > 0 && sig.sample_rate != cfg.sample_rate)
    throw OracleError(kConfigError, "stft.analyze: signal/config sample rate mismatch");
  const std::vector<double> window = make_window(cfg);
  const int f_count = cfg.num_bins();
  FftPlan plan(cfg.fft_size);
  std::vector<double> frame(cfg.fft_size);
  std::vector<cd> spec(f_count), scratch;
  for (int m = 0; m < m_count; ++m) {
    const std::vector<double> padded = pad_reflect(sig.channels[m], pad, pad);
    for (int64_t t = 0; t < t_count; ++t) {
      const double* src = padded.data() + t * cfg.shift;
      for (int i = 0; i < cfg.fft_size; ++i) frame[i] = src[i] * window[i];
      plan.forward_real(frame.data(), spec.data(), scratch);
      for (int f = 0; f < f_count; ++f) out.at(f, t, m) = static_cast<cf>(spec[f]);
    }
  }
  return out;
}

/// stft.hpp:179-229
inline Signal synthesize(const Spec& spec) {
  const StftConfig& cfg = spec.config;
  cfg.validate();
  if (spec.num_bins != cfg.num_bins())
    throw OracleError(kConfigError, "stft.synthesize: tensor bins do not match config");
  const int64_t t_count = spec.num_frames;
  const int m_count = spec.num_channels;
  const int pad = cfg.fft_size / 2;
  const int64_t padded_len = (t_count - 1) * cfg.shift + cfg.fft_size;
  const int64_t out_len = spec.num_samples > 0
                              ? spec.num_samples
                              : std::max<int64_t>(0, padded_len - 2 * (int64_t)pad);
  const std::vector<double> window = make_window(cfg);
  std::vector<double> wsum(padded_len, 0.0);
  for (int64_t t = 0; t < t_count; ++t) {
    double* dst = wsum.data() + t * cfg.shift;
    for (int i = 0; i < cfg.fft_size; ++i) dst[i] += window[i] * window[i];
  }
  Signal out;
  out.sample_rate = cfg.sample_rate;
  out.channels.assign(m_count, std::vector<float>(out_len, 0.0f));
  FftPlan plan(cfg.fft_size);
  std::vector<cd> bins(spec.num_bins), scratch;
  std::vector<double> frame(cfg.fft_size), ola(padded_len);
  for (int m = 0; m < m_count; ++m) {
    std::fill(ola.begin(), ola.end(), 0.0);
    for (int64_t t = 0; t < t_count; ++t) {
      for (int f = 0; f < spec.num_bins; ++f) bins[f] = static_cast<cd>(spec.at(f, t, m));
      plan.inverse_real(bins.data(), frame.data(), scratch);
      double* dst = ola.data() + t * cfg.shift;
      for (int i = 0; i < cfg.fft_size; ++i) dst[i] += frame[i] * window[i];
    }
    for (int64_t i = 0; i < out_len; ++i) {
      const int64_t p = i + pad;
      if (p < padded_len && wsum[p] > 1e-8)
        out.channels[m][i] = static_cast<float>(ola[p] / wsum[p]);
    }
  }
  return out;
}

// ---------------------------------------------------------------------------
// WPE (wpe.hpp)
// ---------------------------------------------------------------------------
struct WpeConfig {  // wpe.hpp:15-30
  int taps = 10, delay = 2, iterations = 3, psd_context = 0;
  double regularization = 1e-10;
  void validate() const {
    if (taps < 1 || delay < 1 || iterations < 1)
      throw OracleError(kConfigError, "wpe: taps, delay and iterations must be >= 1");
    if (psd_context < 0 || regularization < 0.0)
      throw OracleError(kConfigError, "wpe: psd_context and regularization must be >= 0");
  }
};

constexpr double kPowerFloor = 1e-10;  // wpe.hpp:37

/// wpe.hpp:40-56
inline void frame_powers(const cf* x, int64_t t_count, int m, int context,
                         std::vector<float>& lambda) {
  lambda.resize(t_count);
  std::vector<double> p(t_count);
  for (int64_t t = 0; t < t_count; ++t) {
    // Eigen's squaredNorm on a cfloat row accumulates in float
    float s = 0.0f;
    for (int c = 0; c < m; ++c) s += std::norm(x[t * m + c]);
    p[t] = s / static_cast<double>(m);
  }
  for (int64_t t = 0; t < t_count; ++t) {
    const int64_t lo = std::max<int64_t>(0, t - context);
    const int64_t hi = std::min<int64_t>(t_count - 1, t + context);
    double acc = 0.0;
    for (int64_t u = lo; u <= hi; ++u) acc += p[u];
    lambda[t] = static_cast<float>(std::max(kPowerFloor, acc / static_cast<double>(hi - lo + 1)));
  }
}

/// wpe.hpp:61-98; y is the T x M block of one bin, rewritten in place
inline void dereverberate_bin(cf* y, int64_t t_count, int m, const WpeConfig& cfg, long f) {
  const int taps = cfg.taps, delay = cfg.delay, km = taps * m, cols = km + m;
  const std::vector<cf> observed(y, y + t_count * m);
  std::vector<cf> aug(static_cast<size_t>(t_count) * cols, cf{});
  for (int64_t t = 0; t < t_count; ++t) {
    for (int k = 0; k < taps; ++k) {
      const int64_t src = t - delay - k;
      if (src < 0) continue;
      for (int c = 0; c < m; ++c) aug[t * cols + k * m + c] = observed[src * m + c];
    }
    for (int c = 0; c < m; ++c) aug[t * cols + km + c] = observed[t * m + c];
  }
  std::vector<float> weights(t_count), lambda;
  std::vector<cf> gconj(static_cast<size_t>(km) * m);
  for (int it = 0; it < cfg.iterations; ++it) {
    frame_powers(y, t_count, m, cfg.psd_context, lambda);
    for (int64_t t = 0; t < t_count; ++t) weights[t] = 1.0f / lambda[t];
    const CMat gram = weighted_gram(aug.data(), t_count, cols, weights.data());
    CMat r(km, km), p(km, m);
    for (int j = 0; j < km; ++j)
      for (int i = 0; i < km; ++i) r(i, j) = gram(i, j);
    r = regularize(hermitize(r), cfg.regularization);
    for (int j = 0; j < m; ++j)
      for (int i = 0; i < km; ++i) p(i, j) = gram(i, km + j);
    const CMat g = hermitian_solve(r, p, f);
    for (int i = 0; i < km; ++i)
      for (int c = 0; c < m; ++c) gconj[static_cast<size_t>(i) * m + c] = static_cast<cf>(std::conj(g(i, c)));
    for (int64_t t = 0; t < t_count; ++t) {
      const cf* hist = &aug[t * cols];
      for (int c = 0; c < m; ++c) {
        cf s = 0;
        for (int i = 0; i < km; ++i) s += hist[i] * gconj[static_cast<size_t>(i) * m + c];
        y[t * m + c] = observed[t * m + c] - s;
      }
    }
  }
}

/// wpe.hpp:105-120
inline Spec dereverberate(const Spec& y, const WpeConfig& cfg) {
  cfg.validate();
  if (y.num_frames <= cfg.taps + cfg.delay) return y;  // pass-through (warning in the reference)
  Spec out = y;
  const int64_t block = y.num_frames * y.num_channels;
  parallel_for(y.num_bins, [&](int64_t f) {
    dereverberate_bin(out.data.data() + f * block, y.num_frames, y.num_channels, cfg, (long)f);
  });
  return out;
}

/// wpe.hpp:124-140
inline Spec unit_normalize(const Spec& y) {
  Spec out = y;
  const int m = y.num_channels;
  parallel_for(y.num_bins, [&](int64_t f) {
    cf* bin = out.data.data() + f * y.num_frames * m;
    for (int64_t t = 0; t < y.num_frames; ++t) {
      cf* p = bin + t * m;
      double ns = 0.0;
      for (int c = 0; c < m; ++c) ns += std::norm(static_cast<cd>(p[c]));
      const float scale = static_cast<float>(1.0 / (std::sqrt(ns) + 1e-10));
      for (int c = 0; c < m; ++c) p[c] *= scale;
    }
  });
  return out;
}

// ---------------------------------------------------------------------------
// Activity guide (manifests.hpp:58-68, 372-414)
// ---------------------------------------------------------------------------
struct Segment {  // manifests.hpp:42-51
  std::string id, recording_id, speaker;
  double start = 0.0, duration = 0.0;
  double end() const { return start + duration; }
};

struct Activity {  // manifests.hpp:58-68
  int64_t frames = 0;
  std::vector<std::string> classes;
  int target_index = -1, noise_index = -1;
  std::vector<uint8_t> grid;  // frames x classes
  int num_classes() const { return static_cast<int>(classes.size()); }
  uint8_t at(int64_t t, int k) const { return grid[t * classes.size() + k]; }
  void set(int64_t t, int k, uint8_t v) { grid[t * classes.size() + k] = v; }
};

/// manifests.hpp:372-414
inline Activity build_activity_at(const std::vector<Segment>& segments,
                                  const std::vector<int64_t>& centers, int sample_rate,
                                  const std::string& target, bool noise_class) {
  Activity act;
  act.frames = static_cast<int64_t>(centers.size());
  std::set<std::string> speakers;
  for (const auto& s : segments) speakers.insert(s.speaker);
  speakers.insert(target);
  act.classes.assign(speakers.begin(), speakers.end());
  act.target_index = static_cast<int>(
      std::find(act.classes.begin(), act.classes.end(), target) - act.classes.begin());
  if (noise_class) {
    act.noise_index = static_cast<int>(act.classes.size());
    act.classes.push_back("noise");
  }
  act.grid.assign(act.frames * act.classes.size(), 0);
  for (const auto& seg : segments) {
    const int k = static_cast<int>(
        std::find(act.classes.begin(), act.classes.end(), seg.speaker) - act.classes.begin());
    const double lo = seg.start * sample_rate, hi = seg.end() * sample_rate;
    for (int64_t t = 0; t < act.frames; ++t) {
      const double c = static_cast<double>(centers[t]);
      if (c >= lo && c < hi) act.set(t, k, 1);
    }
  }
  if (act.noise_index >= 0)
    for (int64_t t = 0; t < act.frames; ++t) act.set(t, act.noise_index, 1);
  bool on = false;
  for (int64_t t = 0; t < act.frames && !on; ++t) on = act.at(t, act.target_index) != 0;
  if (!on) throw OracleError(kEmptyTargetError, "target speaker has no active frame in the window");
  return act;
}

// ---------------------------------------------------------------------------
// cACGMM (cacgmm.hpp)
// ---------------------------------------------------------------------------
constexpr double kQuadraticFormFloor = 1e-10;  // cacgmm.hpp:17
constexpr double kWeightFloor = 1e-10;         // cacgmm.hpp:18

struct CacgmmState {  // cacgmm.hpp:22-49
  int num_bins = 0, num_classes = 0, num_channels = 0;
  std::vector<double> weights;  // (F,K)
  std::vector<CMat> shapes;     // (F,K) of MxM
  double& weight(int f, int k) { return weights[f * num_classes + k]; }
  double weight(int f, int k) const { return weights[f * num_classes + k]; }
  CMat& shape(int f, int k) { return shapes[f * num_classes + k]; }
  const CMat& shape(int f, int k) const { return shapes[f * num_classes + k]; }
  static CacgmmState uniform(int bins, int classes, int channels) {
    CacgmmState s;
    s.num_bins = bins;
    s.num_classes = classes;
    s.num_channels = channels;
    s.weights.assign(static_cast<size_t>(bins) * classes, 1.0 / classes);
    s.shapes.assign(static_cast<size_t>(bins) * classes, CMat::identity(channels));
    return s;
  }
};

/// cacgmm.hpp:66-82
inline double cacg_log_pdf(const std::vector<cd>& y, const CMat& b) {
  const int m = static_cast<int>(y.size());
  if (b.r != m || b.c != m) throw OracleError(kShapeError, "cacg_log_pdf: B does not match y");
  InverseLogDet f;
  try {
    f = hermitian_inverse_logdet(b);
  } catch (const OracleError& e) {
    if (e.code != kSingularMatrixError) throw;
    f = hermitian_inverse_logdet(regularize(b));
  }
  cd q = 0;
  for (int i = 0; i < m; ++i)
    for (int j = 0; j < m; ++j) q += std::conj(y[i]) * f.inverse(i, j) * y[j];
  const double quad = std::max(kQuadraticFormFloor, q.real());
  return -m * std::log(2.0 * M_PI) + std::lgamma(m) - f.log_det - m * std::log(quad);
}

/// cacgmm.hpp:87-112
inline std::vector<double> time_varying_weights(const std::vector<double>& pi,
                                                const std::vector<uint8_t>& activity,
                                                int noise_index = -1) {
  const int k_count = static_cast<int>(pi.size());
  if (static_cast<int>(activity.size()) != k_count)
    throw OracleError(kShapeError, "time_varying_weights: activity row does not match pi");
  std::vector<double> out(k_count, 0.0);
  double z = 0.0;
  for (int k = 0; k < k_count; ++k)
    if (activity[k]) {
      out[k] = pi[k];
      z += pi[k];
    }
  if (z <= 0.0) {
    if (noise_index >= 0 && noise_index < k_count) {
      std::fill(out.begin(), out.end(), 0.0);
      out[noise_index] = 1.0;
    } else {
      std::fill(out.begin(), out.end(), 1.0 / k_count);
    }
    return out;
  }
  for (double& v : out) v /= z;
  return out;
}

struct ShapeKernels {
  std::vector<cf> binv;         // (F,K,M,M) row-major
  std::vector<double> log_det;  // (F,K)
};

/// cacgmm.hpp:124-152
inline ShapeKernels invert_shapes(const CacgmmState& st) {
  const int F = st.num_bins, K = st.num_classes, m = st.num_channels;
  ShapeKernels out;
  out.binv.assign(static_cast<size_t>(F) * K * m * m, cf{});
  out.log_det.assign(static_cast<size_t>(F) * K, 0.0);
  parallel_for(F, [&](int64_t f) {
    for (int k = 0; k < K; ++k) {
      InverseLogDet ild;
      try {
        ild = hermitian_inverse_logdet(st.shape((int)f, k), (long)f);
      } catch (const OracleError& e) {
        if (e.code != kSingularMatrixError) throw;
        ild = hermitian_inverse_logdet(regularize(st.shape((int)f, k)), (long)f);
      }
      out.log_det[f * K + k] = ild.log_det;
      cf* dst = out.binv.data() + ((f * K + k) * m) * m;
      for (int r = 0; r < m; ++r)
        for (int c = 0; c < m; ++c) dst[r * m + c] = static_cast<cf>(ild.inverse(r, c));
    }
  });
  return out;
}

/// q_{ftk} = max(1e-10, Re sum_{mn} conj(y_m) Binv_{kmn} y_n) in cfloat
/// arithmetic -- cacgmm.hpp:156-174 (the reference routes this through its
/// einsum planner, numerics.hpp:756; the contraction is hard-coded here).
/// `precise` (oracle-only diagnostic) evaluates in double instead.
inline std::vector<float> quad_forms(const Spec& y, const std::vector<cf>& binv, int K,
                                     bool precise = false) {
  const int F = y.num_bins, m = y.num_channels;
  const int64_t T = y.num_frames;
  std::vector<float> q(static_cast<size_t>(F) * T * K);
  parallel_for(F, [&](int64_t f) {
    for (int64_t t = 0; t < T; ++t) {
      const cf* yt = &y.data[(f * T + t) * m];
      for (int k = 0; k < K; ++k) {
        const cf* b = &binv[((f * K + k) * m) * m];
        float val;
        if (!precise) {
          cf acc = 0;
          for (int r = 0; r < m; ++r) {
            cf z = 0;
            for (int c = 0; c < m; ++c) z += b[r * m + c] * yt[c];
            acc += std::conj(yt[r]) * z;
          }
          val = acc.real();
        } else {
          cd acc = 0;
          for (int r = 0; r < m; ++r) {
            cd z = 0;
            for (int c = 0; c < m; ++c) z += static_cast<cd>(b[r * m + c]) * static_cast<cd>(yt[c]);
            acc += std::conj(static_cast<cd>(yt[r])) * z;
          }
          val = static_cast<float>(acc.real());
        }
        q[(f * T + t) * K + k] = std::max(static_cast<float>(kQuadraticFormFloor), val);
      }
    }
  });
  return q;
}

/// cacgmm.hpp:189-257
inline double estep_bin(const CacgmmState& st, const Activity& act, int f,
                        const double* log_det_f, const float* qf, float* gamma_f) {
  const int K = st.num_classes, m = st.num_channels;
  const int64_t T = act.frames;
  const double c0 = -m * std::log(2.0 * M_PI) + std::lgamma(m);
  constexpr float kNegInf = -std::numeric_limits<float>::infinity();
  std::vector<float> logq(static_cast<size_t>(T) * K);
  for (size_t i = 0; i < logq.size(); ++i) logq[i] = std::log(qf[i]);  // float log
  std::vector<double> log_pi(K);
  for (int k = 0; k < K; ++k) log_pi[k] = std::log(std::max(kWeightFloor, st.weight(f, k)));
  double ll = 0.0;
  std::vector<float> u(static_cast<size_t>(T) * K);
  std::vector<double> lse(T);
  for (int64_t t = 0; t < T; ++t) {
    double z = 0.0;
    for (int k = 0; k < K; ++k)
      if (act.at(t, k)) z += st.weight(f, k);
    double max_u = -std::numeric_limits<double>::infinity();
    const bool degenerate = z <= 0.0;
    for (int k = 0; k < K; ++k) {
      const int64_t i = t * K + k;
      bool active = act.at(t, k) != 0;
      double lp;
      if (degenerate) {
        active = act.noise_index >= 0 ? k == act.noise_index : true;
        lp = act.noise_index >= 0 ? 0.0 : -std::log((double)K);
      } else {
        lp = log_pi[k] - std::log(z);
      }
      if (!active) {
        u[i] = kNegInf;
        continue;
      }
      const double val = lp + c0 - log_det_f[k] - m * static_cast<double>(logq[i]);
      u[i] = static_cast<float>(val);
      max_u = std::max(max_u, val);
    }
    double sum = 0.0;
    for (int k = 0; k < K; ++k) {
      const float v = u[t * K + k];
      if (v != kNegInf) sum += std::exp(static_cast<double>(v) - max_u);
    }
    lse[t] = max_u + std::log(sum);
    ll += lse[t];
  }
  for (int64_t t = 0; t < T; ++t)
    for (int k = 0; k < K; ++k) {
      const int64_t i = t * K + k;
      gamma_f[i] = u[i] == kNegInf
                       ? 0.0f
                       : static_cast<float>(std::exp(static_cast<double>(u[i]) - lse[t]));
    }
  return ll;
}

struct EmResult {  // cacgmm.hpp:178-182
  CacgmmState state;
  std::vector<float> gamma;  // (F,T,K)
  std::vector<double> likelihood_trace;
};

/// cacgmm.hpp:264-340
inline EmResult em_fit(const Spec& y, const Activity& act, int iterations = 20,
                       bool precise_quad = false) {
  if (iterations < 1) throw OracleError(kConfigError, "cacgmm: iterations must be >= 1");
  if (act.frames != y.num_frames)
    throw OracleError(kShapeError, "cacgmm: activity frames do not match tensor");
  const int F = y.num_bins, m = y.num_channels, K = act.num_classes();
  const int64_t T = y.num_frames;
  EmResult res;
  res.state = CacgmmState::uniform(F, K, m);
  res.gamma.assign(static_cast<size_t>(F) * T * K, 0.0f);
  CacgmmState& st = res.state;
  std::vector<double> bin_ll(F);
  for (int it = 0; it <= iterations; ++it) {
    ShapeKernels kern = invert_shapes(st);
    std::vector<float> q = quad_forms(y, kern.binv, K, precise_quad);
    parallel_for(F, [&](int64_t f) {
      bin_ll[f] = estep_bin(st, act, (int)f, kern.log_det.data() + f * K,
                            q.data() + f * T * K, res.gamma.data() + f * T * K);
    });
    double ll = 0.0;
    for (int f = 0; f < F; ++f) ll += bin_ll[f];
    res.likelihood_trace.push_back(ll);
    if (it == iterations) break;
    parallel_for(F, [&](int64_t f) {
      const cf* yf = y.data.data() + f * T * m;
      const float* qf = q.data() + f * T * K;
      const float* gf = res.gamma.data() + f * T * K;
      std::vector<float> w(T);
      for (int k = 0; k < K; ++k) {
        double mass = 0.0;
        for (int64_t t = 0; t < T; ++t) mass += gf[t * K + k];
        if (mass <= 0.0) {
          st.weight((int)f, k) = kWeightFloor;
          continue;
        }
        for (int64_t t = 0; t < T; ++t) w[t] = gf[t * K + k] / qf[t * K + k];
        CMat b = weighted_gram(yf, T, m, w.data());
        const double s = static_cast<double>(m) / mass;
        for (auto& v : b.v) v *= s;
        b = hermitize(b);
        double tr = 0;
        for (int i = 0; i < m; ++i) tr += b(i, i).real();
        if (tr > 0.0) {
          const double g = static_cast<double>(m) / tr;
          for (auto& v : b.v) v *= g;
        }
        st.shape((int)f, k) = regularize(b);
        st.weight((int)f, k) = std::max(kWeightFloor, mass / static_cast<double>(T));
      }
    });
  }
  return res;
}

/// cacgmm.hpp:343-370
inline double log_likelihood(const Spec& y, const CacgmmState& st, const Activity& act) {
  if (act.frames != y.num_frames || act.num_classes() != st.num_classes)
    throw OracleError(kShapeError, "log_likelihood: inconsistent shapes");
  const int F = y.num_bins, K = st.num_classes;
  const int64_t T = y.num_frames;
  ShapeKernels kern = invert_shapes(st);
  std::vector<float> q = quad_forms(y, kern.binv, K);
  std::vector<double> bin_ll(F);
  parallel_for(F, [&](int64_t f) {
    std::vector<float> scratch(static_cast<size_t>(T) * K);
    bin_ll[f] = estep_bin(st, act, (int)f, kern.log_det.data() + f * K, q.data() + f * T * K,
                          scratch.data());
  });
  double ll = 0.0;
  for (int f = 0; f < F; ++f) ll += bin_ll[f];
  return ll;
}

// ---------------------------------------------------------------------------
// Souden MVDR (beamform.hpp)
// ---------------------------------------------------------------------------
struct BeamformerStats {  // beamform.hpp:18-24
  int num_bins = 0, num_channels = 0;
  int64_t frame_count = 0;
  std::vector<CMat> target, background;
};

struct BeamformerFilter {  // beamform.hpp:26-31
  int num_channels = 0, ref_channel = 0;
  std::vector<std::vector<cd>> h;
  int64_t zeroed_bins = 0;
};

/// beamform.hpp:35-85
inline BeamformerStats accumulate_stats(const Spec& y, const std::vector<float>& gamma, int K,
                                        int target) {
  const int F = y.num_bins, m = y.num_channels;
  const int64_t T = y.num_frames;
  if (static_cast<int64_t>(gamma.size()) != (int64_t)F * T * K)
    throw OracleError(kShapeError, "accumulate_stats: posterior does not match tensor");
  if (target < 0 || target >= K)
    throw OracleError(kShapeError, "accumulate_stats: target class out of range");
  BeamformerStats st;
  st.num_bins = F;
  st.num_channels = m;
  st.frame_count = T;
  st.target.assign(F, CMat());
  st.background.assign(F, CMat());
  std::vector<double> target_mass(F, 0.0);
  parallel_for(F, [&](int64_t f) {
    const cf* yf = y.data.data() + f * T * m;
    const float* gf = gamma.data() + f * T * K;
    std::vector<float> wt(T), wb(T);
    double mass = 0.0;
    for (int64_t t = 0; t < T; ++t) {
      wt[t] = gf[t * K + target];
      float other = 0.0f;
      for (int k = 0; k < K; ++k)
        if (k != target) other += gf[t * K + k];
      wb[t] = other;
      mass += wt[t];
    }
    target_mass[f] = mass;
    const double inv_t = 1.0 / static_cast<double>(T);
    st.target[f] = weighted_gram(yf, T, m, wt.data());
    st.background[f] = weighted_gram(yf, T, m, wb.data());
    for (auto& v : st.target[f].v) v *= inv_t;
    for (auto& v : st.background[f].v) v *= inv_t;
  });
  double total = 0.0;
  for (double v : target_mass) total += v;
  if (total <= 0.0)
    throw OracleError(kDegenerateStatsError, "accumulate_stats: target mask is all zero");
  return st;
}

/// beamform.hpp:89-107
inline int select_reference(const BeamformerStats& st) {
  const int m = st.num_channels;
  std::vector<double> num(m, 0.0), den(m, 0.0);
  for (int f = 0; f < st.num_bins; ++f)
    for (int c = 0; c < m; ++c) {
      num[c] += st.target[f](c, c).real();
      den[c] += st.background[f](c, c).real();
    }
  int best = 0;
  double best_snr = -std::numeric_limits<double>::infinity();
  for (int c = 0; c < m; ++c) {
    const double snr = num[c] / std::max(den[c], 1e-10);
    if (snr > best_snr) {
      best_snr = snr;
      best = c;
    }
  }
  return best;
}

/// beamform.hpp:111-135
inline BeamformerFilter mvdr(const BeamformerStats& st, int ref) {
  const int m = st.num_channels;
  if (ref < 0 || ref >= m) throw OracleError(kShapeError, "mvdr: reference channel out of range");
  BeamformerFilter flt;
  flt.num_channels = m;
  flt.ref_channel = ref;
  flt.h.assign(st.num_bins, std::vector<cd>(m, cd{}));
  std::vector<uint8_t> zeroed(st.num_bins, 0);
  parallel_for(st.num_bins, [&](int64_t f) {
    const CMat c = hermitian_solve(regularize(hermitize(st.background[f])), st.target[f], (long)f);
    cd tr = 0;
    for (int i = 0; i < m; ++i) tr += c(i, i);
    if (std::abs(tr) < 1e-10) {
      zeroed[f] = 1;
      return;
    }
    for (int i = 0; i < m; ++i) flt.h[f][i] = c(i, ref) / tr;
  });
  for (uint8_t z : zeroed) flt.zeroed_bins += z;
  return flt;
}

/// beamform.hpp:138-165: out_{f,t} = sum_m y_{ftm} conj(h_{fm}) in cfloat
inline Spec apply_filter(const BeamformerFilter& flt, const Spec& y) {
  if (flt.num_channels != y.num_channels || static_cast<int>(flt.h.size()) != y.num_bins)
    throw OracleError(kShapeError, "beamform.apply: filter does not match tensor");
  const int64_t T = y.num_frames;
  const int m = y.num_channels;
  Spec out;
  out.config = y.config;
  out.num_bins = y.num_bins;
  out.num_frames = T;
  out.num_channels = 1;
  out.origin_samples = y.origin_samples;
  out.num_samples = y.num_samples;
  out.data.assign(static_cast<size_t>(y.num_bins) * T, cf{});
  parallel_for(y.num_bins, [&](int64_t f) {
    std::vector<cf> hc(m);
    for (int c = 0; c < m; ++c) hc[c] = std::conj(static_cast<cf>(flt.h[f][c]));
    const cf* yf = y.data.data() + f * T * m;
    cf* of = out.data.data() + f * T;
    for (int64_t t = 0; t < T; ++t) {
      cf s = 0;
      for (int c = 0; c < m; ++c) s += yf[t * m + c] * hc[c];
      of[t] = s;
    }
  });
  return out;
}

// ---------------------------------------------------------------------------
// Assembly index math + enhance_batch (scheduler.hpp)
// ---------------------------------------------------------------------------
struct PipelineConfig {  // the fields enhance_batch reads, scheduler.hpp:30-44
  int bss_iterations = 20;
  bool enable_wpe = true;
  WpeConfig wpe;
  StftConfig stft;
};

struct Part {  // scheduler.hpp:168-172
  int64_t sample_begin = 0, sample_end = 0;
};

struct AssemblyPlan {
  std::vector<std::pair<int64_t, int64_t>> spans;  // source [begin,end)
  std::vector<int64_t> span_offsets;               // assembled offset per span
  std::vector<Part> parts;
  std::vector<int64_t> frame_centers;
  int64_t total = 0;
  double context_left = 0, context_right = 0;
};

/// The integer part of scheduler::assemble (scheduler.hpp:196-266): span list,
/// part offsets, frame-centre -> source-sample map. No audio I/O.
inline AssemblyPlan assemble_indices(const std::vector<std::pair<double, double>>& parts_start_dur,
                                     int sr, int64_t rec_samples, double context_duration,
                                     const StftConfig& stft) {
  AssemblyPlan ap;
  if (parts_start_dur.empty()) throw OracleError(kShapeError, "assemble: no parts");
  const int64_t first_start = std::llround(parts_start_dur.front().first * sr);
  const int64_t ctx = std::llround(context_duration * sr);
  const int64_t left_begin = std::max<int64_t>(0, first_start - ctx);
  if (left_begin < first_start) ap.spans.emplace_back(left_begin, first_start);
  ap.context_left = static_cast<double>(first_start - left_begin) / sr;
  std::vector<size_t> part_span;
  for (const auto& [start, dur] : parts_start_dur) {
    const int64_t s0 = std::llround(start * sr);
    const int64_t s1 = std::min<int64_t>(rec_samples, std::llround((start + dur) * sr));
    if (s1 <= s0) throw OracleError(kShapeError, "segment maps to an empty sample range");
    part_span.push_back(ap.spans.size());
    ap.spans.emplace_back(s0, s1);
  }
  const int64_t last_end = ap.spans.back().second;
  const int64_t right_end = std::min(rec_samples, last_end + ctx);
  if (right_end > last_end) ap.spans.emplace_back(last_end, right_end);
  ap.context_right = static_cast<double>(right_end - last_end) / sr;
  int64_t off = 0;
  for (const auto& [b, e] : ap.spans) {
    ap.span_offsets.push_back(off);
    off += e - b;
  }
  ap.total = off;
  for (size_t p = 0; p < parts_start_dur.size(); ++p) {
    Part part;
    part.sample_begin = ap.span_offsets[part_span[p]];
    part.sample_end = part.sample_begin + (ap.spans[part_span[p]].second - ap.spans[part_span[p]].first);
    ap.parts.push_back(part);
  }
  const int64_t t_count = frame_count(ap.total, stft);
  ap.frame_centers.resize(t_count);
  for (int64_t t = 0; t < t_count; ++t) {
    const int64_t c = std::min<int64_t>(t * stft.shift, ap.total - 1);
    size_t s = 0;
    while (s + 1 < ap.spans.size() &&
           c >= ap.span_offsets[s] + (ap.spans[s].second - ap.spans[s].first))
      ++s;
    ap.frame_centers[t] = ap.spans[s].first + (c - ap.span_offsets[s]);
  }
  return ap;
}

struct EnhanceOut {  // scheduler.hpp:283-294 (without timings / paths)
  std::vector<std::vector<float>> outputs;  // one mono cut per part
  std::vector<float> mono;                  // full-window synthesis (diagnostic)
  double ll_final = 0.0;
  int64_t zeroed_bins = 0;
  int ref_channel = 0;
  int64_t frames = 0;
  double stage_seconds[5] = {0, 0, 0, 0, 0};  // stft, wpe, mask, beamform, istft
  // diagnostics for parity probes
  std::vector<float> gamma;
  std::vector<cd> h;  // (F,M)
};

/// scheduler.hpp:314-365
inline EnhanceOut enhance_batch(const Signal& audio, const Activity& act,
                                const std::vector<Part>& parts, const PipelineConfig& cfg,
                                bool keep_diag = false);

}  // namespace gss_oracle

#include <chrono>

namespace gss_oracle {

inline EnhanceOut enhance_batch(const Signal& audio, const Activity& act,
                                const std::vector<Part>& parts, const PipelineConfig& cfg,
                                bool keep_diag) {
  using clk = std::chrono::steady_clock;
  auto secs = [](clk::time_point a) { return std::chrono::duration<double>(clk::now() - a).count(); };
  EnhanceOut res;
  auto t0 = clk::now();
  Spec tensor = analyze(audio, cfg.stft);
  res.frames = tensor.num_frames;
  res.stage_seconds[0] = secs(t0);
  t0 = clk::now();
  if (cfg.enable_wpe) tensor = dereverberate(tensor, cfg.wpe);
  res.stage_seconds[1] = secs(t0);
  t0 = clk::now();
  EmResult em;
  {
    const Spec normalized = unit_normalize(tensor);
    em = em_fit(normalized, act, cfg.bss_iterations);
  }
  res.ll_final = em.likelihood_trace.back();
  res.stage_seconds[2] = secs(t0);
  t0 = clk::now();
  BeamformerStats stats = accumulate_stats(tensor, em.gamma, act.num_classes(), act.target_index);
  res.ref_channel = select_reference(stats);
  BeamformerFilter flt = mvdr(stats, res.ref_channel);
  res.zeroed_bins = flt.zeroed_bins;
  Spec enhanced = apply_filter(flt, tensor);
  res.stage_seconds[3] = secs(t0);
  t0 = clk::now();
  Signal wave = synthesize(enhanced);
  res.stage_seconds[4] = secs(t0);
  const auto& mono = wave.channels[0];
  for (const auto& p : parts) {
    const int64_t hi = std::min<int64_t>(p.sample_end, static_cast<int64_t>(mono.size()));
    res.outputs.emplace_back(mono.begin() + p.sample_begin, mono.begin() + hi);
  }
  if (keep_diag) {
    res.mono = mono;
    res.gamma = std::move(em.gamma);
    const int m = tensor.num_channels;
    res.h.resize(static_cast<size_t>(tensor.num_bins) * m);
    for (int f = 0; f < tensor.num_bins; ++f)
      for (int c = 0; c < m; ++c) res.h[static_cast<size_t>(f) * m + c] = flt.h[f][c];
  }
  return res;
}

}  // namespace gss_oracle
