// linalg.cuh -- small dense complex-double linear algebra shared by the CUDA
// kernels (per-thread, M <= kMaxDim) and by the host-side unit tests
// (tests/host_linalg_check.cpp compiles this header with g++).
//
// Mirrors the reference's Hermitian helpers, numerics.hpp:28-122:
//   hermitize / regularize / LLT solve / inverse+logdet with the
//   eigenvalue-floor fallback (floor = 1e-10 * lambda_max).
// Matrices are row-major arrays of cdbl with leading dimension `ld`.
#pragma once

#include <math.h>

#ifdef __CUDACC__
#define GSS_HD __host__ __device__ __forceinline__
#define GSS_HD_NOINLINE inline __host__ __device__ __noinline__
#else
#define GSS_HD inline
#define GSS_HD_NOINLINE inline
#endif

namespace gssb {

struct cdbl {
  double re, im;
};

GSS_HD cdbl cd_make(double r, double i) {
  cdbl z;
  z.re = r;
  z.im = i;
  return z;
}
GSS_HD cdbl cd_add(cdbl a, cdbl b) { return cd_make(a.re + b.re, a.im + b.im); }
GSS_HD cdbl cd_sub(cdbl a, cdbl b) { return cd_make(a.re - b.re, a.im - b.im); }
GSS_HD cdbl cd_mul(cdbl a, cdbl b) { return cd_make(a.re * b.re - a.im * b.im, a.re * b.im + a.im * b.re); }
// a * conj(b)
GSS_HD cdbl cd_mulc(cdbl a, cdbl b) { return cd_make(a.re * b.re + a.im * b.im, a.im * b.re - a.re * b.im); }
// conj(a) * b
GSS_HD cdbl cd_cmul(cdbl a, cdbl b) { return cd_make(a.re * b.re + a.im * b.im, a.re * b.im - a.im * b.re); }
GSS_HD cdbl cd_scale(cdbl a, double s) { return cd_make(a.re * s, a.im * s); }
GSS_HD cdbl cd_conj(cdbl a) { return cd_make(a.re, -a.im); }
GSS_HD double cd_norm(cdbl a) { return a.re * a.re + a.im * a.im; }
GSS_HD cdbl cd_div(cdbl a, cdbl b) {
  // Smith's algorithm (what std::complex<double> division does up to rounding)
  if (fabs(b.re) >= fabs(b.im)) {
    const double r = b.im / b.re, d = b.re + b.im * r;
    return cd_make((a.re + a.im * r) / d, (a.im - a.re * r) / d);
  }
  const double r = b.re / b.im, d = b.re * r + b.im;
  return cd_make((a.re * r + a.im) / d, (a.im * r - a.re) / d);
}

constexpr double kRegEps = 1e-10;              // numerics.hpp:28
constexpr double kEigFloorRatio = 1e-10;       // numerics.hpp:29

/// A <- (A + A^H)/2 in place (numerics.hpp:32-38)
GSS_HD void hermitize_inplace(cdbl* a, int n, int ld) {
  for (int i = 0; i < n; ++i) {
    a[i * ld + i].im = 0.5 * (a[i * ld + i].im - a[i * ld + i].im);
    for (int j = 0; j < i; ++j) {
      const cdbl lo = a[i * ld + j], up = a[j * ld + i];
      const cdbl avg = cd_make(0.5 * (lo.re + up.re), 0.5 * (lo.im - up.im));
      a[i * ld + j] = avg;
      a[j * ld + i] = cd_conj(avg);
    }
  }
}

/// A += eps * max(tr/n -> 1 if not positive) * I (numerics.hpp:41-49)
GSS_HD void regularize_inplace(cdbl* a, int n, int ld, double eps) {
  double tr = 0.0;
  for (int i = 0; i < n; ++i) tr += a[i * ld + i].re;
  double scale = tr / (double)n;
  if (!(scale > 0.0)) scale = 1.0;
  for (int i = 0; i < n; ++i) a[i * ld + i].re += eps * scale;
}

/// In-place lower Cholesky reading the lower triangle only; false iff a pivot
/// is <= 0 (Eigen LLT's failure criterion, numerics.hpp:88,105).
GSS_HD bool cholesky_lower(cdbl* a, int n, int ld) {
  for (int k = 0; k < n; ++k) {
    double x = a[k * ld + k].re;
    for (int j = 0; j < k; ++j) x -= cd_norm(a[k * ld + j]);
    if (x <= 0.0) return false;
    x = sqrt(x);
    a[k * ld + k] = cd_make(x, 0.0);
    const double inv = 1.0 / x;
    for (int i = k + 1; i < n; ++i) {
      cdbl s = a[i * ld + k];
      for (int j = 0; j < k; ++j) s = cd_sub(s, cd_mulc(a[i * ld + j], a[k * ld + j]));
      a[i * ld + k] = cd_scale(s, inv);
    }
  }
  return true;
}

/// Solve L L^H x = b for one right-hand side stored with stride `bs`.
GSS_HD void cholesky_solve_vec(const cdbl* l, int n, int ld, cdbl* b, int bs) {
  for (int i = 0; i < n; ++i) {
    cdbl s = b[i * bs];
    for (int j = 0; j < i; ++j) s = cd_sub(s, cd_mul(l[i * ld + j], b[j * bs]));
    b[i * bs] = cd_scale(s, 1.0 / l[i * ld + i].re);
  }
  for (int i = n - 1; i >= 0; --i) {
    cdbl s = b[i * bs];
    for (int j = i + 1; j < n; ++j) s = cd_sub(s, cd_cmul(l[j * ld + i], b[j * bs]));
    b[i * bs] = cd_scale(s, 1.0 / l[i * ld + i].re);
  }
}

/// Cyclic two-sided Jacobi eigendecomposition of a Hermitian matrix (lower
/// triangle is read). a is overwritten; v receives eigenvectors (columns),
/// w the eigenvalues. Returns false on non-finite values.
/// Stands in for Eigen::SelfAdjointEigenSolver (numerics.hpp:59).
GSS_HD_NOINLINE bool hermitian_eig_jacobi(cdbl* a, int n, int ld, cdbl* v, int ldv, double* w) {
  for (int i = 0; i < n; ++i) {
    a[i * ld + i].im = 0.0;
    for (int j = 0; j < i; ++j) a[j * ld + i] = cd_conj(a[i * ld + j]);
    for (int j = 0; j < n; ++j) v[i * ldv + j] = cd_make(i == j ? 1.0 : 0.0, 0.0);
  }
  for (int sweep = 0; sweep < 60; ++sweep) {
    double off = 0.0, diag = 0.0;
    for (int i = 0; i < n; ++i)
      for (int j = 0; j < n; ++j) {
        const double s = cd_norm(a[i * ld + j]);
        if (i == j) diag += s; else off += s;
      }
    if (!isfinite(off + diag)) return false;
    if (off <= 1e-30 * diag || off == 0.0) break;
    for (int p = 0; p < n - 1; ++p) {
      for (int q = p + 1; q < n; ++q) {
        const cdbl apq = a[p * ld + q];
        const double mag = sqrt(cd_norm(apq));
        if (mag == 0.0) continue;
        const double app = a[p * ld + p].re, aqq = a[q * ld + q].re;
        const cdbl ph = cd_make(apq.re / mag, apq.im / mag);  // e^{i phi}
        const double tau = (aqq - app) / (2.0 * mag);
        const double t = (tau >= 0.0 ? 1.0 : -1.0) / (fabs(tau) + sqrt(1.0 + tau * tau));
        const double c = 1.0 / sqrt(1.0 + t * t), s = t * c;
        // J columns: p -> [c ; -s e^{-i phi}], q -> [s ; c e^{-i phi}]
        const cdbl jpp = cd_make(c, 0.0), jqp = cd_make(-s * ph.re, s * ph.im);
        const cdbl jpq = cd_make(s, 0.0), jqq = cd_make(c * ph.re, -c * ph.im);
        for (int i = 0; i < n; ++i) {  // A <- A J
          const cdbl aip = a[i * ld + p], aiq = a[i * ld + q];
          a[i * ld + p] = cd_add(cd_mul(aip, jpp), cd_mul(aiq, jqp));
          a[i * ld + q] = cd_add(cd_mul(aip, jpq), cd_mul(aiq, jqq));
        }
        for (int j = 0; j < n; ++j) {  // A <- J^H A
          const cdbl apj = a[p * ld + j], aqj = a[q * ld + j];
          a[p * ld + j] = cd_add(cd_cmul(jpp, apj), cd_cmul(jqp, aqj));
          a[q * ld + j] = cd_add(cd_cmul(jpq, apj), cd_cmul(jqq, aqj));
        }
        a[p * ld + q] = cd_make(0.0, 0.0);
        a[q * ld + p] = cd_make(0.0, 0.0);
        a[p * ld + p].im = 0.0;
        a[q * ld + q].im = 0.0;
        for (int i = 0; i < n; ++i) {  // V <- V J
          const cdbl vip = v[i * ldv + p], viq = v[i * ldv + q];
          v[i * ldv + p] = cd_add(cd_mul(vip, jpp), cd_mul(viq, jqp));
          v[i * ldv + q] = cd_add(cd_mul(vip, jpq), cd_mul(viq, jqq));
        }
      }
    }
  }
  for (int i = 0; i < n; ++i) {
    w[i] = a[i * ld + i].re;
    if (!isfinite(w[i])) return false;
  }
  return true;
}

enum LinalgStatus { kLinOk = 0, kLinSingular = 1 };

/// Floors eigenvalues at 1e-10*lambda_max (numerics.hpp:58-73).
/// Returns kLinSingular when there is no positive finite eigenvalue.
GSS_HD int eigen_floor_values(double* w, int n) {
  double emax = w[0];
  for (int i = 1; i < n; ++i) emax = fmax(emax, w[i]);
  if (!(emax > 0.0) || !isfinite(emax)) return kLinSingular;
  const double fl = kEigFloorRatio * emax;
  for (int i = 0; i < n; ++i) w[i] = fmax(w[i], fl);
  return kLinOk;
}

/// inverse and log|A| of a Hermitian PD matrix, Cholesky first, eigenvalue
/// floor fallback second (numerics.hpp:103-122). `a` (n x n, ld) is destroyed,
/// `inv` receives the inverse, `work` must hold n*n cdbl, `wv` n doubles.
template <int NMAX>
GSS_HD_NOINLINE int hermitian_inverse_logdet(cdbl* a, int n, cdbl* inv, double* log_det, cdbl* work,
                                             double* wv) {
  // keep a copy for the fallback (the factorization overwrites the lower triangle)
  for (int i = 0; i < n * n; ++i) work[i] = a[i];
  if (cholesky_lower(a, n, n)) {
    double ld = 0.0;
    for (int i = 0; i < n; ++i) ld += log(a[i * n + i].re);
    *log_det = 2.0 * ld;
    for (int c = 0; c < n; ++c) {
      for (int i = 0; i < n; ++i) inv[i * n + c] = cd_make(i == c ? 1.0 : 0.0, 0.0);
      cholesky_solve_vec(a, n, n, inv + c, n);
    }
    return kLinOk;
  }
  // a <- eigenvectors storage, work <- matrix being diagonalized
  if (!hermitian_eig_jacobi(work, n, n, a, n, wv)) return kLinSingular;
  if (eigen_floor_values(wv, n) != kLinOk) return kLinSingular;
  double ld = 0.0;
  for (int i = 0; i < n; ++i) ld += log(wv[i]);
  *log_det = ld;
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) {
      cdbl s = cd_make(0.0, 0.0);
      for (int e = 0; e < n; ++e) s = cd_add(s, cd_scale(cd_mulc(a[i * n + e], a[j * n + e]), 1.0 / wv[e]));
      inv[i * n + j] = s;
    }
  return kLinOk;
}

/// X = A^{-1} B for Hermitian A (n x n) and B (n x nrhs, row-major ld nrhs):
/// Cholesky, eigenvalue-floor fallback (numerics.hpp:81-94). a is destroyed;
/// b is overwritten with X. work: n*n cdbl, work2: n*n cdbl, wv: n doubles.
GSS_HD_NOINLINE int hermitian_solve(cdbl* a, int n, cdbl* b, int nrhs, cdbl* work, cdbl* work2, double* wv) {
  for (int i = 0; i < n * n; ++i) work[i] = a[i];
  if (cholesky_lower(a, n, n)) {
    for (int c = 0; c < nrhs; ++c) cholesky_solve_vec(a, n, n, b + c, nrhs);
    return kLinOk;
  }
  if (!hermitian_eig_jacobi(work, n, n, a, n, wv)) return kLinSingular;
  if (eigen_floor_values(wv, n) != kLinOk) return kLinSingular;
  // work2 <- diag(1/w) V^H B ; b <- V work2
  for (int e = 0; e < n; ++e)
    for (int c = 0; c < nrhs; ++c) {
      cdbl s = cd_make(0.0, 0.0);
      for (int j = 0; j < n; ++j) s = cd_add(s, cd_cmul(a[j * n + e], b[j * nrhs + c]));
      work2[e * nrhs + c] = cd_scale(s, 1.0 / wv[e]);
    }
  for (int i = 0; i < n; ++i)
    for (int c = 0; c < nrhs; ++c) {
      cdbl s = cd_make(0.0, 0.0);
      for (int e = 0; e < n; ++e) s = cd_add(s, cd_mul(a[i * n + e], work2[e * nrhs + c]));
      b[i * nrhs + c] = s;
    }
  return kLinOk;
}

}  // namespace gssb
