// cacgmm_kernels.cuh -- cACGMM EM kernels (templates; instantiated per channel
// count in cacgmm_m*.cu) and the MVDR statistics kernels that share the same
// Hermitian outer-product machinery.
//
// Reference semantics: cacgmm.hpp:264-340 (em_fit), :124-152 (invert_shapes),
// :156-174 (quad_forms), :189-257 (estep_bin), wpe.hpp:124-140 (unit_normalize),
// numerics.hpp:128-152 (weighted_gram), beamform.hpp:35-85 (accumulate_stats).
//
// One EM iteration = em_pass2_kernel (cacgmm_pass2.cuh: E-step + M-step accumulation fused in one
// sweep over the spectrogram) + em_update_kernel (per-(f,k) M-step
// finalisation in FP64: trace normalisation, regularisation, Cholesky inverse,
// log-det, E-step constants for the next sweep).
//
// The sweep works on the RAW (un-normalised) spectrogram: with s = 1/(|y|+1e-10)
// the unit-norm frame is s*y, so q = s^2 * q_raw and the M-step weight
// gamma/q applied to (s*y)(s*y)^H equals (gamma/q * s^2) applied to y y^H. The
// normalised tensor is therefore never materialised, and the last sweep can
// accumulate the MVDR statistics of the raw tensor (beamform.hpp:35-85) with
// the posteriors still in registers.
#pragma once

#include <math_constants.h>

#include "kernels.h"

namespace gssb {

// ---------------------------------------------------------------------------
// Per-lane view of one frame
// ---------------------------------------------------------------------------
template <int M, int L>
struct FramePlan {
  using Lay = EmLayout<M, L>;
  static constexpr int NZ1 = Lay::NZ > 0 ? Lay::NZ : 1;
  int offx[Lay::RPL];
  int offz[Lay::RPL][NZ1];
  bool lo[Lay::RPL];

  __device__ __forceinline__ void init(int g) {
#pragma unroll
    for (int i = 0; i < Lay::RPL; ++i) {
      int row = g + i * L;
      if (row >= M) row = 0;  // idle row: computes finite values that nobody reads
      offx[i] = row;
#pragma unroll
      for (int d = 1; d <= Lay::D; ++d) offz[i][d - 1] = (row + d) % M;
      if (Lay::HALF) offz[i][Lay::D] = (row + M / 2) % M;
      lo[i] = row < M / 2;
    }
  }

  /// Hermitian outer-product dofs of the frame whose M channels start at fr.
  __device__ __forceinline__ void dofs(const float2* fr, float (&pv)[Lay::NDOF]) const {
#pragma unroll
    for (int i = 0; i < Lay::RPL; ++i) {
      const float2 x = fr[offx[i]];
      pv[i * M] = fmaf(x.x, x.x, x.y * x.y);
#pragma unroll
      for (int d = 1; d <= Lay::D; ++d) {
        const float2 z = fr[offz[i][d - 1]];
        pv[i * M + 2 * d - 1] = fmaf(x.x, z.x, x.y * z.y);
        pv[i * M + 2 * d] = fmaf(x.y, z.x, -(x.x * z.y));
      }
      if (Lay::HALF) {
        const float2 z = fr[offz[i][Lay::D]];
        const float a1 = lo[i] ? x.x : x.y;
        const float a2 = lo[i] ? x.y : -x.x;
        pv[i * M + M - 1] = fmaf(a1, z.x, a2 * z.y);
      }
    }
  }
};

/// Partial-sum cell written per (segment, bin, frame chunk): for every lane g
/// its NA*NDOF accumulators followed by the KT class masses.
template <int M, int L, int KT, int NA>
struct PartLayout {
  static constexpr int NDOF = EmLayout<M, L>::NDOF;
  static constexpr int ACC = NA * NDOF;
  static constexpr int STRIDE = ACC + KT;
  static constexpr int CELL = L * STRIDE;
};

#ifdef GSS_ACCURATE_MATH
// Measurement variant (tools/variant.py accurate -DGSS_ACCURATE_MATH=1): correctly rounded reciprocal / square
// root and the full-precision log2f / exp2f in place of the MUFU approximations, and the soft-max sum in double
// like cacgmm.hpp:239-255. It exists to put a number on how much of the device-vs-oracle mask difference is the
// fast math (profiles/parity_r02.md); the product build uses the approximations below.
__device__ __forceinline__ float rcp_approx(float x) { return __frcp_rn(x); }
__device__ __forceinline__ float lg2_approx(float x) { return log2f(x); }
__device__ __forceinline__ float ex2_approx(float x) { return exp2f(x); }
__device__ __forceinline__ float sqrt_approx(float x) { return __fsqrt_rn(x); }
#else
__device__ __forceinline__ float rcp_approx(float x) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}
__device__ __forceinline__ float lg2_approx(float x) {  // x >= 1e-10 here: no denormal inputs
  float r;
  asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}
__device__ __forceinline__ float ex2_approx(float x) {
  float r;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}
__device__ __forceinline__ float sqrt_approx(float x) {
  float r;
  asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}
#endif  // GSS_ACCURATE_MATH

__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

/// Sweep flavours: kSweepEM accumulates the M-step Grams; kSweepEMGamma does the same and may also store
/// the posteriors (last sweep of the stage entry point); kSweepFinal accumulates the MVDR statistics and
/// may store the posteriors (last sweep of enhance_batch).
enum SweepMode { kSweepEM = 0, kSweepEMGamma = 1, kSweepFinal = 2 };

// ---------------------------------------------------------------------------
// M-step finalisation / state preparation. grid = (F, segments), block = KT warps: warp k owns class k
// of the bin, its M x M matrices live in shared memory and the lanes work on entries / column solves
// in parallel (the single-thread form of the same algebra is latency bound: ~100 us per launch).
// ---------------------------------------------------------------------------
/// In-place lower Cholesky of the Hermitian M x M matrix f (row-major, shared memory) by one warp.
/// Fails (returns false) iff a pivot is <= 0, Eigen LLT's criterion (numerics.hpp:88,105).
template <int M>
__device__ __forceinline__ bool warp_cholesky(cdbl* f, int lane) {
  // lane -> (row, column) of the trailing lower triangle, the same enumeration at every step (found once:
  // this search inside the step loop was a quarter of the kernel's executed instructions)
  int ii = 0;
  while ((ii + 1) * (ii + 2) / 2 <= lane) ++ii;
  const int jj = lane - ii * (ii + 1) / 2;
  for (int k = 0; k < M; ++k) {
    const double d = f[k * M + k].re;
    if (!(d > 0.0)) return false;  // warp-uniform
    const double inv = rsqrt(d), sq = d * inv;
    __syncwarp();
    if (lane == 0) f[k * M + k] = cd_make(sq, 0.0);
    if (lane > k && lane < M) f[lane * M + k] = cd_scale(f[lane * M + k], inv);
    __syncwarp();
    const int r = M - 1 - k;
    if (lane < r * (r + 1) / 2) {
      const int i = k + 1 + ii, j = k + 1 + jj;
      f[i * M + j] = cd_sub(f[i * M + j], cd_mulc(f[i * M + k], f[j * M + k]));
    }
    __syncwarp();
  }
  return true;
}

/// inv <- (L L^H)^-1, lane c solves column c (forward then backward substitution). The M reciprocals of the
/// diagonal are taken once (an FP64 division is a ~30-instruction dependent chain; 2 M of them per column sat on
/// the kernel's critical path) and the loops are unrolled so the factor's entries load ahead of their use.
template <int M>
__device__ __forceinline__ void warp_cholesky_inverse(const cdbl* l, cdbl* inv, int lane) {
  if (lane < M) {
    const int c = lane;
    double rd[M];
#pragma unroll
    for (int i = 0; i < M; ++i) rd[i] = 1.0 / l[i * M + i].re;
    cdbl x[M];
#pragma unroll
    for (int i = 0; i < M; ++i) {
      cdbl s = cd_make(i == c ? 1.0 : 0.0, 0.0);
#pragma unroll
      for (int j = 0; j < i; ++j) s = cd_sub(s, cd_mul(l[i * M + j], x[j]));
      x[i] = cd_scale(s, rd[i]);
    }
#pragma unroll
    for (int i = M - 1; i >= 0; --i) {
      cdbl s = x[i];
#pragma unroll
      for (int j = i + 1; j < M; ++j) s = cd_sub(s, cd_cmul(l[j * M + i], x[j]));
      x[i] = cd_scale(s, rd[i]);
    }
#pragma unroll
    for (int i = 0; i < M; ++i) inv[i * M + c] = x[i];
  }
  __syncwarp();
}

/// Eigenvalue-floor inverse and log-determinant (numerics.hpp:58-73, 103-122) by a whole warp, for the shape
/// matrices Cholesky rejects (rank-deficient classes in the later EM iterations: one such bin, solved by one
/// lane, used to hold its launch up for ~300 us). Two-sided Jacobi with the round-robin pairing: the (M+1)/2
/// rotations of a round touch disjoint row / column pairs and are applied by all lanes at once.
/// b: input (lower triangle read); a: scratch, receives the inverse; v: scratch (eigenvectors); rot: 4 cdbl +
/// 2 ints per pair. Returns false (warp-uniform) on non-finite values or when no eigenvalue is positive.
template <int M>
__device__ __noinline__ bool warp_eig_floor_inverse(const cdbl* b, cdbl* a, cdbl* v, cdbl* rot, double* log_det,
                                                    int lane) {
  constexpr int MM = M * M, NP = (M + 1) & ~1, HALF = NP / 2;
  for (int e = lane; e < MM; e += 32) {
    const int i = e / M, j = e - i * M;
    cdbl x = i >= j ? b[i * M + j] : cd_conj(b[j * M + i]);
    if (i == j) x.im = 0.0;
    a[e] = x;
    v[e] = cd_make(i == j ? 1.0 : 0.0, 0.0);
  }
  __syncwarp();
  int* pq = reinterpret_cast<int*>(rot + 4 * HALF);
  for (int sweep = 0; sweep < 60; ++sweep) {
    double off = 0.0, diag = 0.0;
    for (int e = lane; e < MM; e += 32) {
      const double n2 = cd_norm(a[e]);
      if (e / M == e % M) diag += n2; else off += n2;
    }
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) {
      off += __shfl_xor_sync(0xffffffffu, off, o);
      diag += __shfl_xor_sync(0xffffffffu, diag, o);
    }
    if (!isfinite(off + diag)) return false;
    if (off <= 1e-30 * diag || off == 0.0) break;
    for (int r = 0; r < NP - 1; ++r) {
      if (lane < HALF) {  // this round's rotations, from the matrix as it stands
        int p = lane == 0 ? NP - 1 : (r + lane) % (NP - 1);
        int q = lane == 0 ? r : (r - lane + (NP - 1)) % (NP - 1);
        if (p > q) {
          const int t = p;
          p = q;
          q = t;
        }
        cdbl jpp = cd_make(1.0, 0.0), jqp = cd_make(0.0, 0.0), jpq = cd_make(0.0, 0.0), jqq = cd_make(1.0, 0.0);
        bool act = q < M;
        if (act) {
          const cdbl apq = a[p * M + q];
          const double n2 = cd_norm(apq);
          if (n2 == 0.0) {
            act = false;
          } else {
            // one reciprocal square root serves the phase and tau, another the cosine: the rotation is a chain of
            // dependent FP64 special functions on four lanes while the other 28 wait for it
            const double app = a[p * M + p].re, aqq = a[q * M + q].re;
            const double inv_mag = rsqrt(n2);
            const cdbl ph = cd_make(apq.re * inv_mag, apq.im * inv_mag);  // e^{i phi}
            const double tau = 0.5 * (aqq - app) * inv_mag;
            const double t = (tau >= 0.0 ? 1.0 : -1.0) / (fabs(tau) + sqrt(1.0 + tau * tau));
            const double c = rsqrt(1.0 + t * t), sn = t * c;
            // J columns: p -> [c ; -s e^{-i phi}], q -> [s ; c e^{-i phi}]
            jpp = cd_make(c, 0.0);
            jqp = cd_make(-sn * ph.re, sn * ph.im);
            jpq = cd_make(sn, 0.0);
            jqq = cd_make(c * ph.re, -c * ph.im);
          }
        }
        rot[4 * lane] = jpp;
        rot[4 * lane + 1] = jqp;
        rot[4 * lane + 2] = jpq;
        rot[4 * lane + 3] = jqq;
        pq[2 * lane] = act ? p : -1;
        pq[2 * lane + 1] = q;
      }
      __syncwarp();
      for (int it = lane; it < HALF * M * 2; it += 32) {  // A <- A J, V <- V J (disjoint column pairs)
        const int k = it / (2 * M), rem = it - k * 2 * M, i = rem >> 1;
        const int p = pq[2 * k], q = pq[2 * k + 1];
        if (p < 0) continue;
        cdbl* mx = (rem & 1) ? v : a;
        const cdbl xp = mx[i * M + p], xq = mx[i * M + q];
        mx[i * M + p] = cd_add(cd_mul(xp, rot[4 * k]), cd_mul(xq, rot[4 * k + 1]));
        mx[i * M + q] = cd_add(cd_mul(xp, rot[4 * k + 2]), cd_mul(xq, rot[4 * k + 3]));
      }
      __syncwarp();
      for (int it = lane; it < HALF * M; it += 32) {  // A <- J^H A (disjoint row pairs)
        const int k = it / M, j = it - k * M;
        const int p = pq[2 * k], q = pq[2 * k + 1];
        if (p < 0) continue;
        const cdbl apj = a[p * M + j], aqj = a[q * M + j];
        a[p * M + j] = cd_add(cd_cmul(rot[4 * k], apj), cd_cmul(rot[4 * k + 1], aqj));
        a[q * M + j] = cd_add(cd_cmul(rot[4 * k + 2], apj), cd_cmul(rot[4 * k + 3], aqj));
      }
      __syncwarp();
      if (lane < HALF && pq[2 * lane] >= 0) {
        const int p = pq[2 * lane], q = pq[2 * lane + 1];
        a[p * M + q] = cd_make(0.0, 0.0);
        a[q * M + p] = cd_make(0.0, 0.0);
        a[p * M + p].im = 0.0;
        a[q * M + q].im = 0.0;
      }
      __syncwarp();
    }
  }
  double w[M], emax = -1.0e300;
  bool finite = true;
#pragma unroll
  for (int i = 0; i < M; ++i) {
    w[i] = a[i * M + i].re;
    finite = finite && isfinite(w[i]);
    emax = fmax(emax, w[i]);
  }
  if (!finite || !(emax > 0.0)) return false;
  double ld = 0.0;
#pragma unroll
  for (int i = 0; i < M; ++i) {
    w[i] = fmax(w[i], kEigFloorRatio * emax);
    ld += log(w[i]);
    w[i] = 1.0 / w[i];
  }
  __syncwarp();  // every lane holds the eigenvalues: a can take the inverse V diag(1/w) V^H
  for (int e = lane; e < MM; e += 32) {
    const int i = e / M, j = e - i * M;
    cdbl s = cd_make(0.0, 0.0);
#pragma unroll
    for (int q = 0; q < M; ++q) s = cd_add(s, cd_scale(cd_mulc(v[i * M + q], v[j * M + q]), w[q]));
    a[e] = s;
  }
  __syncwarp();
  *log_det = ld;
  return true;
}

/// Blocks per SM the update is compiled for: about 20 warps (the kernel is FP64 latency chains, more resident
/// warps hide them; measured on cfg2, KT = 4: 2.07 ms per step at 3 blocks, 1.77 at 4, 1.72 at 5 - 6, 1.87 at 8).
constexpr int em_update_min_blocks(int KT) { return 20 / KT < 2 ? 2 : 20 / KT > 8 ? 8 : 20 / KT; }

template <int M, int L, int KT>
__global__ void __launch_bounds__(KT * 32, em_update_min_blocks(KT)) em_update_kernel(EmUpdateArgs a) {
  using Lay = EmLayout<M, L>;
  using PL = PartLayout<M, L, KT, KT>;
  constexpr int NDOF = Lay::NDOF;
  constexpr int MM = M * M;
  __shared__ cdbl s_b[KT][MM], s_f[KT][MM], s_inv[KT][MM];
  __shared__ cdbl s_rot[KT][5 * ((M + 1) / 2)];  // the fallback's rotations: 4 cdbl + 2 ints per pair
  __shared__ double s_pi[KT], s_ld[KT];

  const int k = threadIdx.x >> 5, lane = threadIdx.x & 31;
#ifdef GSS_EXP_UPD_REVERSE
  const int f = (int)gridDim.x - 1 - (int)blockIdx.x, seg = blockIdx.y;
#else
  const int f = blockIdx.x, seg = blockIdx.y;
#endif
  const SegDev sd = a.segs[seg];
  const bool live = k < sd.K;
  const long long fk = sd.fk_off + (long long)f * KT + k;
  const long long cell0 = sd.cell_off + (long long)f * sd.nchunks;

  if (threadIdx.x == 0 && (a.mode == kEmMstep || a.mode == kEmFinal)) {
    double ll = 0.0;
    for (int c = 0; c < sd.nchunks; ++c) ll += a.cell_ll[cell0 + c];
    a.bin_ll[sd.f_off + f] = ll;
  }
  if (a.mode == kEmFinal) return;

  double my_pi = 0.0, my_ld = 0.0;
  cdbl* B = s_b[k];
  if (live) {
    bool have_b = false;      // B holds the (new) shape matrix
    bool need_invert = false;
    if (a.mode == kEmInit) {
      for (int e = lane; e < MM; e += 32) B[e] = cd_make((e / M == e % M) ? 1.0 : 0.0, 0.0);
      my_pi = 1.0 / (double)sd.K;
      have_b = need_invert = true;
    } else if (a.mode == kEmFromState) {
      for (int e = lane; e < MM; e += 32) B[e] = a.bstate[fk * MM + e];
      my_pi = a.pi[fk];
      need_invert = true;
    } else {
      double mass = 0.0;
      for (int c = 0; c < sd.nchunks; ++c) mass += (double)a.part[(cell0 + c) * a.cell_stride + PL::ACC + k];
      if (mass <= 0.0) {
        // dead class at this bin: keep its shape, floor its weight (cacgmm.hpp:319-323)
        my_pi = kWeightFloor;
        my_ld = a.logdet[fk];
      } else {
        for (int e = lane; e < MM; e += 32) B[e] = cd_make(0.0, 0.0);
        __syncwarp();
        // chunk partials -> Gram, summed in double in chunk order; both triangles are written from
        // the same sums, so hermitize (cacgmm.hpp:330) is the identity on this matrix
        for (int d = lane; d < L * NDOF; d += 32) {
          const int g = d / NDOF, j = d - g * NDOF;
          const DofInfo di = dof_info(M, L, g, j);
          if (di.kind == kIdle) continue;
          double v = 0.0;
          for (int c = 0; c < sd.nchunks; ++c)
            v += (double)a.part[(cell0 + c) * a.cell_stride + g * PL::STRIDE + k * NDOF + j];
          dof_scatter(B, M, di, v);
        }
        __syncwarp();
        const double s = (double)M / mass;  // cacgmm.hpp:327-329
        for (int e = lane; e < MM; e += 32) B[e] = cd_scale(B[e], s);
        __syncwarp();
        double tr = 0.0;
        for (int i = 0; i < M; ++i) tr += B[i * M + i].re;
        __syncwarp();
        if (tr > 0.0) {
          const double gsc = (double)M / tr;
          for (int e = lane; e < MM; e += 32) B[e] = cd_scale(B[e], gsc);
        }
        __syncwarp();
        double tr2 = 0.0;  // regularize (numerics.hpp:41-49)
        for (int i = 0; i < M; ++i) tr2 += B[i * M + i].re;
        double scale = tr2 / (double)M;
        if (!(scale > 0.0)) scale = 1.0;
        __syncwarp();
        if (lane < M) B[lane * M + lane].re += kRegEps * scale;
        my_pi = fmax(kWeightFloor, mass / (double)sd.T);
        have_b = need_invert = true;
      }
    }
    __syncwarp();
    if (have_b)
      for (int e = lane; e < MM; e += 32) a.bstate[fk * MM + e] = B[e];
    if (need_invert) {
      cdbl* F = s_f[k];
      cdbl* inv = s_inv[k];
      for (int e = lane; e < MM; e += 32) F[e] = B[e];
      __syncwarp();
      if (warp_cholesky<M>(F, lane)) {
        // log|B| = 2 sum log L_ii; B is trace-normalised to M, so the product of the (<= 8) pivots cannot
        // overflow and one logarithm replaces M of them
        double pd = 1.0;
        for (int i = 0; i < M; ++i) pd *= F[i * M + i].re;
        my_ld = 2.0 * log(pd);
        warp_cholesky_inverse<M>(F, inv, lane);
      } else if (warp_eig_floor_inverse<M>(B, F, inv, s_rot[k], &my_ld, lane)) {
        // eigenvalue-floor fallback (numerics.hpp:103-122), whole warp; the inverse is left in F
        for (int e = lane; e < MM; e += 32) inv[e] = F[e];
        __syncwarp();
      } else {
        // no usable eigenvalue: one lane repeats the decomposition and then retries on regularize(B)
        // (cacgmm.hpp:134-140); practically never taken
        __syncwarp();
        if (lane == 0) {
          cdbl fact[MM], work[MM], linv[MM];
          double wv[M];
          double ld = 0.0;
          for (int i = 0; i < MM; ++i) fact[i] = B[i];
          int st = hermitian_inverse_logdet<M>(fact, M, linv, &ld, work, wv);
          if (st != kLinOk) {
            for (int i = 0; i < MM; ++i) fact[i] = B[i];
            regularize_inplace(fact, M, M, kRegEps);
            st = hermitian_inverse_logdet<M>(fact, M, linv, &ld, work, wv);
          }
          if (st != kLinOk) {
            atomicMin(&a.status[seg], make_status(5 /*SingularMatrixError*/, f));
            ld = 0.0;
            for (int i = 0; i < MM; ++i) linv[i] = cd_make((i / M == i % M) ? 1.0 : 0.0, 0.0);
          }
          for (int i = 0; i < MM; ++i) inv[i] = linv[i];
          F[0].re = ld;
        }
        __syncwarp();
        my_ld = F[0].re;
      }
      // B^-1 is rounded to cfloat before use (cacgmm.hpp:144-149)
      for (int d = lane; d < L * NDOF; d += 32) {
        const int g = d / NDOF, j = d - g * NDOF;
        a.coef[sd.coef_off + ((long long)f * L + g) * (KT * NDOF) + k * NDOF + j] =
            dof_coef(inv, M, dof_info(M, L, g, j));
      }
      if (lane == 0) a.logdet[fk] = my_ld;
    }
    if (lane == 0) a.pi[fk] = my_pi;
  } else if (a.mode == kEmInit || a.mode == kEmFromState) {
    // padded class (K <= k < KT): zero coefficients; it is masked off by ck = -inf
    for (int d = lane; d < L * NDOF; d += 32) {
      const int g = d / NDOF, j = d - g * NDOF;
      a.coef[sd.coef_off + ((long long)f * L + g) * (KT * NDOF) + k * NDOF + j] = 0.f;
    }
  }
  if (lane == 0) {
    s_pi[k] = my_pi;
    s_ld[k] = my_ld;
  }
  __syncthreads();

  // E-step constants per activity pattern (cacgmm.hpp:196-237):
  //   ck = lp + c0 - log|B_k|, lp = log max(1e-10, pi_k) - log z, z = sum of active pi
  const double c0 = a.c0;  // -M log(2 pi) + lgamma(M), from the host
  float* tab = a.ck + sd.tab_off + (long long)f * sd.npat * KT;
  for (int idx = threadIdx.x; idx < sd.npat * KT; idx += KT * 32) {
    const int p = idx / KT, kk = idx - p * KT;
    const uint32_t mask = a.masks[sd.mask_off + p];
    float v = -CUDART_INF_F;
    if (kk < sd.K) {
      double z = 0.0;
      for (int q = 0; q < sd.K; ++q)
        if (mask & (1u << q)) z += s_pi[q];
      bool active;
      double lp;
      if (z <= 0.0) {  // no active class: noise class alone, or uniform (cacgmm.hpp:217-226)
        active = sd.noise >= 0 ? kk == sd.noise : true;
        lp = sd.noise >= 0 ? 0.0 : -log((double)sd.K);
      } else {
        active = (mask >> kk) & 1u;
        lp = log(fmax(kWeightFloor, s_pi[kk])) - log(z);
      }
      if (active) v = (float)((lp + c0 - s_ld[kk]) * 1.4426950408889634074);  // log2 units for the sweep
    }
    tab[idx] = v;
  }
}

// ---------------------------------------------------------------------------
// MVDR statistics from posteriors held in memory (the stage entry point of
// beamform.hpp:35-85). Same lane layout and cell format as the FINAL sweep.
// ---------------------------------------------------------------------------
template <int M, int L, int KT>
__global__ void __launch_bounds__(kEmThreads) mvdr_stats_kernel(StatsPassArgs a) {
  using Lay = EmLayout<M, L>;
  using PL = PartLayout<M, L, KT, 2>;
  constexpr int NDOF = Lay::NDOF;
  constexpr int SLOTS = kEmThreads / L;
  constexpr int NW = kEmThreads / 32;
  extern __shared__ float4 smem_f4[];
  float* red = reinterpret_cast<float*>(smem_f4);

  const int tid = threadIdx.x;
  const WorkItem wi = a.work[blockIdx.x];
  const int f = blockIdx.y;
  const SegDev sd = a.segs[wi.seg];
  const int t0 = wi.chunk * sd.TC;
  const int nt = min(sd.TC, sd.T - t0);
  const int g = tid % L, slot = tid / L;
  const float2* src = a.y + sd.y_off + ((long long)f * sd.T + t0) * M;
  const float* gsrc = a.gamma + sd.g_off + ((long long)f * sd.T + t0) * sd.K;
  FramePlan<M, L> plan;
  plan.init(g);
  float acc_t[NDOF], acc_b[NDOF];
#pragma unroll
  for (int j = 0; j < NDOF; ++j) acc_t[j] = acc_b[j] = 0.f;
  float tmass = 0.f;
  for (int fb = slot; fb < nt; fb += SLOTS) {
    float pv[NDOF];
    plan.dofs(src + (long long)fb * M, pv);  // straight from global/L2: one use per element
    const float* gr = gsrc + (long long)fb * sd.K;
    const float wt = gr[sd.target];
    float wb = 0.f;
    for (int k = 0; k < sd.K; ++k)
      if (k != sd.target) wb += gr[k];
    tmass += wt;
#pragma unroll
    for (int j = 0; j < NDOF; ++j) {
      acc_t[j] = fmaf(wt, pv[j], acc_t[j]);
      acc_b[j] = fmaf(wb, pv[j], acc_b[j]);
    }
  }
#pragma unroll
  for (int o = L; o < 32; o <<= 1) {
#pragma unroll
    for (int j = 0; j < NDOF; ++j) {
      acc_t[j] += __shfl_xor_sync(0xffffffffu, acc_t[j], o);
      acc_b[j] += __shfl_xor_sync(0xffffffffu, acc_b[j], o);
    }
    tmass += __shfl_xor_sync(0xffffffffu, tmass, o);
  }
  const int lane = tid & 31, warp = tid >> 5;
  if (lane < L) {
    float* r = red + (warp * L + lane) * PL::STRIDE;
#pragma unroll
    for (int j = 0; j < NDOF; ++j) {
      r[j] = acc_t[j];
      r[NDOF + j] = acc_b[j];
    }
#pragma unroll
    for (int k = 0; k < KT; ++k) r[PL::ACC + k] = (k == sd.target) ? tmass : 0.f;
  }
  __syncthreads();
  float* out = a.part + (sd.cell_off + (long long)f * sd.nchunks + wi.chunk) * a.cell_stride;
  for (int i = tid; i < PL::CELL; i += kEmThreads) {
    float s = 0.f;
#pragma unroll
    for (int w = 0; w < NW; ++w) s += red[w * PL::CELL + i];
    out[i] = s;
  }
}

/// chunk partials -> Phi_target, Phi_background (x 1/T) in FP64. One thread per (seg, f).
template <int M, int L, int KT>
__global__ void mvdr_stats_final_kernel(StatsFinalArgs a) {
  using PL = PartLayout<M, L, KT, 2>;
  constexpr int NDOF = PL::NDOF;
  const int f = blockIdx.x * blockDim.x + threadIdx.x;
  if (f >= a.F) return;
  const SegDev sd = a.segs[blockIdx.y];
  const long long cell0 = sd.cell_off + (long long)f * sd.nchunks;
  cdbl gt[M * M], gb[M * M];
  for (int i = 0; i < M * M; ++i) gt[i] = gb[i] = cd_make(0.0, 0.0);
  for (int g = 0; g < L; ++g)
    for (int j = 0; j < NDOF; ++j) {
      const DofInfo di = dof_info(M, L, g, j);
      if (di.kind == kIdle) continue;
      double vt = 0.0, vb = 0.0;
      for (int c = 0; c < sd.nchunks; ++c) {
        const float* p = a.part + (cell0 + c) * a.cell_stride + g * PL::STRIDE;
        vt += (double)p[j];
        vb += (double)p[NDOF + j];
      }
      dof_scatter(gt, M, di, vt);
      dof_scatter(gb, M, di, vb);
    }
  double mass = 0.0;
  for (int c = 0; c < sd.nchunks; ++c) mass += (double)a.part[(cell0 + c) * a.cell_stride + PL::ACC + sd.target];
  const double inv_t = 1.0 / (double)sd.T;
  const long long o = (sd.f_off + f) * (long long)(M * M);
  for (int i = 0; i < M * M; ++i) {
    a.phi_t[o + i] = cd_scale(gt[i], inv_t);
    a.phi_b[o + i] = cd_scale(gb[i], inv_t);
  }
  a.tmass[sd.f_off + f] = mass;
}

}  // namespace gssb
