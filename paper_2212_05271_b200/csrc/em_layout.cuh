// em_layout.cuh -- how the M x M Hermitian outer product P = y y^H of one frame
// is split over the L lanes that cooperate on that frame in the cACGMM / MVDR
// accumulation kernels.
//
// P has M^2 real degrees of freedom ("dofs"): M real diagonal entries and
// M(M-1)/2 complex off-diagonal pairs. They are enumerated by cyclic
// diagonals so that every matrix row owns exactly M dofs and every lane runs
// the same instruction stream (only its shared-memory addresses differ):
//
//   row r, jr = 0          : P[r][r]                         (kDiag)
//   row r, jr = 2d-1, 2d   : Re / Im of P[r][(r+d) % M], d = 1..(M-1)/2
//   row r, jr = M-1 (M even): the half diagonal d = M/2 holds M/2 complex
//        pairs; row r < M/2 takes Re P[r][r+M/2] (kHalfRe), row r >= M/2
//        takes Im P[r][r-M/2] (kHalfIm).
//
// Lane g of L owns rows g, g+L, g+2L, ... (RPL of them; rows >= M are idle).
//
// Used for:  q = y^H Binv y = sum_dofs coef * P_dof          (cacgmm.hpp:156-174)
//            Gram = sum_t w_t P(t)                          (numerics.hpp:128-152)
#pragma once

#include "linalg.cuh"

namespace gssb {

enum DofKind { kDiag = 0, kRe = 1, kIm = 2, kHalfRe = 3, kHalfIm = 4, kIdle = 5 };

template <int M, int L>
struct EmLayout {
  static constexpr int RPL = (M + L - 1) / L;         // rows per lane
  static constexpr int D = (M - 1) / 2;               // full cyclic diagonals
  static constexpr int HALF = (M % 2 == 0) ? 1 : 0;   // half diagonal present
  static constexpr int NZ = D + HALF;                 // partner vectors per row
  static constexpr int NDOF = RPL * M;                // dofs per lane
};

struct DofInfo {
  int row, col, kind;
};

/// dof `idx` (0 <= idx < RPL*M) of lane g.
GSS_HD DofInfo dof_info(int M, int L, int g, int idx) {
  DofInfo d;
  const int slot = idx / M, jr = idx % M;
  d.row = g + slot * L;
  d.col = d.row;
  d.kind = kIdle;
  if (d.row >= M) return d;
  const int dfull = (M - 1) / 2;
  if (jr == 0) {
    d.kind = kDiag;
  } else if (jr <= 2 * dfull) {
    const int dd = (jr + 1) / 2;
    d.col = (d.row + dd) % M;
    d.kind = (jr & 1) ? kRe : kIm;
  } else {  // half diagonal (M even)
    d.col = (d.row + M / 2) % M;
    d.kind = d.row < M / 2 ? kHalfRe : kHalfIm;
  }
  return d;
}

/// Coefficient multiplying dof (row,col,kind) in q = sum_{mn} conj(y_m) Binv[m][n] y_n.
GSS_HD float dof_coef(const cdbl* binv, int M, DofInfo d) {
  switch (d.kind) {
    case kDiag: return (float)binv[d.row * M + d.row].re;
    case kRe:
    case kHalfRe: return (float)(2.0 * binv[d.row * M + d.col].re);
    case kIm:
    case kHalfIm: return (float)(2.0 * binv[d.row * M + d.col].im);
    default: return 0.0f;
  }
}

/// Scatter an accumulated dof into the Hermitian Gram matrix (row-major M x M).
GSS_HD void dof_scatter(cdbl* gram, int M, DofInfo d, double v) {
  switch (d.kind) {
    case kDiag:
      gram[d.row * M + d.row].re = v;
      break;
    case kRe:
    case kHalfRe:
      gram[d.row * M + d.col].re = v;
      gram[d.col * M + d.row].re = v;
      break;
    case kIm:
    case kHalfIm:
      gram[d.row * M + d.col].im = v;
      gram[d.col * M + d.row].im = -v;
      break;
    default:
      break;
  }
}

}  // namespace gssb
