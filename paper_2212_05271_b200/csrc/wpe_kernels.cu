// wpe_kernels.cu -- WPE dereverberation (wpe.hpp:40-56 frame powers, :61-98
// per-bin iteration, :105-120 driver; numerics.hpp:81-94 Hermitian solve,
// :128-152 weighted Gram).
//
// Window formulation. The reference materialises, per frame t, the tap-stacked
// row a_t = [y_{t-d}, y_{t-d-1}, ..., y_{t-d-taps+1} | y_t]. With the taps
// stored in REVERSE order the stacked history is one contiguous slice of the
// per-bin slab: element e = u*M + c (u = taps-1-k) of the history of frame t is
// y[t - H + u][c], H = d + taps - 1. So the correlation matrix
//   R[e][e'] = sum_t w_t y[t-H+e/M][e%M] conj(y[t-H+e'/M][e'%M])
// and the cross term P[e][c] = sum_t w_t y[t-H+e/M][e%M] conj(y[t][c]) are
// windowed correlations of the slab with itself; the tap-stacked matrix is
// never built. The solve runs in the same (permuted) ordering; a symmetric
// permutation of R leaves G = R^-1 P unchanged up to rounding order.
//
// Kernels per iteration:
//   wpe_power_kernel  w_t = 1/lambda_t from the current estimate
//   wpe_gram_kernel   8x8 complex register tiles, one warp per tile, one lane
//                     per frame; slab staged channel-major in shared memory
//   wpe_solve2_kernel FP64 Cholesky of the km x km system per (segment, bin)
//   wpe_apply2_kernel Y_f = observed - history * conj(G)
#include "kernels.h"

namespace gssb {

namespace {

constexpr int kGramWarps = 16;  // one CTA of 16 warps per SM: the slab is staged once for 16 tiles
constexpr int kGramThreads = kGramWarps * 32;
constexpr int kGramTileFrames = 512;  // frames staged per shared-memory tile

// Output tiling of the Gram: R's lower triangle in row blocks of 8 window elements x column blocks of
// kTC, followed by the cross term P (km x M) in the same row blocks x ceil(M/kTC) column blocks.
constexpr int kTC = 4;                 // tile columns (8 x 4 complex accumulators = 64 registers per lane)
constexpr int kTileElems = 8 * kTC;
constexpr int kCPR = 8 / kTC;          // column blocks per row block on the diagonal

__host__ __device__ inline int gram_row_blocks(int km) { return (km + 7) / 8; }
__host__ __device__ inline int gram_tri_tiles(int nb) { return kCPR * nb * (nb + 1) / 2; }
__host__ __device__ inline int gram_p_cols(int M) { return (M + kTC - 1) / kTC; }
__host__ __device__ inline int gram_num_tiles(int km, int M) {
  const int nb = gram_row_blocks(km);
  return gram_tri_tiles(nb) + nb * gram_p_cols(M);
}
/// tile holding R[i][j], j <= i
__host__ __device__ inline int gram_r_tile(int i, int j) {
  const int bi = i >> 3;
  return kCPR * bi * (bi + 1) / 2 + j / kTC;
}
/// tile holding P[i][c]
__host__ __device__ inline int gram_p_tile(int i, int c, int nb, int M) {
  return gram_tri_tiles(nb) + (i >> 3) * gram_p_cols(M) + c / kTC;
}

/// tile index -> (row block, column block, is-cross-term)
__device__ __forceinline__ void gram_tile_coords(int tile, int nb, int M, int& bi, int& bj, bool& cross) {
  const int ntri = gram_tri_tiles(nb);
  if (tile >= ntri) {
    const int pc = gram_p_cols(M);
    bi = (tile - ntri) / pc;
    bj = (tile - ntri) % pc;
    cross = true;
    return;
  }
  int r = 0;
  while (kCPR * (r + 1) * (r + 2) / 2 <= tile) ++r;
  bi = r;
  bj = tile - kCPR * r * (r + 1) / 2;
  cross = false;
}

__device__ __forceinline__ void cp_async_bytes8(void* smem_dst, const void* gsrc) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(smem_dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(d), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async_bytes4(void* smem_dst, const void* gsrc) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(smem_dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(d), "l"(gsrc) : "memory");
}

}  // namespace

// ---------------------------------------------------------------------------
// lambda_t and the Gram weights (wpe.hpp:40-56, :86-87). One thread per (f,t).
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) wpe_power_kernel(WpeArgs a) {
  const SegDev sd = a.segs[blockIdx.z];
  if (!sd.wpe_active) return;
  const int f = blockIdx.y;
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= sd.T) return;
  const int M = a.M;
  const float2* y = a.ycur + sd.y_off + (long long)f * sd.T * M;
  const int lo = max(0, t - a.psd_context), hi = min(sd.T - 1, t + a.psd_context);
  double acc = 0.0;
  for (int u = lo; u <= hi; ++u) {
    float s = 0.f;  // Eigen's squaredNorm on a cfloat row accumulates in float
    for (int c = 0; c < M; ++c) {
      const float2 v = y[(long long)u * M + c];
      s += v.x * v.x + v.y * v.y;
    }
    acc += (double)s / (double)M;
  }
  const float lambda = (float)fmax(kPowerFloor, acc / (double)(hi - lo + 1));
  a.w[sd.w_off + (long long)f * sd.T + t] = 1.0f / lambda;
}

// ---------------------------------------------------------------------------
// Weighted Gram. grid (tile groups * wchunks, F, segments), block 256, two CTAs per SM.
// Warp w of group g owns output tile g*8+w (8 x kTC complex accumulators per lane) for the CTA's
// whole frame range; lane l accumulates frames l, l+32, ... and the 32 lanes are summed at the end.
// ---------------------------------------------------------------------------
template <int M>
__global__ void __launch_bounds__(kGramThreads, 1) wpe_gram_kernel(WpeArgs a) {
  extern __shared__ float4 smem_f4[];
  const SegDev sd = a.segs[blockIdx.z];
  if (!sd.wpe_active) return;
  const int f = blockIdx.y;
  const int km = a.taps * M, nb = gram_row_blocks(km), ntiles = gram_num_tiles(km, M);
  const int ngroups = (ntiles + kGramWarps - 1) / kGramWarps;
  const int group = blockIdx.x % ngroups, chunk = blockIdx.x / ngroups;
  if (chunk >= sd.wchunks) return;
  const int H = a.delay + a.taps - 1;
  // Slab layout. Odd M: frame-major [frame][M]; the window of a frame is then ONE contiguous slice, a lane
  // addresses its 8 rows / kTC columns as base + immediate, and lanes (= consecutive frames, odd stride)
  // hit distinct bank pairs. Even M: that stride would be an 8-byte-bank multiple, so the slab is kept
  // channel-major [channel][frame] (odd pitch) and every row / column carries its own offset.
  constexpr bool CONTIG = (M & 1) != 0;
  const int slab_frames = kGramTileFrames + H + 8;  // + 8: padded rows / columns of the last blocks look ahead
  const int pitch = slab_frames | 1;
  const int slab_elems = CONTIG ? M * slab_frames : M * pitch;
  const int buf_floats = 2 * slab_elems + kGramTileFrames;  // one pipeline stage: slab + weights
  float* stage0 = reinterpret_cast<float*>(smem_f4);

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int tile = group * kGramWarps + warp;
  const bool live = tile < ntiles;
  int bi = 0, bj = 0;
  bool cross = false;
  if (live) gram_tile_coords(tile, nb, M, bi, bj, cross);
  int rowoff[8], coloff[kTC];
#pragma unroll
  for (int r = 0; r < 8; ++r) {
    if (CONTIG) {
      rowoff[r] = 8 * bi + r;  // window element = slab offset from the frame's window start
    } else {
      const int e = min(8 * bi + r, km - 1);  // padded rows alias the last valid element
      rowoff[r] = (e % M) * pitch + e / M;
    }
  }
#pragma unroll
  for (int c = 0; c < kTC; ++c) {
    const int e = kTC * bj + c;
    if (CONTIG) {
      coloff[c] = cross ? H * M + e : e;  // unused columns of the last block read finite look-ahead data
    } else if (cross) {
      coloff[c] = (e < M ? e : 0) * pitch + H;
    } else {
      const int e2 = min(e, km - 1);
      coloff[c] = (e2 % M) * pitch + e2 / M;
    }
  }
  float accr[8][kTC], acci[8][kTC];
#pragma unroll
  for (int r = 0; r < 8; ++r)
#pragma unroll
    for (int c = 0; c < kTC; ++c) accr[r][c] = acci[r][c] = 0.f;

  const int t_begin = chunk * sd.WTC, t_end = min(sd.T, t_begin + sd.WTC);
  const float2* yf = a.yobs + sd.y_off + (long long)f * sd.T * M;
  const float* wf = a.w + sd.w_off + (long long)f * sd.T;
  const int ntl = (t_end - t_begin + kGramTileFrames - 1) / kGramTileFrames;

  // stage frames [tb-H, tb+nfr+8); frames < 0 or >= T are zero (wpe.hpp:74-75)
  auto issue = [&](int tl, int buf) {
    const int tb = t_begin + tl * kGramTileFrames;
    const int nfr = min(kGramTileFrames, t_end - tb);
    float2* slab = reinterpret_cast<float2*>(stage0 + buf * buf_floats);
    float* wsm = stage0 + buf * buf_floats + 2 * slab_elems;
    for (int i = tid; i < (nfr + H + 8) * M; i += kGramThreads) {
      const int fr = i / M, c = i - fr * M;
      const int t = tb - H + fr;
      float2* dst = slab + (CONTIG ? i : c * pitch + fr);
      if (t >= 0 && t < sd.T)
        cp_async_bytes8(dst, yf + (long long)t * M + c);
      else
        *dst = make_float2(0.f, 0.f);
    }
    for (int i = tid; i < nfr; i += kGramThreads) cp_async_bytes4(wsm + i, wf + tb + i);
    asm volatile("cp.async.commit_group;\n" ::: "memory");
  };

  issue(0, 0);
  for (int tl = 0; tl < ntl; ++tl) {
    const int buf = tl & 1;
    if (tl + 1 < ntl) {
      issue(tl + 1, buf ^ 1);
      asm volatile("cp.async.wait_group 1;\n" ::: "memory");
    } else {
      asm volatile("cp.async.wait_group 0;\n" ::: "memory");
    }
    __syncthreads();
    const int nfr = min(kGramTileFrames, t_end - (t_begin + tl * kGramTileFrames));
    const float2* slab = reinterpret_cast<const float2*>(stage0 + buf * buf_floats);
    const float* wsm = stage0 + buf * buf_floats + 2 * slab_elems;
    if (live) {
      for (int fi = lane; fi < nfr; fi += 32) {
        const float w = wsm[fi];
        const float2* base = slab + (CONTIG ? fi * M : fi);
        float2 ar[8], bc[kTC];
#pragma unroll
        for (int r = 0; r < 8; ++r) ar[r] = CONTIG ? base[rowoff[0] + r] : base[rowoff[r]];
#pragma unroll
        for (int c = 0; c < kTC; ++c) {
          const float2 v = CONTIG ? base[coloff[0] + c] : base[coloff[c]];
          bc[c] = make_float2(v.x * w, v.y * w);
        }
#pragma unroll
        for (int r = 0; r < 8; ++r)
#pragma unroll
          for (int c = 0; c < kTC; ++c) {
            // a * conj(b)
            accr[r][c] = fmaf(ar[r].x, bc[c].x, accr[r][c]);
            accr[r][c] = fmaf(ar[r].y, bc[c].y, accr[r][c]);
            acci[r][c] = fmaf(ar[r].y, bc[c].x, acci[r][c]);
            acci[r][c] = fmaf(-ar[r].x, bc[c].y, acci[r][c]);
          }
      }
    }
    __syncthreads();  // everyone is done with `buf` before the next iteration refills it
  }
  if (!live) return;
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1)
#pragma unroll
    for (int r = 0; r < 8; ++r)
#pragma unroll
      for (int c = 0; c < kTC; ++c) {
        accr[r][c] += __shfl_xor_sync(0xffffffffu, accr[r][c], o);
        acci[r][c] += __shfl_xor_sync(0xffffffffu, acci[r][c], o);
      }
  float2* out = a.gram + ((sd.wcell_off + (long long)f * sd.wchunks + chunk) * ntiles + tile) * kTileElems;
  // lane l writes entry l (static register indices: select by predicate)
#pragma unroll
  for (int r = 0; r < 8; ++r)
#pragma unroll
    for (int c = 0; c < kTC; ++c) {
      const int idx = r * kTC + c;
      if ((idx & 31) == lane) out[idx] = make_float2(accr[r][c], acci[r][c]);
    }
}

// ---------------------------------------------------------------------------
// Solve R G = P per (segment, bin) in FP64 (wpe.hpp:90-94; numerics.hpp:32-49, 81-94): hermitize, regularize,
// Cholesky, two triangular solves. grid (F, segments), block 128, four blocks per SM.
//
// The first version (full square storage, 256 threads, separate forward / backward substitution) spent 55 %
// of its samples at block barriers (ncu, profiles/ncu_full_r01.md): its serial pieces -- substitution inside
// a panel by <= 7 threads, one row per thread with a 36-deep dependent FP64 chain in the panel solve -- left
// 2 resident blocks x 8 warps mostly idle (4.9 ms per cfg2 step; this form: 3.0 ms). What changed:
//   * packed lower-triangular storage (km(km+1)/2 + M km complex doubles = 48 KB at km = 70): four problems
//     per SM, so one block's serial sections overlap the others' parallel ones;
//   * the right-hand sides ride along as M extra rows W = P^H of the matrix being factored: after the last
//     panel they hold Z^H = (L^-1 P)^H, the forward substitution costs no extra pass;
//   * each 8 x 8 diagonal block is inverted once by warp 0 (it replaces the block in memory); the panel solve
//     and the backward substitution become independent dot products of depth <= 8 per output;
//   * trailing updates split every dot product over two accumulators.
// A pivot <= 0 fails like Eigen's LLT and takes the eigenvalue-floor fallback (numerics.hpp:58-73, 90-93).
// ---------------------------------------------------------------------------
namespace {
#ifndef GSS_SOLVE_THREADS
#define GSS_SOLVE_THREADS 128
#define GSS_SOLVE_MINB 4
#endif
constexpr int kSolveThreads = GSS_SOLVE_THREADS;
constexpr int kSolveTY = kSolveThreads / 16;  // thread rows of the trailing update's 16-column thread grid
constexpr int kPB = 8;
__device__ __forceinline__ int tri(int i) { return i * (i + 1) / 2; }
}  // namespace

/// X = A^-1 B through the eigenvalue-floor fallback of numerics.hpp:58-73 / :90-93, by the whole block:
/// parallel-order cyclic Jacobi (round-robin pairing: the n/2 rotations of a round act on disjoint index pairs,
/// so their column updates, then their row updates, run side by side), eigenvalues floored at 1e-10 of the
/// largest, X = V diag(1/w) V^H B. A (n x n, full Hermitian, destroyed), V, C (n x nrhs) and w live in a global
/// scratch slot; `rot` is shared memory for n/2 + 1 rotations (4 complex doubles each) and `red` for the
/// convergence sums. One thread doing the same (the first version) took 60 ms for a single 40 x 40 bin and
/// held its whole launch up; this takes about a millisecond. Returns false when no positive finite eigenvalue
/// exists (SingularMatrixError). Must be called by every thread of the block.
__device__ bool block_eig_floor_solve(cdbl* A, int n, cdbl* B, int nrhs, cdbl* V, cdbl* C, double* w, cdbl* rot,
                                      double* red, int tid, int nth) {
  for (int idx = tid; idx < n * n; idx += nth) V[idx] = cd_make(idx / n == idx % n ? 1.0 : 0.0, 0.0);
  for (int i = tid; i < n; i += nth) A[i * n + i].im = 0.0;
  const int np = (n + 1) & ~1, half = np / 2;  // players of the round-robin (an odd n gets a bye)
  __syncthreads();
  for (int sweep = 0; sweep < 60; ++sweep) {
    double off = 0.0, diag = 0.0;
    for (int idx = tid; idx < n * n; idx += nth) {
      const double v = cd_norm(A[idx]);
      if (idx / n == idx % n) diag += v; else off += v;
    }
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) {
      off += __shfl_xor_sync(0xffffffffu, off, o);
      diag += __shfl_xor_sync(0xffffffffu, diag, o);
    }
    if ((tid & 31) == 0) {
      red[2 * (tid >> 5)] = off;
      red[2 * (tid >> 5) + 1] = diag;
    }
    __syncthreads();
    off = diag = 0.0;
    for (int wq = 0; wq < nth / 32; ++wq) {
      off += red[2 * wq];
      diag += red[2 * wq + 1];
    }
    __syncthreads();
    if (!isfinite(off + diag)) return false;
    if (off <= 1e-30 * diag || off == 0.0) break;
    for (int r = 0; r < np - 1; ++r) {
      // 1. the round's rotations, from the matrix as it stands
      if (tid < half) {
        int p = tid == 0 ? np - 1 : (r + tid) % (np - 1);
        int q = tid == 0 ? r : (r - tid + (np - 1)) % (np - 1);
        if (p > q) {
          const int t = p;
          p = q;
          q = t;
        }
        cdbl jpp = cd_make(1.0, 0.0), jqp = cd_make(0.0, 0.0), jpq = cd_make(0.0, 0.0), jqq = cd_make(1.0, 0.0);
        bool act = q < n;
        if (act) {
          const cdbl apq = A[p * n + q];
          const double mag = sqrt(cd_norm(apq));
          if (mag == 0.0) {
            act = false;
          } else {
            const double app = A[p * n + p].re, aqq = A[q * n + q].re;
            const cdbl ph = cd_make(apq.re / mag, apq.im / mag);  // e^{i phi}
            const double tau = (aqq - app) / (2.0 * mag);
            const double t = (tau >= 0.0 ? 1.0 : -1.0) / (fabs(tau) + sqrt(1.0 + tau * tau));
            const double c = 1.0 / sqrt(1.0 + t * t), sn = t * c;
            // J columns: p -> [c ; -s e^{-i phi}], q -> [s ; c e^{-i phi}]
            jpp = cd_make(c, 0.0);
            jqp = cd_make(-sn * ph.re, sn * ph.im);
            jpq = cd_make(sn, 0.0);
            jqq = cd_make(c * ph.re, -c * ph.im);
          }
        }
        rot[4 * tid] = jpp;
        rot[4 * tid + 1] = jqp;
        rot[4 * tid + 2] = jpq;
        rot[4 * tid + 3] = jqq;
        reinterpret_cast<int*>(rot + 4 * half)[2 * tid] = act ? p : -1;
        reinterpret_cast<int*>(rot + 4 * half)[2 * tid + 1] = q;
      }
      __syncthreads();
      const int* pq = reinterpret_cast<const int*>(rot + 4 * half);
      // 2. A <- A J and V <- V J (disjoint column pairs)
      for (int it = tid; it < half * n * 2; it += nth) {
        const int k = it / (2 * n), rem = it - k * 2 * n, i = rem >> 1;
        const int p = pq[2 * k], q = pq[2 * k + 1];
        if (p < 0) continue;
        cdbl* Mx = (rem & 1) ? V : A;
        const cdbl xp = Mx[i * n + p], xq = Mx[i * n + q];
        Mx[i * n + p] = cd_add(cd_mul(xp, rot[4 * k]), cd_mul(xq, rot[4 * k + 1]));
        Mx[i * n + q] = cd_add(cd_mul(xp, rot[4 * k + 2]), cd_mul(xq, rot[4 * k + 3]));
      }
      __syncthreads();
      // 3. A <- J^H A (disjoint row pairs)
      for (int it = tid; it < half * n; it += nth) {
        const int k = it / n, j = it - k * n;
        const int p = pq[2 * k], q = pq[2 * k + 1];
        if (p < 0) continue;
        const cdbl apj = A[p * n + j], aqj = A[q * n + j];
        A[p * n + j] = cd_add(cd_cmul(rot[4 * k], apj), cd_cmul(rot[4 * k + 1], aqj));
        A[q * n + j] = cd_add(cd_cmul(rot[4 * k + 2], apj), cd_cmul(rot[4 * k + 3], aqj));
      }
      __syncthreads();
      if (tid < half && pq[2 * tid] >= 0) {
        const int p = pq[2 * tid], q = pq[2 * tid + 1];
        A[p * n + q] = cd_make(0.0, 0.0);
        A[q * n + p] = cd_make(0.0, 0.0);
        A[p * n + p].im = 0.0;
        A[q * n + q].im = 0.0;
      }
      __syncthreads();
    }
  }
  // eigenvalues, floored at 1e-10 of the largest (numerics.hpp:64-72)
  double emax = -1.0e300;
  bool finite = true;
  for (int i = 0; i < n; ++i) {
    const double v = A[i * n + i].re;
    finite = finite && isfinite(v);
    emax = fmax(emax, v);
  }
  if (!finite || !(emax > 0.0)) return false;
  for (int i = tid; i < n; i += nth) w[i] = fmax(A[i * n + i].re, kEigFloorRatio * emax);
  __syncthreads();
  for (int idx = tid; idx < n * nrhs; idx += nth) {  // C = diag(1/w) V^H B
    const int e = idx / nrhs, c = idx - e * nrhs;
    cdbl sacc = cd_make(0.0, 0.0);
    for (int j = 0; j < n; ++j) sacc = cd_add(sacc, cd_cmul(V[j * n + e], B[j * nrhs + c]));
    C[idx] = cd_scale(sacc, 1.0 / w[e]);
  }
  __syncthreads();
  for (int idx = tid; idx < n * nrhs; idx += nth) {  // X = V C, written over B
    const int i = idx / nrhs, c = idx - i * nrhs;
    cdbl sacc = cd_make(0.0, 0.0);
    for (int e = 0; e < n; ++e) sacc = cd_add(sacc, cd_mul(V[i * n + e], C[e * nrhs + c]));
    B[idx] = sacc;
  }
  __syncthreads();
  return true;
}

__global__ void __launch_bounds__(kSolveThreads, GSS_SOLVE_MINB) wpe_solve2_kernel(WpeArgs a) {
  extern __shared__ float4 smem_f4[];
  const SegDev sd = a.segs[blockIdx.y];
  if (!sd.wpe_active) return;
  const int f = blockIdx.x;
  const int M = a.M, km = a.taps * M, nb = gram_row_blocks(km), ntiles = gram_num_tiles(km, M);
  cdbl* Lp = reinterpret_cast<cdbl*>(smem_f4);         // packed lower triangle, row i at tri(i)
  cdbl* W = Lp + tri(km);                              // M x km: P^H, then Z^H, then X^H
  cdbl* s_linv = W + (size_t)M * km;                   // kPB x kPB scratch of warp 0
  __shared__ double s_tr;
  __shared__ int s_fail, s_slot;
  const int tid = threadIdx.x, nth = kSolveThreads;
  const int lane = tid & 31, warp = tid >> 5;
  const float2* tiles = a.gram + (sd.wcell_off + (long long)f * sd.wchunks) * ntiles * kTileElems;
  const long long chunk_stride = (long long)ntiles * kTileElems;
  const int KMP = (km + 7) & ~7, NR = wpe_tc_operand_rows(km), N2 = NR > 128 ? NR - 128 : 0, NCT = NR + N2;
  const float* raw = a.gram_raw + (sd.wcell_off + (long long)f) * (long long)(128 * NCT);

  // hermitized R[i][j] (j <= i) and P[i][c] in double from this iteration's Gram (either producer)
  auto G = [&](int x, int y) -> double {
    if (x < 128) return (double)raw[x * NCT + y];
    if (y < 128) return (double)raw[y * NCT + x];
    // corner accumulator (M = 64 MMA on rows NR-64..NR): row r sits in tensor-memory lane 32 (r / 16) + r % 16,
    // and the Gram kernel writes lane l to row l of `raw`
    const int r = x - (NR - 64);
    return (double)raw[((r >> 4) * 32 + (r & 15)) * NCT + NR + (y - 128)];
  };
  auto load_r = [&](int i, int j) -> cdbl {
    double re, im;
    if (a.use_tc) {
      re = G(i, j) + G(KMP + i, KMP + j);
      im = G(KMP + i, j) - G(i, KMP + j);
    } else {
      const float2* p = tiles + (long long)gram_r_tile(i, j) * kTileElems + (i & 7) * kTC + j % kTC;
      re = im = 0.0;
      for (int c = 0; c < sd.wchunks; ++c) {
        const float2 v = p[c * chunk_stride];
        re += (double)v.x;
        im += (double)v.y;
      }
    }
    return cd_make(re, i == j ? 0.0 : im);  // hermitize (numerics.hpp:32-38): both triangles from the same sums
  };
  auto load_p = [&](int i, int c) -> cdbl {
    if (a.use_tc)
      return cd_make(G(i, 2 * KMP + c) + G(KMP + i, 2 * KMP + 8 + c), G(KMP + i, 2 * KMP + c) - G(i, 2 * KMP + 8 + c));
    const float2* p = tiles + (long long)gram_p_tile(i, c, nb, M) * kTileElems + (i & 7) * kTC + c % kTC;
    double re = 0.0, im = 0.0;
    for (int ch = 0; ch < sd.wchunks; ++ch) {
      const float2 v = p[ch * chunk_stride];
      re += (double)v.x;
      im += (double)v.y;
    }
    return cd_make(re, im);
  };

  for (int idx = tid; idx < km * km; idx += nth) {
    const int i = idx / km, j = idx - i * km;
    if (j <= i) Lp[tri(i) + j] = load_r(i, j);
  }
  for (int idx = tid; idx < km * M; idx += nth) {
    const int i = idx / M, c = idx - i * M;
    W[c * km + i] = cd_conj(load_p(i, c));
  }
  if (tid == 0) s_fail = 0;
  __syncthreads();
  if (a.debug_rp != nullptr) {  // test hook: expose the assembled Gram
    cdbl* o = a.debug_rp + (long long)f * (km * km + km * M);
    for (int idx = tid; idx < km * km; idx += nth) {
      const int i = idx / km, j = idx - i * km;
      o[idx] = j <= i ? Lp[tri(i) + j] : cd_conj(Lp[tri(j) + i]);
    }
    for (int idx = tid; idx < km * M; idx += nth) o[km * km + idx] = cd_conj(W[(idx % M) * km + idx / M]);
    return;
  }
  if (tid == 0) {  // regularize (numerics.hpp:41-49)
    double tr = 0.0;
    for (int i = 0; i < km; ++i) tr += Lp[tri(i) + i].re;
    double scale = tr / (double)km;
    if (!(scale > 0.0)) scale = 1.0;
    s_tr = a.regularization * scale;
  }
  __syncthreads();
  for (int i = tid; i < km; i += nth) Lp[tri(i) + i].re += s_tr;
  __syncthreads();

  // ---- blocked right-looking Cholesky of [R ; W]: A = L L^H, W <- W L^-H. A pivot <= 0 fails (numerics.hpp:88).
  for (int kb = 0; kb < km; kb += kPB) {
    const int pb = min(kPB, km - kb);
    if (warp == 0) {
      // 1. factor the diagonal block in place, then replace it by its inverse
      bool ok = true;
      for (int k = 0; k < pb; ++k) {
        cdbl* rowk = Lp + tri(kb + k) + kb;
        const double d = rowk[k].re;
        if (!(d > 0.0)) {
          ok = false;
          break;  // warp-uniform
        }
        const double inv = rsqrt(d), sq = d * inv;
        __syncwarp();
        if (lane == 0) rowk[k] = cd_make(sq, 0.0);
        if (lane > k && lane < pb) {
          cdbl* e = Lp + tri(kb + lane) + kb + k;
          *e = cd_scale(*e, inv);
        }
        __syncwarp();
        const int r = pb - 1 - k;
        if (lane < r * (r + 1) / 2) {
          int ii = 0;
          while ((ii + 1) * (ii + 2) / 2 <= lane) ++ii;
          const int i = k + 1 + ii, jj = k + 1 + (lane - ii * (ii + 1) / 2);
          cdbl* e = Lp + tri(kb + i) + kb + jj;
          *e = cd_sub(*e, cd_mulc(Lp[tri(kb + i) + kb + k], Lp[tri(kb + jj) + kb + k]));
        }
        __syncwarp();
      }
      if (!ok) {
        if (lane == 0) s_fail = 1;
      } else {
        if (lane < pb) {  // column `lane` of L11^-1 by forward substitution
          const int s0 = lane;
          for (int r = 0; r < pb; ++r) {
            cdbl v = cd_make(0.0, 0.0);
            if (r == s0) {
              v = cd_make(1.0 / Lp[tri(kb + r) + kb + r].re, 0.0);
            } else if (r > s0) {
              cdbl sacc = cd_make(0.0, 0.0);
              for (int q = s0; q < r; ++q) sacc = cd_add(sacc, cd_mul(Lp[tri(kb + r) + kb + q], s_linv[q * kPB + s0]));
              v = cd_scale(sacc, -1.0 / Lp[tri(kb + r) + kb + r].re);
            }
            s_linv[r * kPB + s0] = v;
          }
        }
        __syncwarp();
        for (int e = lane; e < pb * pb; e += 32) {
          const int r = e / pb, c = e - r * pb;
          if (c <= r) Lp[tri(kb + r) + kb + c] = s_linv[r * kPB + c];
        }
      }
    }
    __syncthreads();
    if (s_fail) break;
    const int r0 = kb + pb;        // first row below the panel
    const int nbelow = km - r0;    // matrix rows below; the M rows of W follow
    // 2. panel: row x solves x L11^H = a, i.e. x[c] = sum_{q <= c} a[q] conj(Linv[c][q])
    for (int t = tid; t < nbelow + M; t += nth) {
      cdbl* row = t < nbelow ? Lp + tri(r0 + t) + kb : W + (t - nbelow) * km + kb;
      cdbl av[kPB], x[kPB];
#pragma unroll
      for (int q = 0; q < kPB; ++q) av[q] = q < pb ? row[q] : cd_make(0.0, 0.0);
#pragma unroll
      for (int c = 0; c < kPB; ++c) {
        cdbl sacc = cd_make(0.0, 0.0);
        if (c < pb) {
          const cdbl* li = Lp + tri(kb + c) + kb;
#pragma unroll
          for (int q = 0; q < kPB; ++q)
            if (q <= c) sacc = cd_add(sacc, cd_mulc(av[q], li[q]));
        }
        x[c] = sacc;
      }
#pragma unroll
      for (int c = 0; c < kPB; ++c)
        if (c < pb) row[c] = x[c];
    }
    __syncthreads();
    // 3. trailing update: A22 -= L21 L21^H (lower triangle), W2 -= W1 L21^H. Thread grid 8 x 16 over (row, col);
    //    a thread takes two rows at a time so that every panel row it reads from shared memory feeds two
    //    products (the loop is bound by those 16-byte loads, not by the FP64 pipe).
    {
      const int ty = tid >> 4, tx = tid & 15;
      const int nrows = nbelow + M;
      for (int t = ty; t < nrows; t += 2 * kSolveTY) {
        const int t1 = t + kSolveTY;
        const bool has1 = t1 < nrows;
        const bool isw0 = t >= nbelow, isw1 = has1 && t1 >= nbelow;
        cdbl* row0 = isw0 ? W + (t - nbelow) * km : Lp + tri(r0 + t);
        cdbl* row1 = !has1 ? row0 : isw1 ? W + (t1 - nbelow) * km : Lp + tri(r0 + t1);
        cdbl a0[kPB], a1[kPB];
#pragma unroll
        for (int c = 0; c < kPB; ++c) {
          a0[c] = c < pb ? row0[kb + c] : cd_make(0.0, 0.0);
          a1[c] = (has1 && c < pb) ? row1[kb + c] : cd_make(0.0, 0.0);
        }
        const int jmax0 = isw0 ? km - 1 : r0 + t;  // last column of each row to update
        const int jmax1 = !has1 ? -1 : isw1 ? km - 1 : r0 + t1;
        const int jmax = jmax0 > jmax1 ? jmax0 : jmax1;
        for (int jj = r0 + tx; jj <= jmax; jj += 16) {
          const cdbl* lj = Lp + tri(jj) + kb;
          cdbl s00 = cd_make(0.0, 0.0), s01 = s00, s10 = s00, s11 = s00;
#pragma unroll
          for (int c = 0; c < kPB; c += 2) {
            if (c < pb) {
              const cdbl l = lj[c];
              s00 = cd_add(s00, cd_mulc(a0[c], l));
              s10 = cd_add(s10, cd_mulc(a1[c], l));
            }
            if (c + 1 < pb) {
              const cdbl l = lj[c + 1];
              s01 = cd_add(s01, cd_mulc(a0[c + 1], l));
              s11 = cd_add(s11, cd_mulc(a1[c + 1], l));
            }
          }
          if (jj <= jmax0) row0[jj] = cd_sub(row0[jj], cd_add(s00, s01));
          if (jj <= jmax1) row1[jj] = cd_sub(row1[jj], cd_add(s10, s11));
        }
      }
    }
    __syncthreads();
  }
  float2* g = a.gconj + sd.g_wpe_off + (long long)f * km * M;
  if (s_fail) {
    // Eigenvalue-floor fallback (numerics.hpp:58-73, 90-93). Rare. The block takes one of the launch's global
    // scratch slots (it waits for one when all are busy: a holder never waits for anybody), assembles the
    // regularized system again from the Gram and solves it with the block-parallel Jacobi above.
    if (tid == 0) {
      int slot = -1;
      for (int attempt = 0; slot < 0; ++attempt) {
        const int cand = (f + attempt) % a.fb_slots;
        if (atomicCAS(a.fb_ticket + cand, 0, 1) == 0) slot = cand;
        else if (attempt % a.fb_slots == a.fb_slots - 1) __nanosleep(2000);
      }
      s_slot = slot;
    }
    __syncthreads();
    cdbl* Ag = a.fb_scratch + (size_t)s_slot * wpe_fallback_slot_elems(km, M);
    cdbl* work = Ag + (size_t)km * km;
    cdbl* work2 = work + (size_t)km * km;
    cdbl* Bg = work2 + (size_t)km * km;
    double* wv = reinterpret_cast<double*>(Bg + (size_t)km * M);
    for (int idx = tid; idx < km * km; idx += nth) {
      const int i = idx / km, j = idx - i * km;
      cdbl v = j <= i ? load_r(i, j) : cd_conj(load_r(j, i));
      if (i == j) v.re += s_tr;
      Ag[idx] = v;
    }
    for (int idx = tid; idx < km * M; idx += nth) Bg[idx] = load_p(idx / M, idx % M);
    __syncthreads();
    // the factorisation's shared memory is free: rotations and reduction scratch live there
    cdbl* rot = Lp;
    double* red = reinterpret_cast<double*>(rot + 4 * ((km + 2) / 2) + (km + 2) / 2 + 2);
    const bool ok = block_eig_floor_solve(Ag, km, Bg, M, work, work2, wv, rot, red, tid, nth);
    if (ok) {
      for (int idx = tid; idx < km * M; idx += nth) g[idx] = make_float2((float)Bg[idx].re, (float)(-Bg[idx].im));
    } else {
      if (tid == 0) atomicMin(a.status + blockIdx.y, make_status(5, f));
      for (int idx = tid; idx < km * M; idx += nth) g[idx] = make_float2(0.f, 0.f);
    }
    __syncthreads();
    if (tid == 0) {
      __threadfence();
      atomicExch(a.fb_ticket + s_slot, 0);
    }
    return;
  }
  // ---- backward: L^H X = Z with W = Z^H, i.e. V = X^H solves V L = W. Panels from the last to the first:
  // V1 = W1 L11^-1 (the stored inverse), then W[:, j] -= sum_q V1[:, q] L[kb + q][j] for the columns j < kb.
  for (int kb = ((km - 1) / kPB) * kPB; kb >= 0; kb -= kPB) {
    const int pb = min(kPB, km - kb);
    {
      const int c = tid / kPB, jq = tid % kPB;
      const bool act = c < M && jq < pb;
      cdbl v = cd_make(0.0, 0.0);
      if (act) {
        const cdbl* wr = W + c * km + kb;
        for (int q = jq; q < pb; ++q) v = cd_add(v, cd_mul(wr[q], Lp[tri(kb + q) + kb + jq]));
      }
      __syncwarp();  // a row of W belongs to one warp (kPB divides 32): all its readers are done
      if (act) W[c * km + kb + jq] = v;
    }
    __syncthreads();
    for (int idx = tid; idx < kb * M; idx += nth) {
      const int c = idx / kb, j = idx - c * kb;
      const cdbl* v1 = W + c * km + kb;
      cdbl s0 = cd_make(0.0, 0.0), s1 = cd_make(0.0, 0.0);
#pragma unroll
      for (int q = 0; q < kPB; q += 2) {
        if (q < pb) s0 = cd_add(s0, cd_mul(v1[q], Lp[tri(kb + q) + j]));
        if (q + 1 < pb) s1 = cd_add(s1, cd_mul(v1[q + 1], Lp[tri(kb + q + 1) + j]));
      }
      W[c * km + j] = cd_sub(W[c * km + j], cd_add(s0, s1));
    }
    __syncthreads();
  }
  // conj(G) rounded to cfloat (wpe.hpp:95-96): G = X, W = X^H, so conj(G)[i][c] = W[c][i]
  for (int idx = tid; idx < km * M; idx += nth) {
    const int i = idx / M, c = idx - i * M;
    const cdbl v = W[c * km + i];
    g[idx] = make_float2((float)v.re, (float)v.im);
  }
}

// ---------------------------------------------------------------------------
// Y_f = observed - history * conj(G) (wpe.hpp:95-96), two frames per thread, slab channel-major in shared
// memory, conj(G) broadcast from shared memory. The first version (one frame per thread, an 8-byte filter
// load per 4 FFMA) issued 88 % of its slots with only 58 % of them FMAs (ncu, profiles/ncu_full_r01.md);
// here a 16-byte load of two filter entries feeds 16 FFMA. Products and their order per output are unchanged.
// (Measured and rejected on B200: the packed fma.rn.f32x2 form -- FFMA2 issues no faster than two FFMA here
// and the operand packing costs extra moves: 6.9 ms against 6.0 ms per cfg2 step.)
// grid (512-frame tiles, F, segments), block 256.
// ---------------------------------------------------------------------------
namespace {
constexpr int kApplyFrames = 512;
}  // namespace

template <int M>
__global__ void __launch_bounds__(256) wpe_apply2_kernel(WpeArgs a) {
  extern __shared__ float4 smem_f4[];
  const SegDev sd = a.segs[blockIdx.z];
  if (!sd.wpe_active) return;
  const int tb = blockIdx.x * kApplyFrames;
  if (tb >= sd.T) return;
  const int f = blockIdx.y;
  const int taps = a.taps, km = taps * M, H = a.delay + taps - 1;
  const int SF = kApplyFrames + H, pitch = SF | 1;
  constexpr int MP = (M + 1) & ~1;                                       // filter row padded to whole float4s
  float2* gs = reinterpret_cast<float2*>(smem_f4);                       // km * MP
  float2* slab = gs + km * MP;                                           // M * pitch, channel-major
  const int tid = threadIdx.x;
  const int nfr = min(kApplyFrames, sd.T - tb);
  const float2* yf = a.yobs + sd.y_off + (long long)f * sd.T * M;
  for (int i = tid; i < (nfr + H) * M; i += 256) {
    const int fr = i / M, c = i - fr * M;
    const int t = tb - H + fr;
    slab[c * pitch + fr] = t >= 0 ? yf[(long long)t * M + c] : make_float2(0.f, 0.f);
  }
  const float2* g = a.gconj + sd.g_wpe_off + (long long)f * km * M;
  for (int i = tid; i < km * MP; i += 256) {
    const int r = i / MP, c2 = i - r * MP;
    gs[i] = c2 < M ? g[r * M + c2] : make_float2(0.f, 0.f);
  }
  __syncthreads();
  float2 acc0[M], acc1[M];
#pragma unroll
  for (int c = 0; c < M; ++c) acc0[c] = acc1[c] = make_float2(0.f, 0.f);
  const int f0 = min(tid, nfr - 1), f1 = min(tid + 256, nfr - 1);
  for (int u = 0; u < taps; ++u) {
#pragma unroll
    for (int c = 0; c < M; ++c) {
      const float2 v0 = slab[c * pitch + f0 + u], v1 = slab[c * pitch + f1 + u];
      const float4* gr = reinterpret_cast<const float4*>(gs + (u * M + c) * MP);
#pragma unroll
      for (int p = 0; p < MP / 2; ++p) {
        const float4 gg = gr[p];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int c2 = 2 * p + h;
          if (c2 < M) {
            const float gx = h ? gg.z : gg.x, gy = h ? gg.w : gg.y;
            acc0[c2].x = fmaf(v0.x, gx, acc0[c2].x);
            acc0[c2].x = fmaf(-v0.y, gy, acc0[c2].x);
            acc0[c2].y = fmaf(v0.x, gy, acc0[c2].y);
            acc0[c2].y = fmaf(v0.y, gx, acc0[c2].y);
            acc1[c2].x = fmaf(v1.x, gx, acc1[c2].x);
            acc1[c2].x = fmaf(-v1.y, gy, acc1[c2].x);
            acc1[c2].y = fmaf(v1.x, gy, acc1[c2].y);
            acc1[c2].y = fmaf(v1.y, gx, acc1[c2].y);
          }
        }
      }
    }
  }
  // observed - prediction, staged through shared memory for contiguous stores
  float2 res0[M], res1[M];
#pragma unroll
  for (int c = 0; c < M; ++c) {
    const float2 o0 = slab[c * pitch + f0 + H], o1 = slab[c * pitch + f1 + H];
    res0[c] = make_float2(o0.x - acc0[c].x, o0.y - acc0[c].y);
    res1[c] = make_float2(o1.x - acc1[c].x, o1.y - acc1[c].y);
  }
  __syncthreads();
  float2* stage = slab;  // 512 * M <= M * pitch
  if (tid < nfr) {
#pragma unroll
    for (int c = 0; c < M; ++c) stage[tid * M + c] = res0[c];
  }
  if (tid + 256 < nfr) {
#pragma unroll
    for (int c = 0; c < M; ++c) stage[(tid + 256) * M + c] = res1[c];
  }
  __syncthreads();
  float2* out = a.yout + sd.y_off + ((long long)f * sd.T + tb) * M;
  for (int i = tid; i < nfr * M; i += 256) out[i] = stage[i];
}

// ---------------------------------------------------------------------------
// launchers
// ---------------------------------------------------------------------------
int wpe_gram_cell_elems(int km, int M) { return gram_num_tiles(km, M) * kTileElems; }
int wpe_fallback_slot_elems_host(int km, int M) { return wpe_fallback_slot_elems(km, M); }

template <int M>
static cudaError_t launch_wpe_step_m(int step, const WpeArgs& a, int nseg, int F, int max_frames, int max_wchunks,
                                     cudaStream_t st) {
  const int km = a.taps * M, H = a.delay + a.taps - 1;
  if (step == 0) {
    dim3 grid((max_frames + 255) / 256, F, nseg);
    wpe_power_kernel<<<grid, 256, 0, st>>>(a);
  } else if (step == 1 && a.use_tc) {
    return launch_wpe_gram_tc(a, nseg, F, st);
  } else if (step == 1) {
    const int ngroups = (gram_num_tiles(km, M) + kGramWarps - 1) / kGramWarps;
    const size_t smem = 2 * (sizeof(float2) * (size_t)M * ((kGramTileFrames + H + 8) | 1) + sizeof(float) * kGramTileFrames);
    if (smem > 220 * 1024) return cudaErrorInvalidConfiguration;
    cudaError_t e = cudaFuncSetAttribute(wpe_gram_kernel<M>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    dim3 grid(ngroups * max_wchunks, F, nseg);
    wpe_gram_kernel<M><<<grid, kGramThreads, smem, st>>>(a);
  } else if (step == 2) {
    const size_t smem = sizeof(cdbl) * ((size_t)km * (km + 1) / 2 + (size_t)km * M + kPB * kPB);
    if (smem > 220 * 1024) return cudaErrorInvalidConfiguration;
    cudaError_t e = cudaFuncSetAttribute(wpe_solve2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    dim3 grid(F, nseg);
    wpe_solve2_kernel<<<grid, kSolveThreads, smem, st>>>(a);
  } else if (a.apply_tc) {
    return launch_wpe_apply_tc(a, nseg, F, st);
  } else {
    const size_t smem = sizeof(float2) * ((size_t)M * ((kApplyFrames + H) | 1) + (size_t)km * ((M + 1) & ~1));
    if (smem > 220 * 1024) return cudaErrorInvalidConfiguration;
    cudaError_t e = cudaFuncSetAttribute(wpe_apply2_kernel<M>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    dim3 grid((max_frames + kApplyFrames - 1) / kApplyFrames, F, nseg);
    wpe_apply2_kernel<M><<<grid, 256, smem, st>>>(a);
  }
  return cudaGetLastError();
}

/// step: 0 power, 1 gram, 2 solve, 3 apply
cudaError_t launch_wpe_step(int step, const WpeArgs& a, int nseg, int F, int max_frames, int max_wchunks,
                            cudaStream_t st) {
  switch (a.M) {
    case 1: return launch_wpe_step_m<1>(step, a, nseg, F, max_frames, max_wchunks, st);
    case 2: return launch_wpe_step_m<2>(step, a, nseg, F, max_frames, max_wchunks, st);
    case 3: return launch_wpe_step_m<3>(step, a, nseg, F, max_frames, max_wchunks, st);
    case 4: return launch_wpe_step_m<4>(step, a, nseg, F, max_frames, max_wchunks, st);
    case 5: return launch_wpe_step_m<5>(step, a, nseg, F, max_frames, max_wchunks, st);
    case 6: return launch_wpe_step_m<6>(step, a, nseg, F, max_frames, max_wchunks, st);
    case 7: return launch_wpe_step_m<7>(step, a, nseg, F, max_frames, max_wchunks, st);
    case 8: return launch_wpe_step_m<8>(step, a, nseg, F, max_frames, max_wchunks, st);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace gssb
