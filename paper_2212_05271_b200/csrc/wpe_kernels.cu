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
//   wpe_solve_kernel  FP64 Cholesky of the km x km system per (segment, bin)
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
// Solve R G = P per (segment, bin) in FP64 (wpe.hpp:90-94; numerics.hpp:32-49,
// 81-94). grid (F, segments), block 256. Right-looking Cholesky in shared
// memory, then forward / backward substitution of the M right-hand sides.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) wpe_solve_kernel(WpeArgs a) {
  extern __shared__ float4 smem_f4[];
  const SegDev sd = a.segs[blockIdx.y];
  if (!sd.wpe_active) return;
  const int f = blockIdx.x;
  const int M = a.M, km = a.taps * M, nb = gram_row_blocks(km), ntiles = gram_num_tiles(km, M);
  const int ld = km + 1;
  cdbl* A = reinterpret_cast<cdbl*>(smem_f4);  // km x ld
  cdbl* B = A + (size_t)km * ld;               // km x M
  double* diag0 = reinterpret_cast<double*>(B + (size_t)km * M);  // regularized diagonal, for the fallback
  __shared__ double s_tr;
  __shared__ int s_fail, s_slot;
  const int tid = threadIdx.x, nth = blockDim.x;
  const float2* tiles = a.gram + (sd.wcell_off + (long long)f * sd.wchunks) * ntiles * kTileElems;
  const long long chunk_stride = (long long)ntiles * kTileElems;

  if (a.use_tc) {
    // raw real accumulators of the tensor-core Gram (wpe_gram_tc.cu): D1 = S[0..128) S^T (NR columns),
    // D2 = S[NR-128..NR) S[128..NR)^T (N2 columns); G(a,b) by symmetry
    // operand rows: [Re a (KMP)] [Im a (KMP)] [Re y (8)] [Im y (8)], KMP = km rounded up to 8
    const int KMP = (km + 7) & ~7, NR = ((2 * KMP + 16 + 15) / 16) * 16, N2 = NR > 128 ? NR - 128 : 0, NCT = NR + N2;
    const float* raw = a.gram_raw + (sd.wcell_off + (long long)f) * (long long)(128 * NCT);
    auto G = [&](int x, int y) -> double {
      if (x < 128) return (double)raw[x * NCT + y];
      if (y < 128) return (double)raw[y * NCT + x];
      return (double)raw[(x - (NR - 128)) * NCT + NR + (y - 128)];
    };
    for (int idx = tid; idx < km * km; idx += nth) {
      const int i = idx / km, j = idx - i * km;
      if (j > i) continue;
      const double re = G(i, j) + G(KMP + i, KMP + j);
      const double im = i == j ? 0.0 : G(KMP + i, j) - G(i, KMP + j);
      A[i * ld + j] = cd_make(re, im);
      A[j * ld + i] = cd_make(re, -im);
    }
    for (int idx = tid; idx < km * M; idx += nth) {
      const int i = idx / M, c = idx - i * M;
      B[i * M + c] = cd_make(G(i, 2 * KMP + c) + G(KMP + i, 2 * KMP + 8 + c),
                             G(KMP + i, 2 * KMP + c) - G(i, 2 * KMP + 8 + c));
    }
  } else {
  // lower triangle of R (upper mirrored by hermitize) and P, summed over chunks in double
  for (int idx = tid; idx < km * km; idx += nth) {
    const int i = idx / km, j = idx - i * km;
    if (j > i) continue;
    const float2* p = tiles + (long long)gram_r_tile(i, j) * kTileElems + (i & 7) * kTC + j % kTC;
    double re = 0.0, im = 0.0;
    for (int c = 0; c < sd.wchunks; ++c) {
      const float2 v = p[c * chunk_stride];
      re += (double)v.x;
      im += (double)v.y;
    }
    // hermitize (numerics.hpp:32-38): both triangles come from the same sums
    if (i == j) im = 0.0;
    A[i * ld + j] = cd_make(re, im);
    A[j * ld + i] = cd_make(re, -im);
  }
  for (int idx = tid; idx < km * M; idx += nth) {
    const int i = idx / M, c = idx - i * M;
    const float2* p = tiles + (long long)gram_p_tile(i, c, nb, M) * kTileElems + (i & 7) * kTC + c % kTC;
    double re = 0.0, im = 0.0;
    for (int ch = 0; ch < sd.wchunks; ++ch) {
      const float2 v = p[ch * chunk_stride];
      re += (double)v.x;
      im += (double)v.y;
    }
    B[i * M + c] = cd_make(re, im);
  }
  }
  if (tid == 0) s_fail = 0;
  __syncthreads();
  if (a.debug_rp != nullptr) {  // test hook: expose the assembled Gram
    cdbl* o = a.debug_rp + (long long)f * (km * km + km * M);
    for (int idx = tid; idx < km * km; idx += nth) o[idx] = A[(idx / km) * ld + idx % km];
    for (int idx = tid; idx < km * M; idx += nth) o[km * km + idx] = B[idx];
    return;
  }
  if (tid == 0) {  // regularize (numerics.hpp:41-49)
    double tr = 0.0;
    for (int i = 0; i < km; ++i) tr += A[i * ld + i].re;
    double scale = tr / (double)km;
    if (!(scale > 0.0)) scale = 1.0;
    s_tr = a.regularization * scale;
  }
  __syncthreads();
  for (int i = tid; i < km; i += nth) {
    A[i * ld + i].re += s_tr;
    diag0[i] = A[i * ld + i].re;
  }
  __syncthreads();

  // Blocked right-looking Cholesky on the lower triangle (panels of PB columns: 3 barriers per panel
  // instead of 3 per column). A pivot <= 0 fails, Eigen LLT's criterion (numerics.hpp:88).
  constexpr int PB = 8;
  const int lane = tid & 31, warp = tid >> 5;
  for (int kb = 0; kb < km; kb += PB) {
    const int pb = min(PB, km - kb);
    if (warp == 0) {  // 1. factor the diagonal block in place
      cdbl* D = A + kb * ld + kb;
      bool ok = true;
      for (int k = 0; k < pb; ++k) {
        const double d = D[k * ld + k].re;
        if (!(d > 0.0)) {
          ok = false;
          break;  // warp-uniform
        }
        const double sq = sqrt(d), inv = 1.0 / sq;
        __syncwarp();
        if (lane == 0) D[k * ld + k] = cd_make(sq, 0.0);
        if (lane > k && lane < pb) D[lane * ld + k] = cd_scale(D[lane * ld + k], inv);
        __syncwarp();
        const int r = pb - 1 - k;
        if (lane < r * (r + 1) / 2) {
          int ii = 0;
          while ((ii + 1) * (ii + 2) / 2 <= lane) ++ii;
          const int i = k + 1 + ii, jj = k + 1 + (lane - ii * (ii + 1) / 2);
          D[i * ld + jj] = cd_sub(D[i * ld + jj], cd_mulc(D[i * ld + k], D[jj * ld + k]));
        }
        __syncwarp();
      }
      if (!ok && lane == 0) s_fail = 1;
    }
    __syncthreads();
    if (s_fail) break;
    const int r0 = kb + pb;  // first row below the panel
    // 2. panel: row i of L21 solves x L11^H = A[i][kb..kb+pb)
    for (int i = r0 + tid; i < km; i += nth) {
      cdbl x[PB];
#pragma unroll
      for (int c = 0; c < PB; ++c) {
        if (c < pb) {
          cdbl sacc = A[i * ld + kb + c];
#pragma unroll
          for (int q = 0; q < PB; ++q)
            if (q < c) sacc = cd_sub(sacc, cd_mulc(x[q], A[(kb + c) * ld + kb + q]));
          x[c] = cd_scale(sacc, 1.0 / A[(kb + c) * ld + kb + c].re);
          A[i * ld + kb + c] = x[c];
        }
      }
    }
    __syncthreads();
    // 3. trailing update: A22 -= L21 L21^H (lower triangle)
    for (int i = r0 + (tid >> 4); i < km; i += 16) {
      cdbl li[PB];
#pragma unroll
      for (int c = 0; c < PB; ++c) li[c] = c < pb ? A[i * ld + kb + c] : cd_make(0.0, 0.0);
      for (int jj = r0 + (tid & 15); jj <= i; jj += 16) {
        cdbl sacc = A[i * ld + jj];
#pragma unroll
        for (int c = 0; c < PB; ++c)
          if (c < pb) sacc = cd_sub(sacc, cd_mulc(li[c], A[jj * ld + kb + c]));
        A[i * ld + jj] = sacc;
      }
    }
    __syncthreads();
  }
  if (s_fail) {
    // Eigenvalue-floor fallback (numerics.hpp:58-73, 90-93). Rare: one thread, FP64 cyclic Jacobi in a global
    // scratch slot. The factorization only touched the lower triangle and the diagonal, so the regularized
    // matrix is rebuilt from the untouched upper triangle and the saved diagonal; P is still intact.
    float2* g = a.gconj + sd.g_wpe_off + (long long)f * km * M;
    if (tid == 0) {
      const int t = atomicAdd(a.fb_ticket, 1);
      s_slot = t < a.fb_slots ? t : -1;
    }
    __syncthreads();
    if (s_slot >= 0) {
      cdbl* Ag = a.fb_scratch + (size_t)s_slot * wpe_fallback_slot_elems(km, M);
      cdbl* work = Ag + (size_t)km * km;
      cdbl* work2 = work + (size_t)km * km;
      cdbl* Bg = work2 + (size_t)km * km;
      double* wv = reinterpret_cast<double*>(Bg + (size_t)km * M);
      for (int idx = tid; idx < km * km; idx += nth) {
        const int i = idx / km, j = idx - i * km;
        Ag[idx] = i == j ? cd_make(diag0[i], 0.0) : (j > i ? A[i * ld + j] : cd_conj(A[j * ld + i]));
      }
      for (int idx = tid; idx < km * M; idx += nth) Bg[idx] = B[idx];
      __threadfence_block();
      __syncthreads();
      if (tid == 0) s_fail = hermitian_solve(Ag, km, Bg, M, work, work2, wv) == kLinOk ? 2 : 3;
      __threadfence_block();
      __syncthreads();
      if (s_fail == 2) {
        for (int idx = tid; idx < km * M; idx += nth) g[idx] = make_float2((float)Bg[idx].re, (float)(-Bg[idx].im));
        return;
      }
    }
    if (tid == 0) atomicMin(a.status + blockIdx.y, make_status(5, f));
    for (int idx = tid; idx < km * M; idx += nth) g[idx] = make_float2(0.f, 0.f);
    return;
  }
  // forward: L Z = B, blocked like the factorization (thread c < M owns right-hand side c inside a panel)
  for (int kb = 0; kb < km; kb += PB) {
    const int pb = min(PB, km - kb);
    if (tid < M) {
      for (int k = 0; k < pb; ++k) {
        cdbl sacc = B[(kb + k) * M + tid];
        for (int q = 0; q < k; ++q) sacc = cd_sub(sacc, cd_mul(A[(kb + k) * ld + kb + q], B[(kb + q) * M + tid]));
        B[(kb + k) * M + tid] = cd_scale(sacc, 1.0 / A[(kb + k) * ld + kb + k].re);
      }
    }
    __syncthreads();
    const int r0 = kb + pb;
    for (int idx = tid; idx < (km - r0) * M; idx += nth) {
      const int i = r0 + idx / M, c = idx % M;
      cdbl sacc = B[i * M + c];
      for (int q = 0; q < pb; ++q) sacc = cd_sub(sacc, cd_mul(A[i * ld + kb + q], B[(kb + q) * M + c]));
      B[i * M + c] = sacc;
    }
    __syncthreads();
  }
  // backward: L^H X = Z
  for (int kb = ((km - 1) / PB) * PB; kb >= 0; kb -= PB) {
    const int pb = min(PB, km - kb);
    if (tid < M) {
      for (int k = pb - 1; k >= 0; --k) {
        cdbl sacc = B[(kb + k) * M + tid];
        for (int q = k + 1; q < pb; ++q) sacc = cd_sub(sacc, cd_cmul(A[(kb + q) * ld + kb + k], B[(kb + q) * M + tid]));
        B[(kb + k) * M + tid] = cd_scale(sacc, 1.0 / A[(kb + k) * ld + kb + k].re);
      }
    }
    __syncthreads();
    for (int idx = tid; idx < kb * M; idx += nth) {
      const int i = idx / M, c = idx % M;
      cdbl sacc = B[i * M + c];
      for (int q = 0; q < pb; ++q) sacc = cd_sub(sacc, cd_cmul(A[(kb + q) * ld + i], B[(kb + q) * M + c]));
      B[i * M + c] = sacc;
    }
    __syncthreads();
  }
  // conj(G) rounded to cfloat (wpe.hpp:95-96)
  float2* g = a.gconj + sd.g_wpe_off + (long long)f * km * M;
  for (int idx = tid; idx < km * M; idx += nth) g[idx] = make_float2((float)B[idx].re, (float)(-B[idx].im));
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
    const size_t smem = sizeof(cdbl) * ((size_t)km * (km + 1) + (size_t)km * M) + sizeof(double) * km;
    if (smem > 220 * 1024) return cudaErrorInvalidConfiguration;
    cudaError_t e = cudaFuncSetAttribute(wpe_solve_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    dim3 grid(F, nseg);
    wpe_solve_kernel<<<grid, 256, smem, st>>>(a);
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
