// stft_kernels.cu -- batched STFT analysis, beamformer application and fused
// inverse STFT / overlap-add.
//
// Reference semantics: stft.hpp:100-116 (reflect padding without edge repeat),
// :120-129 (frame geometry), :131-175 (analyze), :179-229 (synthesize),
// beamform.hpp:138-165 (apply).
//
// FFTs: one warp transforms one complex sequence of n points in shared memory
// (radix-2 decimation in time). Two real sequences ride in one complex
// transform (x1 + i x2), which halves the work of the real transforms.
#include <algorithm>

#include "kernels.h"

namespace gssb {

namespace {

constexpr int kStftThreads = 256;   // inverse transform
constexpr int kStftWarps = kStftThreads / 32;
constexpr int kAnaThreads = 512;    // forward transform: 16 warps keep more FP64 FFTs in flight per SM
constexpr int kAnaWarps = kAnaThreads / 32;

/// In-place radix-2 DIT over bit-reversed input; tw[k] = exp(-2 pi i k / n).
/// INVERSE conjugates the twiddles (unscaled inverse).
template <bool INVERSE, typename C2>
__device__ __forceinline__ void warp_fft(C2* buf, const C2* __restrict__ tw, int n, int log2n, int lane) {
  for (int s = 1; s <= log2n; ++s) {
    const int half = 1 << (s - 1);
    const int tstep = n >> s;
    for (int b = lane; b < (n >> 1); b += 32) {
      const int pos = b & (half - 1);
      const int i0 = ((b >> (s - 1)) << s) + pos;
      const int i1 = i0 + half;
      C2 w = tw[pos * tstep];
      if (INVERSE) w.y = -w.y;
      const C2 u = buf[i0], x = buf[i1];
      C2 v, r0, r1;
      v.x = x.x * w.x - x.y * w.y;
      v.y = x.x * w.y + x.y * w.x;
      r0.x = u.x + v.x;
      r0.y = u.y + v.y;
      r1.x = u.x - v.x;
      r1.y = u.y - v.y;
      buf[i0] = r0;
      buf[i1] = r1;
    }
    __syncwarp();
  }
}

/// Source index of padded position p (stft.hpp:100-116); N >= 2.
__device__ __forceinline__ long long reflect_index(long long idx, long long N) {
  if (idx < 0) return -idx;  // left pad: out[i] = x[pad - i]
  if (idx >= N) {
    long long src = N - 2 - (idx - N);
    while (src < 0 || src >= N) {
      if (src < 0) src = -src;
      if (src >= N) src = 2 * (N - 1) - src;
    }
    return src;
  }
  return idx;
}

}  // namespace

// ---------------------------------------------------------------------------
// analyze: grid (frame tiles, segments). A CTA transforms TB frames of all M
// channels, assembles the (f, frame, channel) tile in shared memory and writes
// runs of TB*M contiguous cfloats per bin (the (F,T,M) layout of stft.hpp:52-80).
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kAnaThreads) stft_kernel(StftArgs a) {
  // The forward transform runs in FP64 like the reference's (stft.hpp:158-170,
  // double FFT then a cast to cfloat): an FP32 FFT leaves an error proportional
  // to the frame's LOUDEST bin in every bin, which the EM iterations amplify in
  // the quiet bins.
  extern __shared__ float4 smem_f4[];
  double2* fftbuf = reinterpret_cast<double2*>(smem_f4);
  const int n = a.p.fft_size, log2n = a.p.log2n, F = a.p.F, M = a.M, TB = a.TB, NFW = a.fft_warps;
  float2* tile = reinterpret_cast<float2*>(fftbuf + NFW * n);
  double2* s_tw = reinterpret_cast<double2*>(tile + (size_t)F * ((TB * M) | 1) + (((size_t)F * ((TB * M) | 1)) & 1));
  const int run = TB * M;
  const int pitch = run | 1;
  const SegDev sd = a.segs[blockIdx.y];
  const int t0 = blockIdx.x * TB;
  if (t0 >= sd.T) return;
  for (int i = threadIdx.x; i < n / 2; i += kAnaThreads) s_tw[i] = a.tw_d[i];
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int pad = n / 2;
  const long long N = sd.N;
  double2* buf = fftbuf + (warp < NFW ? warp : 0) * n;
  const int npairs = (run + 1) / 2;
  for (int pair = warp; pair < npairs && warp < NFW; pair += NFW) {
    const int s1 = 2 * pair, s2 = s1 + 1;
    const int tl1 = s1 / M, m1 = s1 % M, tl2 = s2 / M, m2 = s2 % M;
    const bool v1 = t0 + tl1 < sd.T;
    const bool v2 = s2 < run && t0 + tl2 < sd.T;
    const float* x1 = a.audio + sd.audio_off + (long long)m1 * N;
    const float* x2 = a.audio + sd.audio_off + (long long)m2 * N;
    const long long b1 = (long long)(t0 + tl1) * a.p.shift - pad;
    const long long b2 = (long long)(t0 + tl2) * a.p.shift - pad;
    for (int i = lane; i < n; i += 32) {
      const double w = a.win_d[i];
      const double r1 = v1 ? (double)x1[reflect_index(b1 + i, N)] * w : 0.0;
      const double r2 = v2 ? (double)x2[reflect_index(b2 + i, N)] * w : 0.0;
      buf[__brev((unsigned)i) >> (32 - log2n)] = make_double2(r1, r2);
    }
    __syncwarp();
    warp_fft<false>(buf, s_tw, n, log2n, lane);
    for (int f = lane; f <= n / 2; f += 32) {
      const double2 zf = buf[f], zn = buf[(n - f) & (n - 1)];
      if (v1) tile[f * pitch + s1] = make_float2((float)(0.5 * (zf.x + zn.x)), (float)(0.5 * (zf.y - zn.y)));
      if (v2) tile[f * pitch + s2] = make_float2((float)(0.5 * (zf.y + zn.y)), (float)(0.5 * (zn.x - zf.x)));
    }
    __syncwarp();
  }
  __syncthreads();
  const int nvalid = min(TB, sd.T - t0) * M;
  float2* out = a.y + sd.y_off + (long long)t0 * M;
  for (int e = threadIdx.x; e < F * nvalid; e += kAnaThreads) {
    const int f = e / nvalid, r = e - f * nvalid;
    out[(long long)f * sd.T * M + r] = tile[f * pitch + r];
  }
}

// ---------------------------------------------------------------------------
// analyze, n = 512 (the BASELINE configurations): radix-8 x 8 x 8 in registers.
//
// 64 threads transform one complex sequence (two real frames, x1 + i x2): every thread holds 8 points, does
// an 8-point DFT in registers, and the three passes exchange data through 9 KB of shared memory per group
// (2 exchanges + the final natural-order write: 48 bytes of shared-memory traffic per point, against 360 for
// the radix-2 form above, which is shared-memory-bandwidth bound). FP64 like the reference (stft.hpp:158-170).
//
// Index algebra (W = exp(-2 pi i / 512), n = 64 n2 + 8 n1 + n0, k = k0 + 8 q0 + 64 q1):
//   pass 1, thread m = 8 n1 + n0 : B[k0]  = sum_n2 x[64 n2 + m] W8^(n2 k0),         times W^(m k0)
//   pass 2, thread (k0, n0)      : D[q0]  = sum_n1 B[8 n1 + n0][k0] W8^(n1 q0),      times W^(8 n0 q0)
//   pass 3, thread (k0, q0)      : X[k]   = sum_n0 D[k0][n0][q0] W8^(n0 q1)
// ---------------------------------------------------------------------------
namespace {

constexpr int kR8Threads = 256;            // 4 groups of 64
constexpr int kR8Groups = kR8Threads / 64;
constexpr int kR8Frames = 4;               // frames per CTA
constexpr int kR8Xch = 576;                // double2 per group: 8 x 72 (padded) >= 575 (natural order, padded)

__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__device__ __forceinline__ double2 mul_mi(double2 a) { return make_double2(a.y, -a.x); }  // a * (-i)

/// In-register forward 8-point DFT: v[k] <- sum_n v[n] exp(-2 pi i n k / 8).
__device__ __forceinline__ void dft8(double2 (&v)[8]) {
  constexpr double h = 0.70710678118654752440;
  const double2 a0 = cadd(v[0], v[4]), a4 = csub(v[0], v[4]);
  const double2 a1 = cadd(v[1], v[5]), t5 = csub(v[1], v[5]);
  const double2 a2 = cadd(v[2], v[6]), a6 = mul_mi(csub(v[2], v[6]));
  const double2 a3 = cadd(v[3], v[7]), t7 = csub(v[3], v[7]);
  const double2 a5 = make_double2((t5.x + t5.y) * h, (t5.y - t5.x) * h);    // * W8
  const double2 a7 = make_double2((t7.y - t7.x) * h, -(t7.x + t7.y) * h);   // * W8^3
  const double2 b0 = cadd(a0, a2), b2 = csub(a0, a2), b1 = cadd(a1, a3), b3 = mul_mi(csub(a1, a3));
  const double2 b4 = cadd(a4, a6), b6 = csub(a4, a6), b5 = cadd(a5, a7), b7 = mul_mi(csub(a5, a7));
  v[0] = cadd(b0, b1);
  v[4] = csub(b0, b1);
  v[2] = cadd(b2, b3);
  v[6] = csub(b2, b3);
  v[1] = cadd(b4, b5);
  v[5] = csub(b4, b5);
  v[3] = cadd(b6, b7);
  v[7] = csub(b6, b7);
}

/// v[k] *= w^k, k = 1..7 (powers by recurrence; FP64, far below the final cast to float).
__device__ __forceinline__ void twiddle8(double2 (&v)[8], double2 w) {
  double2 p = w;
#pragma unroll
  for (int k = 1; k < 8; ++k) {
    v[k] = cmul(v[k], p);
    if (k < 7) p = cmul(p, w);
  }
}

__device__ __forceinline__ void group_sync(int group) {
  asm volatile("bar.sync %0, 64;" ::"r"(group + 1) : "memory");
}

}  // namespace

__global__ void __launch_bounds__(kR8Threads, 2) stft512_kernel(StftArgs a) {
  extern __shared__ float4 smem_f4[];
  constexpr int n = 512, F = 257, pad = 256;
  const int M = a.M;
  const int run = kR8Frames * M, pitch = run | 1;
  double2* xch = reinterpret_cast<double2*>(smem_f4);                       // [groups][kR8Xch]
  double* s_win = reinterpret_cast<double*>(xch + kR8Groups * kR8Xch);      // [512]
  float2* tile = reinterpret_cast<float2*>(s_win + n);                      // [F][pitch]
  const SegDev sd = a.segs[blockIdx.y];
  const int t0 = blockIdx.x * kR8Frames;
  if (t0 >= sd.T) return;
  for (int i = threadIdx.x; i < n; i += kR8Threads) s_win[i] = a.win_d[i];
  __syncthreads();
  const int group = threadIdx.x >> 6, j = threadIdx.x & 63;
  const int hi = j >> 3, lo = j & 7;  // pass 2: (k0, n0); pass 3: (k0, q0)
  const double2 w1 = a.tw_d[j];       // W^m, m = j
  const double2 w2 = a.tw_d[8 * lo];  // W^(8 n0)
  double2* xg = xch + group * kR8Xch;
  const long long N = sd.N;
  const int npairs = (run + 1) / 2;
  for (int pair = group; pair < npairs; pair += kR8Groups) {
    const int s1 = 2 * pair, s2 = s1 + 1;
    const int tl1 = s1 / M, m1 = s1 % M, tl2 = s2 / M, m2 = s2 % M;
    const bool v1 = t0 + tl1 < sd.T;
    const bool v2 = s2 < run && t0 + tl2 < sd.T;
    const float* x1 = a.audio + sd.audio_off + (long long)m1 * N;
    const float* x2 = a.audio + sd.audio_off + (long long)m2 * N;
    const long long b1 = (long long)(t0 + tl1) * a.p.shift - pad;
    const long long b2 = (long long)(t0 + tl2) * a.p.shift - pad;
    // all 16 samples of this thread are fetched before any is used; frames that do not touch the signal's
    // ends (all but a handful per segment) skip the reflection arithmetic (group-uniform branches)
    float r1[8], r2[8];
    if (!v1) {
#pragma unroll
      for (int n2 = 0; n2 < 8; ++n2) r1[n2] = 0.f;
    } else if (b1 >= 0 && b1 + n <= N) {
      const float* q = x1 + b1 + j;
#pragma unroll
      for (int n2 = 0; n2 < 8; ++n2) r1[n2] = q[64 * n2];
    } else {
#pragma unroll
      for (int n2 = 0; n2 < 8; ++n2) r1[n2] = x1[reflect_index(b1 + 64 * n2 + j, N)];
    }
    if (!v2) {
#pragma unroll
      for (int n2 = 0; n2 < 8; ++n2) r2[n2] = 0.f;
    } else if (b2 >= 0 && b2 + n <= N) {
      const float* q = x2 + b2 + j;
#pragma unroll
      for (int n2 = 0; n2 < 8; ++n2) r2[n2] = q[64 * n2];
    } else {
#pragma unroll
      for (int n2 = 0; n2 < 8; ++n2) r2[n2] = x2[reflect_index(b2 + 64 * n2 + j, N)];
    }
    double2 v[8];
#pragma unroll
    for (int n2 = 0; n2 < 8; ++n2) {
      const double w = s_win[64 * n2 + j];
      v[n2] = make_double2((double)r1[n2] * w, (double)r2[n2] * w);
    }
    dft8(v);
    twiddle8(v, w1);
#pragma unroll
    for (int k0 = 0; k0 < 8; ++k0) xg[k0 * 72 + j] = v[k0];
    group_sync(group);
#pragma unroll
    for (int n1 = 0; n1 < 8; ++n1) v[n1] = xg[hi * 72 + 8 * n1 + lo];
    dft8(v);
    twiddle8(v, w2);
    group_sync(group);  // every thread has read its pass-2 inputs
#pragma unroll
    for (int q0 = 0; q0 < 8; ++q0) xg[hi * 72 + q0 * 9 + lo] = v[q0];
    group_sync(group);
#pragma unroll
    for (int n0 = 0; n0 < 8; ++n0) v[n0] = xg[hi * 72 + lo * 9 + n0];
    dft8(v);
    group_sync(group);
    // natural order, padded by one slot per 8 (conflict-free): Z[k] at k + k / 8, k = k0 + 8 q0 + 64 q1
#pragma unroll
    for (int q1 = 0; q1 < 8; ++q1) xg[hi + 9 * lo + 72 * q1] = v[q1];
    group_sync(group);
    // split the two real transforms (X1 = (Z[f] + conj Z[n-f]) / 2, X2 = (Z[f] - conj Z[n-f]) / 2i)
    for (int f = j; f < F; f += 64) {
      const int fn = (n - f) & (n - 1);
      const double2 zf = xg[f + (f >> 3)], zn = xg[fn + (fn >> 3)];
      if (v1) tile[f * pitch + s1] = make_float2((float)(0.5 * (zf.x + zn.x)), (float)(0.5 * (zf.y - zn.y)));
      if (v2) tile[f * pitch + s2] = make_float2((float)(0.5 * (zf.y + zn.y)), (float)(0.5 * (zn.x - zf.x)));
    }
    group_sync(group);  // the exchange buffer is rewritten by the next pair
  }
  __syncthreads();
  const int nvalid = min(kR8Frames, sd.T - t0) * M;
  float2* out = a.y + sd.y_off + (long long)t0 * M;
  for (int e = threadIdx.x; e < F * nvalid; e += kR8Threads) {
    const int f = e / nvalid, r = e - f * nvalid;
    out[(long long)f * sd.T * M + r] = tile[f * pitch + r];
  }
}

// ---------------------------------------------------------------------------
// apply: X(t,f) = sum_c y(f,t,c) * conj(h(f,c)) (beamform.hpp:157-163), written
// frame-major so the inverse transform reads each frame's bins contiguously.
// grid (frame tiles of 32, bin tiles of 32, segments), block 32 x 8.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) beamform_apply_kernel(ApplyArgs a) {
  __shared__ float2 tile[32][33];
  const SegDev sd = a.segs[blockIdx.z];
  const int t0 = blockIdx.x * 32, f0 = blockIdx.y * 32;
  if (t0 >= sd.T) return;
  const int tx = threadIdx.x, ty = threadIdx.y;
  const int M = a.M, F = a.F;
  const int t = t0 + tx;
  for (int fy = ty; fy < 32; fy += 8) {
    const int f = f0 + fy;
    float2 s = make_float2(0.f, 0.f);
    if (f < F && t < sd.T) {
      const float2* y = a.y + sd.y_off + ((long long)f * sd.T + t) * M;
      const float2* hc = a.hconj + (sd.f_off + f) * (long long)M;
      for (int c = 0; c < M; ++c) {
        const float2 v = y[c], h = hc[c];
        // complex<float> multiply-accumulate, as Eigen's cfloat GEMV does
        s.x += v.x * h.x - v.y * h.y;
        s.y += v.x * h.y + v.y * h.x;
      }
    }
    tile[fy][tx] = s;
    if (!a.frame_major && f < F && t < sd.T) a.x[sd.x_off + (long long)f * sd.T + t] = s;
  }
  if (!a.frame_major) return;
  __syncthreads();
  for (int ty2 = ty; ty2 < 32; ty2 += 8) {
    const int tt = t0 + ty2, f = f0 + tx;
    if (tt < sd.T && f < F) a.x[sd.x_off + (long long)tt * F + f] = tile[tx][ty2];
  }
}

// ---------------------------------------------------------------------------
// synthesize: inverse real FFT (scaled 1/n), window, overlap-add, divide by the
// window-power sum, trim the padding (stft.hpp:196-227). grid (hop blocks,
// segments); a CTA produces HB hops of output and transforms the HB+R-1 frames
// that overlap them, so the overlap-add is a gather (no atomics, fixed order).
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kStftThreads) istft_kernel(IstftArgs a) {
  extern __shared__ float4 smem_f4[];
  float2* fftbuf = reinterpret_cast<float2*>(smem_f4);
  const int n = a.p.fft_size, log2n = a.p.log2n, F = a.p.F, shift = a.p.shift, HB = a.HB;
  float* frames = reinterpret_cast<float*>(fftbuf + kStftWarps * n);
  const SegDev sd = a.segs[blockIdx.y];
  const long long out_len = sd.N;
  const int pad = n / 2, R = n / shift;
  const long long p_lo = (long long)pad + (long long)blockIdx.x * HB * shift;
  if (p_lo - pad >= out_len) return;
  const long long h_lo = p_lo / shift;
  const long long t_first = h_lo - R + 1;
  const int NF = HB + R - 1;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  float2* buf = fftbuf + warp * n;
  const float inv_n = 1.0f / (float)n;
  const float2* X = a.x + sd.x_off;
  for (int pair = warp; pair < (NF + 1) / 2; pair += kStftWarps) {
    const int la = 2 * pair, lb = la + 1;
    const long long ta = t_first + la, tb = t_first + lb;
    const bool va = ta >= 0 && ta < sd.T;
    const bool vb = lb < NF && tb >= 0 && tb < sd.T;
    if (va || vb) {
      for (int k = lane; k <= n / 2; k += 32) {
        const float2 xa = va ? X[ta * F + k] : make_float2(0.f, 0.f);
        const float2 xb = vb ? X[tb * F + k] : make_float2(0.f, 0.f);
        if (k == 0 || k == n / 2) {
          // imaginary parts of DC / Nyquist are ignored by the real inverse
          buf[__brev((unsigned)k) >> (32 - log2n)] = make_float2(xa.x, xb.x);
        } else {
          buf[__brev((unsigned)k) >> (32 - log2n)] = make_float2(xa.x - xb.y, xa.y + xb.x);
          buf[__brev((unsigned)(n - k)) >> (32 - log2n)] = make_float2(xa.x + xb.y, xb.x - xa.y);
        }
      }
      __syncwarp();
      warp_fft<true>(buf, a.tw, n, log2n, lane);
    }
    for (int i = lane; i < n; i += 32) {
      const float w = a.win[i] * inv_n;
      const float2 z = (va || vb) ? buf[i] : make_float2(0.f, 0.f);
      frames[la * n + i] = va ? z.x * w : 0.f;
      if (lb < NF) frames[lb * n + i] = vb ? z.y * w : 0.f;
    }
    __syncwarp();
  }
  __syncthreads();
  float* out = a.wave + sd.wave_off;
  for (int j = threadIdx.x; j < HB * shift; j += kStftThreads) {
    const long long p = p_lo + j;
    const long long i = p - pad;
    if (i >= out_len) break;
    const long long h = p / shift;
    float acc = 0.f, ws = 0.f;
    for (int r = R - 1; r >= 0; --r) {  // ascending frame index, as the reference adds them
      const long long t = h - r;
      if (t < 0 || t >= sd.T) continue;
      const int off = (int)(p - t * shift);
      const float w = a.win[off];
      acc += frames[(int)(t - t_first) * n + off];
      ws = fmaf(w, w, ws);
    }
    out[i] = ws > 1e-8f ? acc / ws : 0.f;
  }
}

// ---------------------------------------------------------------------------
// synthesize, n = 512: the radix-8 x 8 x 8 register transform of stft512_kernel run backwards (conjugated
// twiddles, FP32 like istft_kernel), 64 threads per complex transform (two frames ride in one: x_a + i x_b).
// Overlap-add, window-power normalisation and trimming are istft_kernel's.
// ---------------------------------------------------------------------------
namespace {

__device__ __forceinline__ float2 caddf(float2 a, float2 b) { return make_float2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ float2 csubf(float2 a, float2 b) { return make_float2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ float2 cmulf(float2 a, float2 b) {
  return make_float2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__device__ __forceinline__ float2 mul_pi(float2 a) { return make_float2(-a.y, a.x); }  // a * (+i)

/// In-register inverse (unscaled) 8-point DFT: v[k] <- sum_n v[n] exp(+2 pi i n k / 8).
__device__ __forceinline__ void idft8f(float2 (&v)[8]) {
  constexpr float h = 0.70710678118654752440f;
  const float2 a0 = caddf(v[0], v[4]), a4 = csubf(v[0], v[4]);
  const float2 a1 = caddf(v[1], v[5]), t5 = csubf(v[1], v[5]);
  const float2 a2 = caddf(v[2], v[6]), a6 = mul_pi(csubf(v[2], v[6]));
  const float2 a3 = caddf(v[3], v[7]), t7 = csubf(v[3], v[7]);
  const float2 a5 = make_float2((t5.x - t5.y) * h, (t5.x + t5.y) * h);     // * conj(W8)
  const float2 a7 = make_float2(-(t7.x + t7.y) * h, (t7.x - t7.y) * h);    // * conj(W8)^3
  const float2 b0 = caddf(a0, a2), b2 = csubf(a0, a2), b1 = caddf(a1, a3), b3 = mul_pi(csubf(a1, a3));
  const float2 b4 = caddf(a4, a6), b6 = csubf(a4, a6), b5 = caddf(a5, a7), b7 = mul_pi(csubf(a5, a7));
  v[0] = caddf(b0, b1);
  v[4] = csubf(b0, b1);
  v[2] = caddf(b2, b3);
  v[6] = csubf(b2, b3);
  v[1] = caddf(b4, b5);
  v[5] = csubf(b4, b5);
  v[3] = caddf(b6, b7);
  v[7] = csubf(b6, b7);
}

__device__ __forceinline__ void twiddle8f(float2 (&v)[8], float2 w) {
  float2 p = w;
#pragma unroll
  for (int k = 1; k < 8; ++k) {
    v[k] = cmulf(v[k], p);
    if (k < 7) p = cmulf(p, w);
  }
}

}  // namespace

__global__ void __launch_bounds__(kR8Threads) istft512_kernel(IstftArgs a) {
  extern __shared__ float4 smem_f4[];
  constexpr int n = 512, F = 257, pad = 256;
  const int shift = a.p.shift, HB = a.HB;
  float2* xch = reinterpret_cast<float2*>(smem_f4);                 // [groups][kR8Xch]
  float* frames = reinterpret_cast<float*>(xch + kR8Groups * kR8Xch);
  const SegDev sd = a.segs[blockIdx.y];
  const long long out_len = sd.N;
  const int R = n / shift;
  const long long p_lo = (long long)pad + (long long)blockIdx.x * HB * shift;
  if (p_lo - pad >= out_len) return;
  const long long h_lo = p_lo / shift;
  const long long t_first = h_lo - R + 1;
  const int NF = HB + R - 1;
  const int group = threadIdx.x >> 6, j = threadIdx.x & 63;
  const int hi = j >> 3, lo = j & 7;
  const float2 tw1 = a.tw[j], tw2 = a.tw[8 * lo];                    // exp(-2 pi i k / n): conjugated below
  const float2 w1 = make_float2(tw1.x, -tw1.y), w2 = make_float2(tw2.x, -tw2.y);
  float2* xg = xch + group * kR8Xch;
  const float inv_n = 1.0f / (float)n;
  const float2* X = a.x + sd.x_off;
  for (int pair = group; pair < (NF + 1) / 2; pair += kR8Groups) {
    const int la = 2 * pair, lb = la + 1;
    const long long ta = t_first + la, tb = t_first + lb;
    const bool va = ta >= 0 && ta < sd.T;
    const bool vb = lb < NF && tb >= 0 && tb < sd.T;
    if (va || vb) {  // group-uniform
      float2 v[8];
#pragma unroll
      for (int n2 = 0; n2 < 8; ++n2) {
        const int k = 64 * n2 + j;           // spectrum index of z = x_a + i x_b
        const int kk = k <= n / 2 ? k : n - k;
        const float2 xa = va ? X[ta * F + kk] : make_float2(0.f, 0.f);
        const float2 xb = vb ? X[tb * F + kk] : make_float2(0.f, 0.f);
        if (k == 0 || k == n / 2) v[n2] = make_float2(xa.x, xb.x);  // imaginary parts of DC / Nyquist are ignored
        else if (k < n / 2) v[n2] = make_float2(xa.x - xb.y, xa.y + xb.x);
        else v[n2] = make_float2(xa.x + xb.y, xb.x - xa.y);          // conj(x_a[n-k]) + i conj(x_b[n-k])
      }
      idft8f(v);
      twiddle8f(v, w1);
#pragma unroll
      for (int k0 = 0; k0 < 8; ++k0) xg[k0 * 72 + j] = v[k0];
      group_sync(group);
#pragma unroll
      for (int n1 = 0; n1 < 8; ++n1) v[n1] = xg[hi * 72 + 8 * n1 + lo];
      idft8f(v);
      twiddle8f(v, w2);
      group_sync(group);
#pragma unroll
      for (int q0 = 0; q0 < 8; ++q0) xg[hi * 72 + q0 * 9 + lo] = v[q0];
      group_sync(group);
#pragma unroll
      for (int n0 = 0; n0 < 8; ++n0) v[n0] = xg[hi * 72 + lo * 9 + n0];
      idft8f(v);
      // sample index i = hi + 8 lo + 64 q1: window, 1/n, split the two frames
#pragma unroll
      for (int q1 = 0; q1 < 8; ++q1) {
        const int i = hi + 8 * lo + 64 * q1;
        const float w = a.win[i] * inv_n;
        frames[la * n + i] = va ? v[q1].x * w : 0.f;
        if (lb < NF) frames[lb * n + i] = vb ? v[q1].y * w : 0.f;
      }
      group_sync(group);  // the exchange buffer is rewritten by the next pair
    } else {
      for (int i = j; i < n; i += 64) {
        frames[la * n + i] = 0.f;
        if (lb < NF) frames[lb * n + i] = 0.f;
      }
    }
  }
  __syncthreads();
  float* out = a.wave + sd.wave_off;
  for (int jj = threadIdx.x; jj < HB * shift; jj += kR8Threads) {
    const long long p = p_lo + jj;
    const long long i = p - pad;
    if (i >= out_len) break;
    const long long h = p / shift;
    float acc = 0.f, ws = 0.f;
    for (int r = R - 1; r >= 0; --r) {  // ascending frame index, as the reference adds them
      const long long t = h - r;
      if (t < 0 || t >= sd.T) continue;
      const int off = (int)(p - t * shift);
      const float w = a.win[off];
      acc += frames[(int)(t - t_first) * n + off];
      ws = fmaf(w, w, ws);
    }
    out[i] = ws > 1e-8f ? acc / ws : 0.f;
  }
}

// ---------------------------------------------------------------------------
// launchers
// ---------------------------------------------------------------------------
static int stft_frames_per_cta(int n) { return n >= 2048 ? 1 : 2048 / n; }
static int stft_fft_warps(int n) { return std::max(1, std::min(kAnaWarps, 8192 / n)); }

cudaError_t launch_stft(const StftArgs& args_in, int nseg, int max_frames, cudaStream_t st) {
  StftArgs a = args_in;
  if (a.p.fft_size == 512) {
    const size_t tile = (size_t)a.p.F * ((kR8Frames * a.M) | 1);
    const size_t smem = sizeof(double2) * kR8Groups * kR8Xch + sizeof(double) * 512 + sizeof(float2) * tile;
    cudaError_t e = cudaFuncSetAttribute(stft512_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    dim3 grid((max_frames + kR8Frames - 1) / kR8Frames, nseg);
    stft512_kernel<<<grid, kR8Threads, smem, st>>>(a);
    return cudaGetLastError();
  }
  a.TB = stft_frames_per_cta(a.p.fft_size);
  a.fft_warps = stft_fft_warps(a.p.fft_size);
  const size_t tile_elems = (size_t)a.p.F * ((a.TB * a.M) | 1);
  const size_t smem = sizeof(double2) * ((size_t)a.fft_warps * a.p.fft_size + a.p.fft_size / 2) +
                      sizeof(float2) * (tile_elems + (tile_elems & 1));
  if (smem > 220 * 1024) return cudaErrorInvalidConfiguration;
  cudaError_t e = cudaFuncSetAttribute(stft_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  dim3 grid((max_frames + a.TB - 1) / a.TB, nseg);
  stft_kernel<<<grid, kAnaThreads, smem, st>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_apply(const ApplyArgs& a, int nseg, int max_frames, cudaStream_t st) {
  dim3 grid((max_frames + 31) / 32, (a.F + 31) / 32, nseg);
  beamform_apply_kernel<<<grid, dim3(32, 8), 0, st>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_istft(const IstftArgs& args_in, int nseg, long long max_out_len, cudaStream_t st) {
  IstftArgs a = args_in;
  a.HB = 16;
  const int R = a.p.fft_size / a.p.shift;
  if (a.p.fft_size == 512) {
    const size_t smem = sizeof(float2) * kR8Groups * kR8Xch + sizeof(float) * (size_t)(a.HB + R - 1) * 512;
    cudaError_t e = cudaFuncSetAttribute(istft512_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    const long long per = (long long)a.HB * a.p.shift;
    dim3 grid((unsigned)((max_out_len + per - 1) / per), nseg);
    if (grid.x == 0) return cudaSuccess;
    istft512_kernel<<<grid, kR8Threads, smem, st>>>(a);
    return cudaGetLastError();
  }
  const size_t smem = sizeof(float2) * (size_t)kStftWarps * a.p.fft_size +
                      sizeof(float) * (size_t)(a.HB + R - 1) * a.p.fft_size;
  if (smem > 220 * 1024) return cudaErrorInvalidConfiguration;
  cudaError_t e = cudaFuncSetAttribute(istft_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  const long long per = (long long)a.HB * a.p.shift;
  dim3 grid((unsigned)((max_out_len + per - 1) / per), nseg);
  if (grid.x == 0) return cudaSuccess;
  istft_kernel<<<grid, kStftThreads, smem, st>>>(a);
  return cudaGetLastError();
}

}  // namespace gssb
