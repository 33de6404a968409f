// wpe_apply_tc.cu -- the WPE prediction Y_f = observed - history * conj(G) (wpe.hpp:95-96) on the 5th-generation
// tensor cores: tcgen05.mma kind::tf32 with the 3xTF32 split (hi*hi + hi*lo + lo*hi), FP32 accumulator in
// tensor memory.
//
// Real formulation per (segment, bin). A frame's M complex channels are 2M consecutive floats of the bin's
// slab; padded to 16 they are one K = 16 slice. For tap u the GEMM operand A_u (frames x 16) is the slab
// shifted by u frames, so with the slab staged ONCE in the K-major core-matrix layout whose 8-row groups are
// contiguous (SBO = 128 bytes: row r of a K core sits at r * 16 bytes) the operand of tap u is the same
// buffer addressed from row u: the tap-stacked matrix (taps x larger) is never built, the shift is the
// descriptor's start address. B_u (16 x 16) carries conj(G) of tap u as the real 2x2 blocks of a complex
// product: columns 0..M-1 produce the real parts of the M outputs, columns 8..8+M-1 the imaginary parts.
//     D[t][n] = sum_u sum_kappa A[t + u][kappa] B_u[kappa][n]          (2 k-steps of 8 per tap)
// The MMA streams its 128 x 8 A tile from shared memory every time (4 KB, 32 cycles of shared-memory
// bandwidth for N = 16 columns of work), so the three products of the split are issued as two MMAs per k-step:
// A_hi x [B_hi | B_lo] (N = 32) and A_lo x B_hi (N = 16), into three 16-column accumulators summed at the end.
//
// Block = (segment, bin), 160 threads: warp 0 issues the MMAs of a 128-frame tile; warps 1..4 stage the next
// tile's slab rows (hi / lo split), then subtract the finished tile's prediction from the observation and
// store it. Two staging buffers / accumulators; full / done mbarriers as in wpe_gram_tc.cu.
#include <cuda_fp16.h>

#include "kernels.h"

namespace gssb {

namespace {

constexpr int kTile = 128;                 // frames per MMA tile (the MMA's M)
constexpr int kAppThreads = 160;           // 1 issuer warp + 4 worker warps
constexpr int kKPad = 16;                  // K per tap: 2 M floats padded to 16
#ifndef GSS_APPLY_3BLOCK_FROM
#define GSS_APPLY_3BLOCK_FROM 8
#endif
constexpr int kNOut = 16;                  // N: [Re out (8) | Im out (8)]

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

/// K-major, no swizzle: 8-row groups SBO bytes apart, the two 16-byte K chunks of one MMA LBO bytes apart.
__device__ __forceinline__ uint64_t make_desc(uint32_t addr, uint32_t lbo_bytes, uint32_t sbo_bytes) {
  uint64_t d = 0;
  d |= (uint64_t)((addr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo_bytes >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo_bytes >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;  // descriptor version (Blackwell)
  return d;
}
/// kind::tf32, FP32 accumulate, both operands K-major, M = 128.
__device__ __forceinline__ uint32_t make_idesc(int n) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
}
__device__ __forceinline__ void mma_tf32(uint32_t tmem_d, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                         uint32_t accumulate) {
  asm volatile(
      "{\n\t"
      ".reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t"
      "}\n" ::"r"(tmem_d),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
/// Bounded wait: a protocol error traps (an error for the caller) instead of hanging the device.
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  const uint32_t addr = smem_u32(bar);
  for (int spin = 0; spin < (1 << 27); ++spin) {
    uint32_t ok;
    asm volatile(
        "{\n\t"
        ".reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t"
        "}\n"
        : "=r"(ok)
        : "r"(addr), "r"(parity)
        : "memory");
    if (ok) return;
  }
  __trap();
}
__device__ __forceinline__ void tc_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ float tf32_hi(float v) { return __uint_as_float(__float_as_uint(v) & 0xffffe000u); }

// Staged slab rows per tile: exactly the 128 frames and their H history rows. (Not rounded up to the 8-row core
// matrix: the MMA of tap u reads rows u .. u + 127, and the 1 KB this saves is what lets four blocks share an SM.)
__host__ __device__ inline int app_rows(int H) { return kTile + H; }
// Blocks per SM the register allocation aims at. Four hide more of a tile's load -> stage -> MMA -> store latency
// (M = 5: 3.32 -> 3.09 ms, M = 6: 3.39 -> 3.19 ms per 16-segment step); at M = 8 the serial MMA stream of the SM's one
// tensor pipe is what binds and the fourth block only adds contention (4.39 -> 4.76 ms, TF32 kind), so it keeps three.
__host__ __device__ constexpr int app_min_blocks(int M) { return M >= GSS_APPLY_3BLOCK_FROM ? 3 : 4; }

}  // namespace

template <int M>
__global__ void __launch_bounds__(kAppThreads, app_min_blocks(M)) wpe_apply_tc_kernel(WpeArgs a) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const SegDev sd = a.segs[blockIdx.y];
  if (!sd.wpe_active) return;
  const int f = blockIdx.x;
  const int taps = a.taps, km = taps * M, H = a.delay + taps - 1;
  const int NROWS = app_rows(H);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

  uint64_t* full = reinterpret_cast<uint64_t*>(smem_raw);              // [2] slab of a tile is staged
  uint64_t* done = full + 2;                                           // [2] MMAs of a tile are complete
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem_raw + 32);
  float* bop = reinterpret_cast<float*>(smem_raw + 128);               // [tap][kc 4][hi ng0 ng1, lo ng0 ng1][8 x 4]
  const int bop_words = taps * 4 * 2 * 32;                             // words of one of hi / lo
  float* aop = bop + 2 * bop_words;                                    // [stage 2][hi/lo][kc 4][NROWS][4]
  const int aop_words = 4 * NROWS * 4;

  if (tid == 0) {
    mbar_init(&full[0], 128);
    mbar_init(&full[1], 128);
    mbar_init(&done[0], 1);
    mbar_init(&done[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(128u)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  // conj(G) of this bin as the B operands (real 2x2 blocks of the complex product), hi / lo split
  {
    const float2* g = a.gconj + sd.g_wpe_off + (long long)f * km * M;
    for (int i = tid; i < taps * kKPad * kNOut; i += kAppThreads) {
      const int u = i / (kKPad * kNOut), r = i - u * (kKPad * kNOut), kappa = r / kNOut, n = r - kappa * kNOut;
      const int c = kappa >> 1, part = kappa & 1, c2 = n & 7, im_out = n >> 3;
      float v = 0.f;
      if (c < M && c2 < M) {
        const float2 gg = g[(u * M + c) * M + c2];
        v = part == 0 ? (im_out ? gg.y : gg.x) : (im_out ? gg.x : -gg.y);
      }
      const float hi = tf32_hi(v);
      const int word = ((u * 4 + (kappa >> 2)) * 4 + (n >> 3)) * 32 + (n & 7) * 4 + (kappa & 3);
      bop[word] = hi;            // n-groups 0, 1 of the (tap, K core): B_hi
      bop[word + 64] = v - hi;   // n-groups 2, 3: B_lo
    }
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem_base = *tmem_slot;
  const int ntiles = (sd.T + kTile - 1) / kTile;

  if (warp == 0) {
    // ===== MMA issuer =====
    if (lane == 0) {
      const uint32_t idesc32 = make_idesc(2 * kNOut), idesc16 = make_idesc(kNOut);
      const uint32_t a_lbo = (uint32_t)NROWS * 16u, a_sbo = 128u, b_lbo = 512u, b_sbo = 128u;
      for (int i = 0; i < ntiles; ++i) {
        const int s = i & 1;
        mbar_wait(&full[s], (uint32_t)((i >> 1) & 1));
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t a_hi = smem_u32(aop + (size_t)(2 * s) * aop_words), a_lo = a_hi + 4u * (uint32_t)aop_words;
        const uint32_t b_all = smem_u32(bop);
        const uint32_t d = tmem_base + (uint32_t)(s * 3 * kNOut);  // [A_hi B_hi | A_hi B_lo | A_lo B_hi]
        uint32_t accf = 0u;
        for (int u = 0; u < taps; ++u) {
#pragma unroll
          for (int ks = 0; ks < 2; ++ks) {
            const uint32_t ao = (uint32_t)(2 * ks) * a_lbo + (uint32_t)u * 16u;  // K cores 2ks, 2ks+1; rows from u
            const uint32_t bo = (uint32_t)((u * 4 + 2 * ks) * 4) * 128u;
            const uint64_t ah = make_desc(a_hi + ao, a_lbo, a_sbo), al = make_desc(a_lo + ao, a_lbo, a_sbo);
            const uint64_t bb = make_desc(b_all + bo, b_lbo, b_sbo);
            mma_tf32(d, ah, bb, idesc32, accf);               // N = 32: B_hi then B_lo
            mma_tf32(d + 2 * kNOut, al, bb, idesc16, accf);   // N = 16: B_hi
            accf = 1u;
          }
        }
        tc_commit(&done[s]);
      }
    }
  } else {
    // ===== workers: stage slab rows, then finish the previous tile =====
    const int w = tid - 32;                       // 0..127
    const int q = warp & 3;                       // tensor-memory lane quarter this warp may read
    const float2* yf = a.yobs + sd.y_off + (long long)f * sd.T * M;
    float2* of = a.yout + sd.y_off + (long long)f * sd.T * M;

    // a slab row (one frame, 2 M floats padded to 16) travels global -> registers one tile ahead of its use
    auto load_row = [&](int t0, int row, float (&v)[kKPad]) {
      const int t = t0 - H + row;
#pragma unroll
      for (int k = 0; k < kKPad; ++k) v[k] = 0.f;
      if (t >= 0 && t < sd.T) {
#pragma unroll
        for (int c = 0; c < M; ++c) {
          const float2 y = yf[(long long)t * M + c];
          v[2 * c] = y.x;
          v[2 * c + 1] = y.y;
        }
      }
    };
    auto stage_row = [&](int s, int row, const float (&v)[kKPad]) {
      float* hi_buf = aop + (size_t)(2 * s) * aop_words;
      float* lo_buf = hi_buf + aop_words;
#pragma unroll
      for (int kc = 0; kc < 4; ++kc) {
        float4 h4, l4;
        h4.x = tf32_hi(v[4 * kc]);
        h4.y = tf32_hi(v[4 * kc + 1]);
        h4.z = tf32_hi(v[4 * kc + 2]);
        h4.w = tf32_hi(v[4 * kc + 3]);
        l4.x = v[4 * kc] - h4.x;
        l4.y = v[4 * kc + 1] - h4.y;
        l4.z = v[4 * kc + 2] - h4.z;
        l4.w = v[4 * kc + 3] - h4.w;
        reinterpret_cast<float4*>(hi_buf)[kc * NROWS + row] = h4;
        reinterpret_cast<float4*>(lo_buf)[kc * NROWS + row] = l4;
      }
    };
    auto finish_tile = [&](int i) {
      const int s = i & 1;
      mbar_wait(&done[s], (uint32_t)((i >> 1) & 1));
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      uint32_t r[kNOut], r1[kNOut], r2[kNOut];
      const uint32_t taddr = tmem_base + ((uint32_t)(q * 32) << 16) + (uint32_t)(s * 3 * kNOut);
#define GSS_TMEM_LD16(dst, addr)                                                                                        \
  asm volatile(                                                                                                         \
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15}, [%16];" \
      : "=r"(dst[0]), "=r"(dst[1]), "=r"(dst[2]), "=r"(dst[3]), "=r"(dst[4]), "=r"(dst[5]), "=r"(dst[6]), "=r"(dst[7]),  \
        "=r"(dst[8]), "=r"(dst[9]), "=r"(dst[10]), "=r"(dst[11]), "=r"(dst[12]), "=r"(dst[13]), "=r"(dst[14]),           \
        "=r"(dst[15])                                                                                                   \
      : "r"(addr)                                                                                                       \
      : "memory")
      GSS_TMEM_LD16(r, taddr);
      GSS_TMEM_LD16(r1, taddr + kNOut);
      GSS_TMEM_LD16(r2, taddr + 2 * kNOut);
#undef GSS_TMEM_LD16
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
      for (int n = 0; n < kNOut; ++n)  // hi*hi + (hi*lo + lo*hi)
        r[n] = __float_as_uint(__uint_as_float(r[n]) + (__uint_as_float(r1[n]) + __uint_as_float(r2[n])));
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      const int row = q * 32 + lane;            // tensor-memory lane = tile row = this thread's frame
      const int t = i * kTile + row;
      if (t < sd.T) {
        // the observation is staged row (row + H) of this tile's buffer: hi + lo restores it exactly
        const float4* hi_buf = reinterpret_cast<const float4*>(aop + (size_t)(2 * s) * aop_words);
        const float4* lo_buf = hi_buf + aop_words / 4;
        float o[kKPad];
#pragma unroll
        for (int kc = 0; kc < 4; ++kc) {
          const float4 h4 = hi_buf[kc * NROWS + row + H], l4 = lo_buf[kc * NROWS + row + H];
          o[4 * kc] = h4.x + l4.x;
          o[4 * kc + 1] = h4.y + l4.y;
          o[4 * kc + 2] = h4.z + l4.z;
          o[4 * kc + 3] = h4.w + l4.w;
        }
        float pw = 0.f;  // squared norm of the output frame, accumulated like wpe_power_kernel does
#pragma unroll
        for (int c = 0; c < M; ++c) {
          const float2 v = make_float2(o[2 * c] - __uint_as_float(r[c]), o[2 * c + 1] - __uint_as_float(r[8 + c]));
          of[(long long)t * M + c] = v;
          pw += v.x * v.x + v.y * v.y;
        }
        // the next iteration's lambda_t is the power of exactly this frame (wpe.hpp:40-56 with psd_context 0):
        // writing 1 / lambda here saves that iteration's pass over the tensor
        if (a.w_next != nullptr) {
          // (double)pw / M rounded to float: the reciprocal multiply differs from the division by at most one
          // ulp of a double, which the rounding to float absorbs
          const float lambda = fmaxf((float)kPowerFloor, (float)((double)pw * (1.0 / (double)M)));
          a.w_next[sd.w_off + (long long)f * sd.T + t] = __frcp_rn(lambda);
        }
      }
    };

    const bool extra = w < NROWS - kTile;  // rows past the first 128 of a tile's slab
    float va[kKPad], vb[kKPad];
    load_row(0, w, va);
    if (extra) load_row(0, kTile + w, vb);
    for (int i = 0; i < ntiles; ++i) {
      const int s = i & 1;
      // Buffer s was last read by the MMAs of tile i-2 (finish_tile(i-2) waited for them) and by the OTHER
      // workers' finish_tile(i-2), which takes the observation from it: all 128 workers must be past that.
      asm volatile("bar.sync 1, 128;" ::: "memory");
      stage_row(s, w, va);
      if (extra) stage_row(s, kTile + w, vb);
      if (i + 1 < ntiles) {  // next tile's rows: in flight while this tile's MMAs and the epilogue run
        load_row((i + 1) * kTile, w, va);
        if (extra) load_row((i + 1) * kTile, kTile + w, vb);
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic-proxy stores -> tensor core reads
      mbar_arrive(&full[s]);
      if (i > 0) finish_tile(i - 1);
    }
    finish_tile(ntiles - 1);
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(128u) : "memory");
  }
}

// ---------------------------------------------------------------------------
// The same prediction on kind::f16. Every tcgen05.mma costs ~150 cycles whatever its shape or kind
// (tools/mma_probe.cu) and this kernel is bound by its MMA stream (N = 16 / 32 per instruction), so the lever is
// the instruction count: FP16 operands take K = 16 per MMA, i.e. one instruction per tap where TF32 needs two.
// FP16 has a 5-bit exponent, so both operands are scaled by powers of two -- the slab by the largest magnitude of
// the tile (128 + H frames of one bin), conj(G) by its largest entry -- and split hi + lo exactly as the TF32 kind
// does (hi * hi + hi * lo + lo * hi, each product exact in FP32); the accumulator is rescaled exactly afterwards.
// 11 + 11 bits hold down to 2^-14 of the tile's maximum after scaling to 2^15; the 2^-24 grid below that keeps
// 2^-40 of the maximum absolutely, so a frame 100 dB under the loudest frame of its tile still has FP32-level
// precision and one 140 dB under it 2^-17. The observation is kept in FP32 beside the operands: Y = obs - pred
// subtracts from the exact value.
// ---------------------------------------------------------------------------
namespace {
__device__ __forceinline__ uint32_t make_idesc_f16(int n) {  // kind::f16, FP16 x FP16 -> FP32, K-major, M = 128
  return (1u << 4) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
}
__device__ __forceinline__ void mma_f16(uint32_t tmem_d, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                        uint32_t accumulate) {
  asm volatile(
      "{\n\t"
      ".reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t"
      "}\n" ::"r"(tmem_d),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}
/// 2^e that puts a magnitude bound just under 2^15, clamped so that products of two such factors stay normal floats
__device__ __forceinline__ int scale_exp_f16(float bound) {
  const int eb = (int)((__float_as_uint(bound) >> 23) & 255u) - 127;
  return min(60, max(-60, 14 - eb));
}
__device__ __forceinline__ float pow2f(int e) { return __uint_as_float((uint32_t)(e + 127) << 23); }
__device__ __forceinline__ uint32_t h2_bits(__half2 h) { return *reinterpret_cast<uint32_t*>(&h); }

__host__ __device__ inline size_t app_h_smem(int taps, int H) {
  // header | B operands [tap][K core 2][hi ng0 ng1, lo ng0 ng1][8 x 16 B] | A operands [stage 2][hi, lo][K core 2][rows][16 B]
  // | observations [stage 2][K core 4][rows][4 floats]
  return 128 + (size_t)taps * 1024 + 4 * (size_t)(2 * app_rows(H) * 16) + 2 * (size_t)(4 * app_rows(H) * 16);
}
}  // namespace

template <int M>
__global__ void __launch_bounds__(kAppThreads, app_min_blocks(M)) wpe_apply_h_kernel(WpeArgs a) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const SegDev sd = a.segs[blockIdx.y];
  if (!sd.wpe_active) return;
  const int f = blockIdx.x;
  const int taps = a.taps, km = taps * M, H = a.delay + taps - 1;
  const int NROWS = app_rows(H);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

  uint64_t* full = reinterpret_cast<uint64_t*>(smem_raw);              // [2] slab of a tile is staged
  uint64_t* done = full + 2;                                           // [2] MMAs of a tile are complete
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem_raw + 32);
  float* red_a = reinterpret_cast<float*>(smem_raw + 64);              // [2 parities][4 worker warps] tile maxima
  float* red_g = reinterpret_cast<float*>(smem_raw + 96);              // [5 warps] filter maxima
  __half* bop = reinterpret_cast<__half*>(smem_raw + 128);
  unsigned char* aop = smem_raw + 128 + (size_t)taps * 1024;
  const uint32_t aop_bytes = 2u * (uint32_t)NROWS * 16u;               // one of hi / lo of one stage
  float4* obs = reinterpret_cast<float4*>(aop + 4 * (size_t)aop_bytes);  // [stage][K core 4][NROWS]

  if (tid == 0) {
    mbar_init(&full[0], 128);
    mbar_init(&full[1], 128);
    mbar_init(&done[0], 1);
    mbar_init(&done[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(128u)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  // conj(G) of this bin as the B operands (real 2x2 blocks of the complex product), scaled, hi / lo split
  int eg;
  {
    const float2* g = a.gconj + sd.g_wpe_off + (long long)f * km * M;
    float mg = 0.f;
    for (int i = tid; i < km * M; i += kAppThreads) mg = fmaxf(mg, fmaxf(fabsf(g[i].x), fabsf(g[i].y)));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mg = fmaxf(mg, __shfl_xor_sync(0xffffffffu, mg, o));
    if (lane == 0) red_g[warp] = mg;
    __syncthreads();
    mg = fmaxf(fmaxf(fmaxf(red_g[0], red_g[1]), fmaxf(red_g[2], red_g[3])), red_g[4]);
    eg = scale_exp_f16(mg);
    const float sg = pow2f(eg);
    for (int i = tid; i < taps * kKPad * kNOut; i += kAppThreads) {
      const int u = i / (kKPad * kNOut), r = i - u * (kKPad * kNOut), kappa = r / kNOut, n = r - kappa * kNOut;
      const int c = kappa >> 1, part = kappa & 1, c2 = n & 7, im_out = n >> 3;
      float v = 0.f;
      if (c < M && c2 < M) {
        const float2 gg = g[(u * M + c) * M + c2];
        v = (part == 0 ? (im_out ? gg.y : gg.x) : (im_out ? gg.x : -gg.y)) * sg;
      }
      const __half hi = __float2half_rn(v);
      const __half lo = __float2half_rn(v - __half2float(hi));
      // half index: (((tap, K core), n group), n row, K element); n groups 0, 1 = B_hi, 2, 3 = B_lo
      const int at = (((u * 2 + (kappa >> 3)) * 4 + (n >> 3)) * 8 + (n & 7)) * 8 + (kappa & 7);
      bop[at] = hi;
      bop[at + 2 * 64] = lo;
    }
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem_base = *tmem_slot;
  const int ntiles = (sd.T + kTile - 1) / kTile;

  if (warp == 0) {
    // ===== MMA issuer: one instruction pair per tap =====
    if (lane == 0) {
      const uint32_t idesc32 = make_idesc_f16(2 * kNOut), idesc16 = make_idesc_f16(kNOut);
      const uint32_t a_lbo = (uint32_t)NROWS * 16u, a_sbo = 128u, b_lbo = 512u, b_sbo = 128u;
      for (int i = 0; i < ntiles; ++i) {
        const int s = i & 1;
        mbar_wait(&full[s], (uint32_t)((i >> 1) & 1));
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t a_hi = smem_u32(aop) + (uint32_t)(2 * s) * aop_bytes, a_lo = a_hi + aop_bytes;
        const uint32_t b_all = smem_u32(bop);
        const uint32_t d = tmem_base + (uint32_t)(s * 3 * kNOut);  // [A_hi B_hi | A_hi B_lo | A_lo B_hi]
        for (int u = 0; u < taps; ++u) {
          const uint32_t ao = (uint32_t)u * 16u;  // rows from u
          const uint64_t ah = make_desc(a_hi + ao, a_lbo, a_sbo), al = make_desc(a_lo + ao, a_lbo, a_sbo);
          const uint64_t bb = make_desc(b_all + (uint32_t)u * 1024u, b_lbo, b_sbo);
          mma_f16(d, ah, bb, idesc32, u > 0 ? 1u : 0u);               // N = 32: B_hi then B_lo
          mma_f16(d + 2 * kNOut, al, bb, idesc16, u > 0 ? 1u : 0u);   // N = 16: B_hi
        }
        tc_commit(&done[s]);
      }
    }
  } else {
    // ===== workers: stage slab rows, then finish the previous tile =====
    const int w = tid - 32;                       // 0..127
    const int q = warp & 3;                       // tensor-memory lane quarter this warp may read
    const float2* yf = a.yobs + sd.y_off + (long long)f * sd.T * M;
    float2* of = a.yout + sd.y_off + (long long)f * sd.T * M;
    float inv_s0 = 1.f, inv_s1 = 1.f;             // 2^-(ea + eg) of the tile staged in buffer 0 / 1

    auto load_row = [&](int t0, int row, float (&v)[kKPad]) {
      const int t = t0 - H + row;
#pragma unroll
      for (int k = 0; k < kKPad; ++k) v[k] = 0.f;
      if (t >= 0 && t < sd.T) {
        if constexpr (M % 2 == 0) {  // a frame is a whole number of 16-byte pieces (and 16-byte aligned): half the requests
          const float4* p = reinterpret_cast<const float4*>(yf + (long long)t * M);
#pragma unroll
          for (int c = 0; c < M / 2; ++c) {
            const float4 y = p[c];
            v[4 * c] = y.x;
            v[4 * c + 1] = y.y;
            v[4 * c + 2] = y.z;
            v[4 * c + 3] = y.w;
          }
        } else {
#pragma unroll
          for (int c = 0; c < M; ++c) {
            const float2 y = yf[(long long)t * M + c];
            v[2 * c] = y.x;
            v[2 * c + 1] = y.y;
          }
        }
      }
    };
    auto row_max = [&](const float (&v)[kKPad]) {
      float m = 0.f;
#pragma unroll
      for (int k = 0; k < 2 * M; ++k) m = fmaxf(m, fabsf(v[k]));
      return m;
    };
    auto stage_row = [&](int s, int row, const float (&v)[kKPad], float scl) {
      unsigned char* hi_buf = aop + (size_t)(2 * s) * aop_bytes;
      unsigned char* lo_buf = hi_buf + aop_bytes;
      float4* ob = obs + (size_t)s * 4 * NROWS;
#pragma unroll
      for (int kc = 0; kc < 4; ++kc) ob[kc * NROWS + row] = make_float4(v[4 * kc], v[4 * kc + 1], v[4 * kc + 2], v[4 * kc + 3]);
#pragma unroll
      for (int kc = 0; kc < 2; ++kc) {
        uint32_t h[4], l[4];
#pragma unroll
        for (int p = 0; p < 4; ++p) {
          const float x0 = v[8 * kc + 2 * p] * scl, x1 = v[8 * kc + 2 * p + 1] * scl;
          const __half2 hh = __floats2half2_rn(x0, x1);
          const float2 hf = __half22float2(hh);
          h[p] = h2_bits(hh);
          l[p] = h2_bits(__floats2half2_rn(x0 - hf.x, x1 - hf.y));
        }
        reinterpret_cast<uint4*>(hi_buf)[kc * NROWS + row] = make_uint4(h[0], h[1], h[2], h[3]);
        reinterpret_cast<uint4*>(lo_buf)[kc * NROWS + row] = make_uint4(l[0], l[1], l[2], l[3]);
      }
    };
    auto finish_tile = [&](int i) {
      const int s = i & 1;
      mbar_wait(&done[s], (uint32_t)((i >> 1) & 1));
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      uint32_t r[kNOut], r1[kNOut], r2[kNOut];
      const uint32_t taddr = tmem_base + ((uint32_t)(q * 32) << 16) + (uint32_t)(s * 3 * kNOut);
#define GSS_TMEM_LD16(dst, addr)                                                                                        \
  asm volatile(                                                                                                         \
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15}, [%16];" \
      : "=r"(dst[0]), "=r"(dst[1]), "=r"(dst[2]), "=r"(dst[3]), "=r"(dst[4]), "=r"(dst[5]), "=r"(dst[6]), "=r"(dst[7]),  \
        "=r"(dst[8]), "=r"(dst[9]), "=r"(dst[10]), "=r"(dst[11]), "=r"(dst[12]), "=r"(dst[13]), "=r"(dst[14]),           \
        "=r"(dst[15])                                                                                                   \
      : "r"(addr)                                                                                                       \
      : "memory")
      GSS_TMEM_LD16(r, taddr);
      GSS_TMEM_LD16(r1, taddr + kNOut);
      GSS_TMEM_LD16(r2, taddr + 2 * kNOut);
#undef GSS_TMEM_LD16
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      const float inv = s == 0 ? inv_s0 : inv_s1;
#pragma unroll
      for (int n = 0; n < kNOut; ++n)  // (hi*hi + (hi*lo + lo*hi)) rescaled: a power of two, exact
        r[n] = __float_as_uint((__uint_as_float(r[n]) + (__uint_as_float(r1[n]) + __uint_as_float(r2[n]))) * inv);
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      const int row = q * 32 + lane;            // tensor-memory lane = tile row = this thread's frame
      const int t = i * kTile + row;
      if (t < sd.T) {
        const float4* ob = obs + (size_t)s * 4 * NROWS;  // the observation is slab row (row + H) of this tile
        float o[kKPad];
#pragma unroll
        for (int kc = 0; kc < 4; ++kc) {
          const float4 v4 = ob[kc * NROWS + row + H];
          o[4 * kc] = v4.x;
          o[4 * kc + 1] = v4.y;
          o[4 * kc + 2] = v4.z;
          o[4 * kc + 3] = v4.w;
        }
        float pw = 0.f;  // squared norm of the output frame, accumulated like wpe_power_kernel does
        float2 out[M];
#pragma unroll
        for (int c = 0; c < M; ++c) {
          out[c] = make_float2(o[2 * c] - __uint_as_float(r[c]), o[2 * c + 1] - __uint_as_float(r[8 + c]));
          pw += out[c].x * out[c].x + out[c].y * out[c].y;
        }
        if constexpr (M % 2 == 0) {
          float4* p = reinterpret_cast<float4*>(of + (long long)t * M);
#pragma unroll
          for (int c = 0; c < M / 2; ++c) p[c] = make_float4(out[2 * c].x, out[2 * c].y, out[2 * c + 1].x, out[2 * c + 1].y);
        } else {
#pragma unroll
          for (int c = 0; c < M; ++c) of[(long long)t * M + c] = out[c];
        }
        if (a.w_next != nullptr) {  // the next iteration's Gram weight of this frame (see wpe_apply_tc_kernel)
          const float lambda = fmaxf((float)kPowerFloor, (float)((double)pw * (1.0 / (double)M)));
          a.w_next[sd.w_off + (long long)f * sd.T + t] = __frcp_rn(lambda);
        }
      }
    };

    const bool extra = w < NROWS - kTile;  // rows past the first 128 of a tile's slab
    float va[kKPad], vb[kKPad];
    load_row(0, w, va);
    if (extra) load_row(0, kTile + w, vb);
    for (int i = 0; i < ntiles; ++i) {
      const int s = i & 1;
      // largest magnitude of this tile's slab: every worker's rows, exchanged across the barrier that also orders
      // the reuse of buffer s (last read by the MMAs of tile i-2 and by the other workers' finish_tile(i-2))
      float m = row_max(va);
      if (extra) m = fmaxf(m, row_max(vb));
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
      if (lane == 0) red_a[s * 4 + q] = m;
      asm volatile("bar.sync 1, 128;" ::: "memory");
      m = fmaxf(fmaxf(red_a[s * 4], red_a[s * 4 + 1]), fmaxf(red_a[s * 4 + 2], red_a[s * 4 + 3]));
      const int ea = scale_exp_f16(m);
      const float scl = pow2f(ea);
      if (s == 0) inv_s0 = pow2f(-ea - eg);
      else inv_s1 = pow2f(-ea - eg);
      stage_row(s, w, va, scl);
      if (extra) stage_row(s, kTile + w, vb, scl);
      if (i + 1 < ntiles) {  // next tile's rows: in flight while this tile's MMAs and the epilogue run
        load_row((i + 1) * kTile, w, va);
        if (extra) load_row((i + 1) * kTile, kTile + w, vb);
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic-proxy stores -> tensor core reads
      mbar_arrive(&full[s]);
      if (i > 0) finish_tile(i - 1);
    }
    finish_tile(ntiles - 1);
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(128u) : "memory");
  }
}

// ---------------------------------------------------------------------------
int wpe_apply_tc_supported(int taps, int delay, int M) {
  const int H = delay + taps - 1;
  const size_t smem = 128 + sizeof(float) * (2 * (size_t)taps * 256 + 4 * (size_t)(4 * app_rows(H) * 4));
  // a tile stages row w and, when there are more than kTile rows, row kTile + w: at most 2 * kTile slab rows, so the
  // history H = delay + taps - 1 has to fit the second half (larger H runs the FP32 kernel wpe_apply2_kernel)
  return M >= 1 && M <= 8 && app_rows(H) <= 2 * kTile && smem <= 100 * 1024 ? 1 : 0;
}

template <int M>
static cudaError_t launch_apply_tc_m(const WpeArgs& a, int nseg, int F, cudaStream_t st) {
  const int H = a.delay + a.taps - 1;
  if (a.apply_f16) {
    const size_t smem = app_h_smem(a.taps, H);
    cudaError_t e = cudaFuncSetAttribute(wpe_apply_h_kernel<M>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    wpe_apply_h_kernel<M><<<dim3(F, nseg), kAppThreads, smem, st>>>(a);
    return cudaGetLastError();
  }
  const size_t smem = 128 + sizeof(float) * (2 * (size_t)a.taps * 256 + 4 * (size_t)(4 * app_rows(H) * 4));
  cudaError_t e = cudaFuncSetAttribute(wpe_apply_tc_kernel<M>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  wpe_apply_tc_kernel<M><<<dim3(F, nseg), kAppThreads, smem, st>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_wpe_apply_tc(const WpeArgs& a, int nseg, int F, cudaStream_t st) {
  switch (a.M) {
    case 1: return launch_apply_tc_m<1>(a, nseg, F, st);
    case 2: return launch_apply_tc_m<2>(a, nseg, F, st);
    case 3: return launch_apply_tc_m<3>(a, nseg, F, st);
    case 4: return launch_apply_tc_m<4>(a, nseg, F, st);
    case 5: return launch_apply_tc_m<5>(a, nseg, F, st);
    case 6: return launch_apply_tc_m<6>(a, nseg, F, st);
    case 7: return launch_apply_tc_m<7>(a, nseg, F, st);
    case 8: return launch_apply_tc_m<8>(a, nseg, F, st);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace gssb
