// wpe_gram_tc.cu -- the WPE weighted Gram (wpe.hpp:72-89, numerics.hpp:128-152) on the 5th-generation
// tensor cores: tcgen05.mma kind::tf32 with a 3xTF32 split, FP32 accumulators in tensor memory.
//
// Real formulation. For one (segment, bin) let s_t be the real row vector
//     [ Re a_t (km) | Im a_t (km) | Re y_t (M) | Im y_t (M) | 0-pad ]   scaled by sqrt(w_t),
// a_t = the tap-stacked history window of frame t (reverse tap order, see wpe_kernels.cu), y_t the current
// frame. Then G = sum_t s_t^T s_t (NR x NR, symmetric) holds every real product the complex Gram needs:
//     Re R[e][e'] = G[e][e'] + G[km+e][km+e']          Im R[e][e'] = G[km+e][e'] - G[e][km+e']
//     Re P[e][c]  = G[e][2km+c] + G[km+e][2km+M+c]     Im P[e][c]  = G[km+e][2km+c] - G[e][2km+M+c]
// The SAME staged operand is both MMA operands (A = rows 0..127, B = all NR rows, both K-major with the
// frame index as K), so one expansion of the slab feeds the whole product. Rows >= 128 (NR = 160 at M = 7,
// 176 at M = 8) are covered by a second accumulator D2 = S[NR-64..NR) x S[128..NR)^T (M = 64); symmetry gives the
// rest. FP32 accuracy comes from the split x = hi + lo (hi = top 19 bits): hi*hi + hi*lo + lo*hi.
//
// Pipeline per CTA (one (segment, bin), 256 threads): per chunk of 32 frames all warps expand the slab into
// the canonical no-swizzle K-major core-matrix layout (a warp store = one 8x16-byte core matrix, conflict
// free), fence to the async proxy, and one thread issues the chunk's MMAs and commits them to the
// buffer's mbarrier; the next chunk is expanded into the other buffer while the tensor core runs.
#include <algorithm>

#include <cuda_fp16.h>

#include "kernels.h"

namespace gssb {

namespace {

constexpr int kTcWorkers = 512;             // 16 warps expand the operands and fold the accumulators
constexpr int kTcWorkerWarps = kTcWorkers / 32;
constexpr int kTcThreads = kTcWorkers + 32; // + one warp whose lane 0 issues the MMAs
constexpr int kKW = 64;                     // 32-bit words per operand row and pipeline stage: 8 MMA k-steps of 32 bytes
constexpr int kCoreWords = 32;              // one core matrix: 8 rows x 16 bytes
constexpr int kKCores = kKW / 4;            // core matrices along K per row group (= kTcWorkerWarps)
// Frames per pipeline stage. kind::tf32 takes K = 8 frames per MMA (4 per worker warp and stage), kind::f16 K = 16
// (8 per warp): an MMA costs ~150 cycles whatever its shape or kind (tools/mma_probe.cu), so the FP16 split halves
// the MMA stream per frame -- and the operand bytes, drains and barriers with it.
__host__ __device__ constexpr int tc_kc(int f16) { return f16 ? 128 : 64; }
constexpr int kHead = 256;                  // barriers, the tensor-memory slot, the scale reduction scratch
constexpr int kLook = 8;                    // look-ahead frames read by the padded rows
constexpr int kAccPerThread = 56;           // register accumulators per thread: NCT <= 224 columns / 4 quarters

// Row layout of the staged operand S (each block padded to a multiple of 8 rows so that a row group is
// homogeneous): [Re a (KMP)] [Im a (KMP)] [Re y (8)] [Im y (8)] [zero pad to a multiple of 16].
__host__ __device__ inline int tc_kmp(int km) { return (km + 7) & ~7; }
__host__ __device__ inline int tc_rows(int km, int M) { return wpe_tc_operand_rows(km); }  // NR
__host__ __device__ inline int tc_buf_rows(int km, int M) { return tc_rows(km, M) < 128 ? 128 : tc_rows(km, M); }
__host__ __device__ inline int tc_n2(int km, int M) { return tc_rows(km, M) > 128 ? tc_rows(km, M) - 128 : 0; }
__host__ __device__ inline int tc_cols(int km, int M) { return tc_rows(km, M) + tc_n2(km, M); }         // D1 | D2
/// Bytes ahead of the operand buffers: barriers, Gram weights, three stages of planar slabs (H = history frames).
__host__ __device__ inline size_t tc_head_bytes(int M, int H, int kc) {
  // Gram weights [3][kc], slab planes [3][re, im][frames * M], per-frame slab maxima [frames] (FP16 kind)
  const size_t off = kHead + sizeof(float) * (3 * kc + (6 * (size_t)M + 1) * (size_t)(kc + H + kLook));
  return (off + 127) & ~(size_t)127;
}
__host__ __device__ inline size_t tc_smem_bytes(int km, int M, int H, int stages, int kc) {
  return tc_head_bytes(M, H, kc) + sizeof(float) * 2 * (size_t)stages * (size_t)tc_buf_rows(km, M) * kKW;
}
/// Operand / accumulator pipeline depth. With two stages the tensor core idles while the workers drain and refill
/// the buffer it just finished, which at the small tiles takes longer than a chunk of MMAs (M = 4: 1685 cycles of
/// MMAs against ~3700 of drain + expansion per 64-frame chunk). Three stages fit when the tile is 128 rows, an
/// accumulator set is at most 160 columns and the slabs leave room (M = 4, 5 at the default history: 196 KB of operands).
__host__ __device__ inline int tc_stages(int km, int M, int H, int kc) {
  return tc_buf_rows(km, M) == 128 && tc_cols(km, M) <= 160 && tc_smem_bytes(km, M, H, 3, kc) <= 224 * 1024 ? 3 : 2;
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

/// K-major, no swizzle: 8-row groups SBO bytes apart, the two 16-byte K chunks of one MMA LBO bytes apart.
__device__ __forceinline__ uint64_t make_smem_desc(uint32_t addr, uint32_t lbo_bytes, uint32_t sbo_bytes) {
  uint64_t d = 0;
  d |= (uint64_t)((addr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo_bytes >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo_bytes >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;  // descriptor version (Blackwell)
  return d;                // base offset 0, lbo mode 0, layout type 0 = SWIZZLE_NONE
}

/// kind::tf32, FP32 accumulate, both operands K-major, M = 128.
__device__ __forceinline__ uint32_t make_idesc_tf32(int n, int m = 128) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(m >> 4) << 24);
}

/// kind::f16 with FP16 operands (format 0), FP32 accumulate, both operands K-major.
__device__ __forceinline__ uint32_t make_idesc_f16(int n, int m = 128) {
  return (1u << 4) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(m >> 4) << 24);
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
/// Bounded wait: a protocol error traps (an error for the caller) instead of hanging the device.
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  const uint32_t addr = smem_u32(bar);
  for (int spin = 0; spin < (1 << 28); ++spin) {
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
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void workers_sync() { asm volatile("bar.sync 1, %0;" ::"n"(kTcWorkers) : "memory"); }
__device__ __forceinline__ float sqrt_approx_tc(float x) {
  float r;
  asm("sqrt.approx.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}
__device__ __forceinline__ void tc_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}

}  // namespace

/// TAPS > 0 fixes the tap count at compile time (all loops unroll, no guards); TAPS == 0 reads it from the
/// arguments.
/// F16 = 1: kind::f16 on an FP16 hi / lo split of the operands scaled, per stage, by a power of two that puts the
/// largest magnitude of the stage just under 2^15 (FP16 keeps 11 bits down to 2^-14 and a 2^-24 grid below that, a
/// range of 2^39 in all; the accumulators are rescaled exactly when they are folded). Same products as the TF32
/// split: hi*hi + hi*lo + lo*hi, each exact in FP32.
template <int M, int TAPS, int F16>
__global__ void __launch_bounds__(kTcThreads, 1) wpe_gram_tc_kernel(WpeArgs a) {
  constexpr int kKC = tc_kc(F16);  // frames per pipeline stage
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const SegDev sd = a.segs[blockIdx.y];
  if (!sd.wpe_active) return;
  const int f = blockIdx.x;
  const int taps = TAPS > 0 ? TAPS : a.taps;
  const int km = taps * M, H = a.delay + taps - 1, KMP = tc_kmp(km);
  const int NR = tc_rows(km, M), NB = tc_buf_rows(km, M), N2 = tc_n2(km, M), NCT = NR + N2;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int SF = kKC + H + kLook;  // slab frames per chunk

  // shared memory carve-up
  const int NS = tc_stages(km, M, H, kKC);                               // operand buffers / accumulator sets
  const uint32_t setw = NS == 3 ? 160u : 256u;                        // tensor-memory columns per accumulator set
  uint64_t* full = reinterpret_cast<uint64_t*>(smem_raw);             // [3] operands of a chunk are staged
  uint64_t* done = full + 3;                                          // [3] MMAs of a chunk are complete
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem_raw + 64);
  float* red = reinterpret_cast<float*>(smem_raw + 128);              // [2 parities][history, current frame][4 warps] stage maxima (F16)
  float* wbuf = reinterpret_cast<float*>(smem_raw + kHead);           // [3][kKC] Gram weights
  float* planes = wbuf + 3 * kKC;                                     // [3 stages][re, im][SF * M]
  const int plane_words = SF * M;
  float* fmx = planes + 6 * plane_words;                              // [SF] largest |re|, |im| of a slab frame (F16)
  const size_t off = tc_head_bytes(M, H, kKC);
  const int buf_words = NB * kKW;                                     // one operand buffer (hi or lo)
  float* opbuf = reinterpret_cast<float*>(smem_raw + off);            // [stage][hi/lo][buf_words]

  if (tid == 0) {
    for (int i = 0; i < 3; ++i) {
      mbar_init(&full[i], kTcWorkerWarps);
      mbar_init(&done[i], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  // NS accumulator sets (D1 | D2 each): every chunk's products start from zero and are folded into FP32
  // registers with round-to-nearest. The tensor core's own accumulation truncates; a chain of thousands
  // of MMAs loses ~1e-4 of the Gram, a chain of 12 stays at the 3xTF32 level (1e-6).
  if (warp == kTcWorkerWarps) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(512u)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem_base = *tmem_slot;
  const int nchunk = (sd.T + kKC - 1) / kKC;
  const uint32_t sbo = kKCores * 128, lbo = 128;

  if (warp == kTcWorkerWarps) {
    // ===== MMA issuer =====
    if (lane == 0) {
      const uint32_t idesc1 = F16 ? make_idesc_f16(NR) : make_idesc_tf32(NR);
      const uint32_t idesc2 = F16 ? make_idesc_f16(N2 > 0 ? N2 : 16, 64) : make_idesc_tf32(N2 > 0 ? N2 : 16, 64);
      auto mma = [](uint32_t d, uint64_t da, uint64_t db, uint32_t idesc, uint32_t acc) {
        if constexpr (F16) mma_f16(d, da, db, idesc, acc);
        else mma_tf32(d, da, db, idesc, acc);
      };
      // The corner (rows and columns >= 128) is read back only where an Im a row lies beyond row 127, i.e. when
      // KMP + km > 128 (M = 7, 8). At M = 6 rows 128.. are the y rows, needed as columns only: no corner MMAs, and
      // since every MMA costs ~150 cycles whatever its shape (tools/mma_probe.cu) that is half of the MMA stream.
      const bool corner = N2 > 0 && KMP + km > 128;
      for (int c = 0; c < nchunk; ++c) {
        const int b = c % NS;
        mbar_wait(&full[b], (uint32_t)((c / NS) & 1));
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t a_hi = smem_u32(opbuf + (size_t)(2 * b) * buf_words), a_lo = a_hi + 4u * (uint32_t)buf_words;
        const uint32_t d1 = tmem_base + (uint32_t)b * setw, d2 = d1 + (uint32_t)NR;
#pragma unroll
        for (int ks = 0; ks < kKW / 8; ++ks) {  // 32 bytes of K per MMA: 8 TF32 or 16 FP16 frames
          const uint32_t accf = ks > 0 ? 1u : 0u;  // every chunk starts its accumulator set from zero
          const uint32_t ko = ks * 256;            // two core matrices along K per MMA
          const uint64_t dh = make_smem_desc(a_hi + ko, lbo, sbo), dl = make_smem_desc(a_lo + ko, lbo, sbo);
          mma(d1, dh, dh, idesc1, accf);
          mma(d1, dh, dl, idesc1, 1u);
          mma(d1, dl, dh, idesc1, 1u);
          if (corner) {
            // the corner is an M = 64 MMA on the last 64 rows: the kernel is bound by the operand bytes it
            // streams from shared memory, and a 64-row A tile is half of them (row r of that accumulator
            // lives in tensor-memory lane 32 (r / 16) + r % 16)
            const uint32_t ra = ((NR - 64) / 8) * sbo, rb = 16 * sbo;  // rows NR-64.. and rows 128..
            const uint64_t ah = make_smem_desc(a_hi + ra + ko, lbo, sbo), al = make_smem_desc(a_lo + ra + ko, lbo, sbo);
            const uint64_t bh = make_smem_desc(a_hi + rb + ko, lbo, sbo), bl = make_smem_desc(a_lo + rb + ko, lbo, sbo);
            mma(d2, ah, bh, idesc2, accf);
            mma(d2, ah, bl, idesc2, 1u);
            mma(d2, al, bh, idesc2, 1u);
          }
        }
        tc_commit(&done[b]);
      }
    }
  } else {
    // ===== workers: stage the slab, expand it into MMA operands, fold finished accumulators =====
    const float2* yf = a.yobs + sd.y_off + (long long)f * sd.T * M;
    const float* wf = a.w + sd.w_off + (long long)f * sd.T;
    // slab of chunk c: frames [c*kKC - H, c*kKC + kKC + kLook), planar, zero outside [0, T) (wpe.hpp:74-75)
    auto issue_slab = [&](int c) {
      const int st = c % 3;
      float* re = planes + (size_t)(2 * st) * plane_words;
      float* im = re + plane_words;
      const int t_first = c * kKC - H;
      for (int i = tid; i < plane_words; i += kTcWorkers) {
        const int fr = i / M;
        const int t = t_first + fr;
        if (t >= 0 && t < sd.T) {
          const float* src = reinterpret_cast<const float*>(yf + (long long)t_first * M + i);
          asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(re + i)), "l"(src) : "memory");
          asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(im + i)), "l"(src + 1) : "memory");
        } else {
          re[i] = 0.f;
          im[i] = 0.f;
        }
      }
      if (tid < kKC) {
        const int t = c * kKC + tid;
        if (t < sd.T)
          asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(wbuf + st * kKC + tid)), "l"(wf + t)
                       : "memory");
        else
          wbuf[st * kKC + tid] = 0.f;
      }
      asm volatile("cp.async.commit_group;" ::: "memory");
    };

    // register accumulators: thread (lane quarter q = warp % 4, column quarter cq = warp / 4) owns row
    // 32 q + lane and the columns [cq * NCQ, (cq + 1) * NCQ) of D1 | D2
    const int NCQ = NCT / 4;  // NCT is a multiple of 16
    float acc[kAccPerThread];
#pragma unroll
    for (int i = 0; i < kAccPerThread; ++i) acc[i] = 0.f;
    const int q = warp & 3, qcol = (warp >> 2) * NCQ;

    // F16: the rescale factors of the stage whose accumulators sit in set 0 / 1 / 2: 2^-(ea + ea) for a product of two
    // history rows, 2^-(ea + ey) for history x current frame (powers of two: the rescale is exact)
    float iaa_0 = 1.f, iaa_1 = 1.f, iaa_2 = 1.f, iay_0 = 1.f, iay_1 = 1.f, iay_2 = 1.f;
    auto drain = [&](int set) {
      const float iaa = set == 0 ? iaa_0 : set == 1 ? iaa_1 : iaa_2;
      const float iay = set == 0 ? iay_0 : set == 1 ? iay_1 : iay_2;
      const uint32_t taddr = tmem_base + ((uint32_t)(q * 32) << 16) + (uint32_t)set * setw + (uint32_t)qcol;
      constexpr int kBatch = 32;  // columns in flight per wait
#pragma unroll
      for (int b0 = 0; b0 < kAccPerThread; b0 += kBatch) {
        uint32_t v[kBatch];
#pragma unroll
        for (int j = 0; j < kBatch / 8; ++j) {
          const int col = b0 + j * 8;
          if (col < kAccPerThread && col < NCQ)  // warp-uniform; static when TAPS is
            asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
                         : "=r"(v[j * 8]), "=r"(v[j * 8 + 1]), "=r"(v[j * 8 + 2]), "=r"(v[j * 8 + 3]),
                           "=r"(v[j * 8 + 4]), "=r"(v[j * 8 + 5]), "=r"(v[j * 8 + 6]), "=r"(v[j * 8 + 7])
                         : "r"(taddr + col)
                         : "memory");
        }
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
        for (int j = 0; j < kBatch / 8; ++j) {
          const int col = b0 + j * 8;
          if (col < kAccPerThread && col < NCQ) {
            // columns of D1 are operand rows 0..NR-1, those of D2 rows 128..NR-1; rows >= 2 KMP are the current frame
            const int gc = qcol + col, orow = gc < NR ? gc : 128 + (gc - NR);
            const float inv = orow >= 2 * KMP ? iay : iaa;
#pragma unroll
            for (int i = 0; i < 8; ++i) {
              if constexpr (F16) acc[col + i] = fmaf(__uint_as_float(v[j * 8 + i]), inv, acc[col + i]);
              else acc[col + i] += __uint_as_float(v[j * 8 + i]);
            }
          }
        }
      }
    };

    // expand: warp w owns k chunk w (frames 4w .. 4w+3) and walks all row groups; lane -> (row rg*8 + lane/4,
    // frame 4w + lane%4), so a warp store is one 8 x 16-byte core matrix = 128 contiguous bytes
    static_assert(kTcWorkerWarps == kKCores, "one worker warp per K chunk");
    // FP32 words hold one frame, FP16 words a pair: lane % 4 picks frame k (TF32) or frames k, k + 4 (FP16) of the
    // warp's core matrix. (Which frame sits in which K slot is free -- both MMA operands are this one buffer -- and
    // with the pair 4 apart the 32 lanes read 32 different banks of the slab, and, M even, share most of their loads.)
    const int k = F16 ? warp * 8 + (lane & 3) : warp * 4 + (lane & 3), r8 = lane >> 2;
    const int word0 = warp * kCoreWords + lane;  // core (rg, kc = warp) -> (rg * kKCores + warp) * 32 + lane
    // row groups that carry data: [Re a | Im a | Re y | Im y]; the groups after them (padding up to NB rows: a third
    // of the 128-row tile at M = 4) are zero in every chunk, so they are zeroed once here and never rewritten
    const int nrg_a = KMP / 8, nrg = 2 * nrg_a + 2;
    for (int i = tid; i < 2 * NS * (NB - 8 * nrg) * kKW; i += kTcWorkers) {
      const int per = (NB - 8 * nrg) * kKW;  // zero words per operand buffer
      opbuf[(size_t)(i / per) * buf_words + (size_t)(8 * nrg) * kKW + (i % per)] = 0.f;
    }

    issue_slab(0);
    for (int c = 0; c < nchunk; ++c) {
      const int b = c % NS, st = c % 3;
      if (c + 1 < nchunk) {
        issue_slab(c + 1);  // stage (c+1)%3 was last read by the expansion of chunk c-2
        asm volatile("cp.async.wait_group 1;" ::: "memory");
      } else {
        asm volatile("cp.async.wait_group 0;" ::: "memory");
      }
      workers_sync();  // slab of chunk c has landed for every worker
      if (c >= NS) {
        // MMAs of chunk c - NS are complete: operand buffer b and accumulator set b are ours again
        mbar_wait(&done[b], (uint32_t)((c / NS - 1) & 1));
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        drain(b);
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      }
      const float* re = planes + (size_t)(2 * st) * plane_words;
      const float* im = re + plane_words;
      float* hi_buf = opbuf + (size_t)(2 * b) * buf_words;
      float* lo_buf = hi_buf + buf_words;
      const float* rk = re + k * M + r8;
      const float* ik = im + k * M + r8;
      if constexpr (F16) {
        // Stage scales: the exact largest |x| sqrt(w) over the history rows and over the current-frame rows of the
        // stage. Two, because the two differ by the signal's short-term dynamic range (a burst in the history of a
        // near-silent frame is 10^7 times that frame's own normalised value) and every product needs its smaller
        // factor at full precision too: P = sum w a y^H. An element e of the window of stage frame k is slab word
        // k M + e, i.e. slab frames k .. k + taps (the padded rows reach one frame further); the current frame is k + H.
        for (int fr = tid; fr < SF; fr += kTcWorkers) {
          float m = 0.f;
#pragma unroll
          for (int ch = 0; ch < M; ++ch) m = fmaxf(m, fmaxf(fabsf(re[fr * M + ch]), fabsf(im[fr * M + ch])));
          fmx[fr] = m;
        }
        workers_sync();
        float ma = 0.f, my = 0.f;
        if (tid < kKC) {
          const float sqk = sqrt_approx_tc(wbuf[st * kKC + tid]);
          for (int u = 0; u <= taps; ++u) ma = fmaxf(ma, fmx[tid + u]);
          my = fmaxf(fmx[tid + H], fmx[tid + H + 1]) * sqk;
          ma *= sqk;
        }
        float* rd = red + (c & 1) * 8;  // [4 warps] history maxima, [4 warps] current-frame maxima
        if (warp < kKC / 32) {
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) {
            ma = fmaxf(ma, __shfl_xor_sync(0xffffffffu, ma, o));
            my = fmaxf(my, __shfl_xor_sync(0xffffffffu, my, o));
          }
          if (lane == 0) {
            rd[warp] = ma;
            rd[4 + warp] = my;
          }
        }
        workers_sync();
        ma = fmaxf(fmaxf(rd[0], rd[1]), fmaxf(rd[2], rd[3]));
        my = fmaxf(fmaxf(rd[4], rd[5]), fmaxf(rd[6], rd[7]));
        // bound < 2^(eb + 1): scale by 2^(14 - eb). The exponents are clamped so that the rescale factors stay
        // normal floats; a zero, infinite or NaN bound lands on a clamp and the values go through as they are.
        auto scale_exp = [](float bound) {
          const int eb = (int)((__float_as_uint(bound) >> 23) & 255u) - 127;
          return min(60, max(-60, 14 - eb));
        };
        const int ea = scale_exp(ma), ey = scale_exp(my);
        const float scl_a = __uint_as_float((uint32_t)(ea + 127) << 23), scl_y = __uint_as_float((uint32_t)(ey + 127) << 23);
        const float iaa = __uint_as_float((uint32_t)(127 - 2 * ea) << 23), iay = __uint_as_float((uint32_t)(127 - ea - ey) << 23);
        if (b == 0) iaa_0 = iaa, iay_0 = iay;
        else if (b == 1) iaa_1 = iaa, iay_1 = iay;
        else iaa_2 = iaa, iay_2 = iay;
        const float sqk0 = sqrt_approx_tc(wbuf[st * kKC + k]), sqk1 = sqrt_approx_tc(wbuf[st * kKC + k + 4]);
        const float sa0 = sqk0 * scl_a, sa1 = sqk1 * scl_a, sy0 = sqk0 * scl_y, sy1 = sqk1 * scl_y;
        auto put = [&](int rg, float v0, float v1) {
          const __half2 hi = __floats2half2_rn(v0, v1);
          const float2 hf = __half22float2(hi);
          const __half2 lo = __floats2half2_rn(v0 - hf.x, v1 - hf.y);
          reinterpret_cast<__half2*>(hi_buf)[rg * (kKCores * kCoreWords) + word0] = hi;
          reinterpret_cast<__half2*>(lo_buf)[rg * (kKCores * kCoreWords) + word0] = lo;
        };
        if constexpr (M % 2 == 0) {
          // Window element e of frame k + 4 is element e + 4 M of frame k: row group rg of the later frame is row
          // group rg + M / 2 of the earlier one. One run of loads (issued together, ahead of the stores the compiler
          // cannot move them across) serves both frames.
          constexpr int SH = M / 2, NX = 10 + SH;  // km <= 80: at most 10 row groups per part
          auto part = [&](const float* src, int rg0) {
            float x[NX];
#pragma unroll
            for (int i = 0; i < NX; ++i) x[i] = i < nrg_a + SH ? src[i * 8] : 0.f;
#pragma unroll
            for (int rg = 0; rg < 10; ++rg)
              if (rg < nrg_a) put(rg0 + rg, x[rg] * sa0, x[rg + SH] * sa1);
          };
          part(rk, 0);       // Re a
          part(ik, nrg_a);   // Im a
        } else {
#pragma unroll
          for (int rg = 0; rg < 20; ++rg) {
            if (rg < 2 * nrg_a) {
              const float* src = rg < nrg_a ? rk + rg * 8 : ik + (rg - nrg_a) * 8;
              put(rg, src[0] * sa0, src[4 * M] * sa1);
            }
          }
        }
        put(2 * nrg_a, rk[H * M] * sy0, rk[H * M + 4 * M] * sy1);      // Re y (rows >= M are never read back)
        put(2 * nrg_a + 1, ik[H * M] * sy0, ik[H * M + 4 * M] * sy1);  // Im y
      } else {
        const float sq = sqrt_approx_tc(wbuf[st * kKC + k]);
#pragma unroll
        for (int rg = 0; rg < 24; ++rg) {  // NB <= 192 rows
          if (rg < nrg) {
            // (loading every row group's value ahead of the stores was measured: 8.74 against 8.32 ms at M = 4)
            float v;
            if (rg < nrg_a) v = rk[rg * 8];                              // Re a: element rg*8 + r8 of the window
            else if (rg < 2 * nrg_a) v = ik[(rg - nrg_a) * 8];           // Im a
            else if (rg == 2 * nrg_a) v = rk[H * M];                     // Re y (rows >= M are never read back)
            else if (rg == 2 * nrg_a + 1) v = ik[H * M];                 // Im y
            else v = 0.f;
            v *= sq;
            const float hi = __uint_as_float(__float_as_uint(v) & 0xffffe000u);
            hi_buf[rg * (kKCores * kCoreWords) + word0] = hi;
            lo_buf[rg * (kKCores * kCoreWords) + word0] = v - hi;
          }
        }
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic-proxy stores -> tensor core reads
      __syncwarp();
      if (lane == 0) mbar_arrive(&full[b]);
    }
    // fold in the last NS chunks
    for (int c = max(0, nchunk - NS); c < nchunk; ++c) {
      mbar_wait(&done[c % NS], (uint32_t)((c / NS) & 1));
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      drain(c % NS);
    }
    float* out = a.gram_raw + (sd.wcell_off + (long long)f) * (long long)(128 * NCT) +
                 (long long)(q * 32 + lane) * NCT + qcol;
#pragma unroll
    for (int j = 0; j < kAccPerThread / 4; ++j)
      if (j * 4 < NCQ)
        reinterpret_cast<float4*>(out)[j] = make_float4(acc[4 * j], acc[4 * j + 1], acc[4 * j + 2], acc[4 * j + 3]);
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  }
  __syncthreads();
  if (warp == kTcWorkerWarps) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(512u) : "memory");
  }
}

// ---------------------------------------------------------------------------
int wpe_tc_supported(int km, int M) {
  // accumulator columns per thread come in groups of 8 (tcgen05.ld x8) and must fit the register tile
  return tc_cols(km, M) <= 4 * kAccPerThread && (tc_cols(km, M) / 4) % 8 == 0 ? 1 : 0;
}
int wpe_tc_cell_floats(int km, int M) { return 128 * tc_cols(km, M); }
int wpe_tc_rows(int km, int M) { return tc_rows(km, M); }

template <int M, int TAPS, int F16>
static cudaError_t launch_tc_k(const WpeArgs& a, int nseg, int F, size_t smem, cudaStream_t st) {
  cudaError_t e = cudaFuncSetAttribute(wpe_gram_tc_kernel<M, TAPS, F16>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  wpe_gram_tc_kernel<M, TAPS, F16><<<dim3(F, nseg), kTcThreads, smem, st>>>(a);
  return cudaGetLastError();
}

template <int M>
static cudaError_t launch_tc_m(const WpeArgs& a, int nseg, int F, cudaStream_t st) {
  const int km = a.taps * M, H = a.delay + a.taps - 1;
  // the FP16 kind stages twice the frames: a long history that no longer fits runs the TF32 kind
  int f16 = a.gram_f16;
  if (f16 && tc_smem_bytes(km, M, H, 2, tc_kc(1)) > 224 * 1024) f16 = 0;
  const int kc = tc_kc(f16);
  size_t smem = tc_smem_bytes(km, M, H, tc_stages(km, M, H, kc), kc);
  if (smem > 224 * 1024) return cudaErrorInvalidConfiguration;
  // all 512 tensor-memory columns belong to one CTA: keep a second CTA off the SM
  smem = std::max<size_t>(smem, 120 * 1024);
  if (a.taps == 10) return f16 ? launch_tc_k<M, 10, 1>(a, nseg, F, smem, st) : launch_tc_k<M, 10, 0>(a, nseg, F, smem, st);
  return f16 ? launch_tc_k<M, 0, 1>(a, nseg, F, smem, st) : launch_tc_k<M, 0, 0>(a, nseg, F, smem, st);
}

cudaError_t launch_wpe_gram_tc(const WpeArgs& a, int nseg, int F, cudaStream_t st) {
  switch (a.M) {
    case 1: return launch_tc_m<1>(a, nseg, F, st);
    case 2: return launch_tc_m<2>(a, nseg, F, st);
    case 3: return launch_tc_m<3>(a, nseg, F, st);
    case 4: return launch_tc_m<4>(a, nseg, F, st);
    case 5: return launch_tc_m<5>(a, nseg, F, st);
    case 6: return launch_tc_m<6>(a, nseg, F, st);
    case 7: return launch_tc_m<7>(a, nseg, F, st);
    case 8: return launch_tc_m<8>(a, nseg, F, st);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace gssb
