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
// 176 at M = 8) are covered by a second accumulator D2 = S[NR-128..NR) x S[128..NR)^T; symmetry gives the
// rest. FP32 accuracy comes from the split x = hi + lo (hi = top 19 bits): hi*hi + hi*lo + lo*hi.
//
// Pipeline per CTA (one (segment, bin), 256 threads): per chunk of 32 frames all warps expand the slab into
// the canonical no-swizzle K-major core-matrix layout (a warp store = one 8x16-byte core matrix, conflict
// free), fence to the async proxy, and one thread issues the chunk's MMAs and commits them to the
// buffer's mbarrier; the next chunk is expanded into the other buffer while the tensor core runs.
#include "kernels.h"

namespace gssb {

namespace {

constexpr int kTcThreads = 256;
constexpr int kTcWarps = kTcThreads / 32;
constexpr int kKC = 32;                     // frames per pipeline stage (4 MMA k-steps of 8)
constexpr int kCoreWords = 32;              // one core matrix: 8 rows x 16 bytes
constexpr int kKCores = kKC / 4;            // core matrices along K per row group

__host__ __device__ inline int tc_rows(int km, int M) { return ((2 * km + 2 * M + 15) / 16) * 16; }      // NR
__host__ __device__ inline int tc_buf_rows(int km, int M) { return tc_rows(km, M) < 128 ? 128 : tc_rows(km, M); }
__host__ __device__ inline int tc_n2(int km, int M) { return tc_rows(km, M) > 128 ? tc_rows(km, M) - 128 : 0; }
__host__ __device__ inline int tc_cols(int km, int M) { return tc_rows(km, M) + tc_n2(km, M); }         // D1 | D2

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
__device__ __forceinline__ uint32_t make_idesc_tf32(int n) {
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
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t"
      ".reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@p bra DONE_%=;\n\t"
      "bra WAIT_%=;\n\t"
      "DONE_%=:\n\t"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tc_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}

}  // namespace

template <int M>
__global__ void __launch_bounds__(kTcThreads, 2) wpe_gram_tc_kernel(WpeArgs a) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const SegDev sd = a.segs[blockIdx.y];
  if (!sd.wpe_active) return;
  const int f = blockIdx.x;
  const int taps = a.taps, km = taps * M, H = a.delay + taps - 1;
  const int NR = tc_rows(km, M), NB = tc_buf_rows(km, M), N2 = tc_n2(km, M), NCT = NR + N2;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

  // shared memory carve-up
  uint64_t* mbar = reinterpret_cast<uint64_t*>(smem_raw);             // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem_raw + 16);
  float2* slab = reinterpret_cast<float2*>(smem_raw + 128);           // (kKC + H) frames x M
  float* sqw = reinterpret_cast<float*>(slab + (kKC + H) * M);        // kKC
  const int buf_words = NB * kKC;                                     // one operand buffer (hi or lo)
  size_t off = 128 + sizeof(float2) * (size_t)(kKC + H) * M + sizeof(float) * kKC;
  off = (off + 127) & ~(size_t)127;
  float* opbuf = reinterpret_cast<float*>(smem_raw + off);            // [stage][hi/lo][buf_words]

  if (tid == 0) {
    mbar_init(&mbar[0], 1);
    mbar_init(&mbar[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  uint32_t tmem_cols = 32;
  while ((int)tmem_cols < NCT) tmem_cols <<= 1;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(tmem_cols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem_base = *tmem_slot;

  const float2* yf = a.yobs + sd.y_off + (long long)f * sd.T * M;
  const float* wf = a.w + sd.w_off + (long long)f * sd.T;
  const int nchunk = (sd.T + kKC - 1) / kKC;
  const uint32_t sbo = kKCores * 128, lbo = 128;
  const uint32_t idesc1 = make_idesc_tf32(NR), idesc2 = make_idesc_tf32(N2 > 0 ? N2 : 16);

  for (int c = 0; c < nchunk; ++c) {
    const int b = c & 1;
    const int t0 = c * kKC;
    if (c >= 2) mbar_wait(&mbar[b], (uint32_t)((c / 2 - 1) & 1));  // MMAs of chunk c-2 released this buffer
    // slab: frames [t0 - H, t0 + kKC), zero outside [0, T) (wpe.hpp:74-75); sqrt of the Gram weights
    for (int i = tid; i < (kKC + H) * M; i += kTcThreads) {
      const int fr = i / M;
      const int t = t0 - H + fr;
      slab[i] = (t >= 0 && t < sd.T) ? yf[(long long)t * M + (i - fr * M)] : make_float2(0.f, 0.f);
    }
    if (tid < kKC) sqw[tid] = t0 + tid < sd.T ? sqrtf(wf[t0 + tid]) : 0.f;
    __syncthreads();
    // expand: core matrix (row group rg, k chunk kc) <- lane (row rg*8 + lane/4, frame kc*4 + lane%4)
    float* hi_buf = opbuf + (size_t)(2 * b) * buf_words;
    float* lo_buf = hi_buf + buf_words;
    const int ncores = (NB / 8) * kKCores;
    for (int core = warp; core < ncores; core += kTcWarps) {
      const int rg = core / kKCores, kc = core - rg * kKCores;
      const int r = rg * 8 + (lane >> 2), k = kc * 4 + (lane & 3);
      float v = 0.f;
      if (r < 2 * km) {
        const int e = r < km ? r : r - km;
        const float2 y = slab[(k + e / M) * M + e % M];
        v = r < km ? y.x : y.y;
      } else if (r < 2 * km + 2 * M) {
        const int cc = r - 2 * km;
        const float2 y = slab[(k + H) * M + (cc < M ? cc : cc - M)];
        v = cc < M ? y.x : y.y;
      }
      v *= sqw[k];
      const float hi = __uint_as_float(__float_as_uint(v) & 0xffffe000u);
      hi_buf[core * kCoreWords + lane] = hi;
      lo_buf[core * kCoreWords + lane] = v - hi;
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic-proxy stores -> tensor core reads
    __syncthreads();
    if (tid == 0) {
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint32_t a_hi = smem_u32(hi_buf), a_lo = smem_u32(lo_buf);
#pragma unroll
      for (int ks = 0; ks < kKC / 8; ++ks) {
        const uint32_t acc = (c > 0 || ks > 0) ? 1u : 0u;
        const uint32_t ko = ks * 256;  // two core matrices along K per MMA
        const uint64_t dh = make_smem_desc(a_hi + ko, lbo, sbo), dl = make_smem_desc(a_lo + ko, lbo, sbo);
        mma_tf32(tmem_base, dh, dh, idesc1, acc);
        mma_tf32(tmem_base, dh, dl, idesc1, 1u);
        mma_tf32(tmem_base, dl, dh, idesc1, 1u);
        if (N2 > 0) {
          const uint32_t ra = ((NR - 128) / 8) * sbo, rb = 16 * sbo;  // rows NR-128.. and rows 128..
          const uint64_t ah = make_smem_desc(a_hi + ra + ko, lbo, sbo), al = make_smem_desc(a_lo + ra + ko, lbo, sbo);
          const uint64_t bh = make_smem_desc(a_hi + rb + ko, lbo, sbo), bl = make_smem_desc(a_lo + rb + ko, lbo, sbo);
          mma_tf32(tmem_base + NR, ah, bh, idesc2, acc);
          mma_tf32(tmem_base + NR, ah, bl, idesc2, 1u);
          mma_tf32(tmem_base + NR, al, bh, idesc2, 1u);
        }
      }
      tc_commit(&mbar[b]);
    }
    // no barrier here: the next chunk only touches the slab (free after the sync above) and the other buffer
  }
  // drain: the last use of each buffer
  for (int b = 0; b < 2; ++b) {
    const int uses = (nchunk - b + 1) / 2;
    if (uses > 0) mbar_wait(&mbar[b], (uint32_t)((uses - 1) & 1));
  }
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");

  // epilogue: thread i of warps 0..3 owns accumulator row i (tensor-memory lane i)
  float* out = a.gram_raw + (sd.wcell_off + (long long)f) * (long long)(128 * NCT);
  if (warp < 4) {
    const int row = warp * 32 + lane;
    for (int c0 = 0; c0 < NCT; c0 += 16) {
      uint32_t v[16];
      const uint32_t taddr = tmem_base + ((uint32_t)(warp * 32) << 16) + (uint32_t)c0;
      asm volatile(
          "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
          "%15}, [%16];"
          : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
            "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
          : "r"(taddr)
          : "memory");
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      float4* o4 = reinterpret_cast<float4*>(out + (long long)row * NCT + c0);
#pragma unroll
      for (int j = 0; j < 4; ++j)
        o4[j] = make_float4(__uint_as_float(v[4 * j]), __uint_as_float(v[4 * j + 1]), __uint_as_float(v[4 * j + 2]),
                            __uint_as_float(v[4 * j + 3]));
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(tmem_cols) : "memory");
  }
}

// ---------------------------------------------------------------------------
int wpe_tc_supported(int km, int M) { return tc_rows(km, M) <= 256 && tc_cols(km, M) <= 512 ? 1 : 0; }
int wpe_tc_cell_floats(int km, int M) { return 128 * tc_cols(km, M); }
int wpe_tc_rows(int km, int M) { return tc_rows(km, M); }

template <int M>
static cudaError_t launch_tc_m(const WpeArgs& a, int nseg, int F, cudaStream_t st) {
  const int km = a.taps * M, H = a.delay + a.taps - 1;
  size_t off = 128 + sizeof(float2) * (size_t)(kKC + H) * M + sizeof(float) * kKC;
  off = (off + 127) & ~(size_t)127;
  const size_t smem = off + sizeof(float) * 4 * (size_t)tc_buf_rows(km, M) * kKC;
  if (smem > 110 * 1024) return cudaErrorInvalidConfiguration;
  cudaError_t e = cudaFuncSetAttribute(wpe_gram_tc_kernel<M>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  wpe_gram_tc_kernel<M><<<dim3(F, nseg), kTcThreads, smem, st>>>(a);
  return cudaGetLastError();
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
