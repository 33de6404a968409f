// cacgmm_kernels.cuh -- cACGMM EM kernels (templates; instantiated per channel
// count in cacgmm_m*.cu) and the MVDR statistics kernels that share the same
// Hermitian outer-product machinery.
//
// Reference semantics: cacgmm.hpp:264-340 (em_fit), :124-152 (invert_shapes),
// :156-174 (quad_forms), :189-257 (estep_bin), wpe.hpp:124-140 (unit_normalize),
// numerics.hpp:128-152 (weighted_gram), beamform.hpp:35-85 (accumulate_stats).
//
// One EM iteration = em_pass_kernel (E-step + M-step accumulation fused in one
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

/// How the 32 lanes of a warp map to (frame slot, lane-in-frame g) and the shared-memory frame stride
/// (float2 units), chosen by brute force over the bank model so that the per-lane frame loads of
/// FramePlan::dofs are (nearly) conflict free:
///   SPREAD (L <= 4): g = lane / (32/L), slot = lane % (32/L)  -- the L lanes of a frame are 32/L apart
///   else           : g = lane % L,      slot = lane / L
template <int M, int L>
struct LaneMap {
  static constexpr bool SPREAD = L <= 4;
  static constexpr int SPW = 32 / L;  // frame slots per warp
  static constexpr int STRIDE = !SPREAD ? M
                                : L == 4 ? (M == 7 ? 10 : M == 8 ? 10 : M)
                                         : (M == 8 ? 9 : M == 6 ? 7 : M == 4 ? 5 : M == 2 ? 3 : M);
  __device__ static __forceinline__ int g_of(int lane) { return SPREAD ? lane / SPW : lane % L; }
  __device__ static __forceinline__ int slot_of(int lane) { return SPREAD ? lane % SPW : lane / L; }
  /// xor offsets that stay inside a frame's lane group / that walk over the slots of a warp
  static constexpr int G_LO = SPREAD ? SPW : 1, G_HI = SPREAD ? 32 : L;
  static constexpr int S_LO = SPREAD ? 1 : L, S_HI = SPREAD ? SPW : 32;
  __device__ static __forceinline__ int lane_of_g(int g) { return SPREAD ? g * SPW : g; }
};

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
  float rowmask[Lay::RPL];

  __device__ __forceinline__ void init(int g) {
#pragma unroll
    for (int i = 0; i < Lay::RPL; ++i) {
      int row = g + i * L;
      rowmask[i] = row < M ? 1.f : 0.f;
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

  /// |y|^2 of the frame from this lane's diagonal dofs (sum over the L lanes).
  __device__ __forceinline__ float norm2(const float (&pv)[Lay::NDOF]) const {
    float s = 0.f;
#pragma unroll
    for (int i = 0; i < Lay::RPL; ++i) s = fmaf(rowmask[i], pv[i * M], s);
#pragma unroll
    for (int o = LaneMap<M, L>::G_LO; o < LaneMap<M, L>::G_HI; o <<= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    return s;
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

// Packed FP32 pairs (Blackwell FFMA2): one issue slot for two fused multiply-adds, each rounded exactly like
// a scalar fma.rn, so results are bit-identical to the scalar form.
typedef unsigned long long f32x2;
__device__ __forceinline__ f32x2 pack2(float a, float b) {
  f32x2 r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ void unpack2(f32x2 v, float& a, float& b) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(v));
}
__device__ __forceinline__ f32x2 ffma2(f32x2 a, f32x2 b, f32x2 c) {
  f32x2 d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}

__device__ __forceinline__ void cp_async8(void* smem_dst, const void* gsrc) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(smem_dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(d), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

// ---------------------------------------------------------------------------
// E-step + accumulation sweep. grid = (work items, F), block = 256.
// L lanes share a frame; each owns NDOF dofs of P = y y^H, the matching slice
// of every class's B^-1 (registers) and of every accumulator. Frames stream
// through a two-stage cp.async pipeline in shared memory.
//   FINAL = false: accumulators are the KT M-step Grams (weights gamma/q).
//   FINAL = true : accumulators are the MVDR target / background Grams.
// ---------------------------------------------------------------------------
/// B^-1 coefficients live in shared memory ([lane g][class][NDOFP], NDOFP = NDOF rounded up to 4 so a
/// lane fetches them as float4); that keeps the register tile to the accumulators and lets two CTAs
/// share an SM when the accumulators are small enough.
/// Sweep flavours: kSweepEM accumulates the M-step Grams; kSweepEMGamma does the same and may also store
/// the posteriors (last sweep of the stage entry point); kSweepFinal accumulates the MVDR statistics and
/// may store the posteriors (last sweep of enhance_batch).
enum SweepMode { kSweepEM = 0, kSweepEMGamma = 1, kSweepFinal = 2 };

template <int M, int L, int KT, bool FINAL>
struct EmPassCfg {
  static constexpr int NDOF = EmLayout<M, L>::NDOF;
  static constexpr int NDOFP = (NDOF + 3) & ~3;
  static constexpr int NA = FINAL ? 2 : KT;
  static constexpr int MINB = (NA * NDOF <= 64) ? 2 : 1;
  static constexpr int COEF_G = KT * NDOFP + 4;  // per-lane-group stride, skewed by one float4 against bank conflicts
  static constexpr int COEF_FLOATS = L * COEF_G;
  static constexpr int FS = LaneMap<M, L>::STRIDE;  // frame stride in the pipeline buffers
};

template <int M, int L, int KT, int MODE>
__global__ void __launch_bounds__(kEmThreads, EmPassCfg<M, L, KT, MODE == kSweepFinal>::MINB)
    em_pass_kernel(EmPassArgs a) {
  constexpr bool FINAL = MODE == kSweepFinal;
  using Lay = EmLayout<M, L>;
  using Cfg = EmPassCfg<M, L, KT, FINAL>;
  constexpr int NA = FINAL ? 2 : KT;
  using PL = PartLayout<M, L, KT, NA>;
  constexpr int NDOF = Lay::NDOF;
  constexpr int NDOFP = Cfg::NDOFP;
  constexpr int SLOTS = kEmThreads / L;
  constexpr int TILE = kEmTileFrames;
  constexpr int NW = kEmThreads / 32;
  extern __shared__ float4 smem_f4[];
  using LM = LaneMap<M, L>;
  constexpr int FS = Cfg::FS;
  float2* slab = reinterpret_cast<float2*>(smem_f4);                 // 2 * TILE * FS
  float* s_coef = reinterpret_cast<float*>(slab + 2 * TILE * FS);    // COEF_FLOATS (16-byte aligned)
  float* s_ck = s_coef + Cfg::COEF_FLOATS;                           // npat_max * KT
  unsigned char* s_pat = reinterpret_cast<unsigned char*>(s_ck + a.npat_max * KT);  // 2 * TILE
  unsigned char* s_amask = s_pat + 2 * TILE;                                        // npat_max: active classes

  const int tid = threadIdx.x;
  const WorkItem wi = a.work[blockIdx.x];
  const int f = blockIdx.y;
  const SegDev sd = a.segs[wi.seg];
  const int t0 = wi.chunk * sd.TC;
  const int nt = min(sd.TC, sd.T - t0);
  const int ntiles = (nt + TILE - 1) / TILE;
  const float2* src = a.y + sd.y_off + ((long long)f * sd.T + t0) * M;
  const unsigned char* psrc = a.pat + sd.pat_off + t0;

  auto issue_tile = [&](int tile, int buf) {
    const int n = min(TILE, nt - tile * TILE) * M;
    const float2* s = src + (long long)tile * TILE * M;
    float2* d = slab + buf * TILE * FS;
    for (int i = tid; i < n; i += kEmThreads) cp_async8(d + (FS == M ? i : (i / M) * FS + i % M), s + i);
    cp_async_commit();
  };

  issue_tile(0, 0);
  {
    const float* cks = a.ck + sd.tab_off + (long long)f * sd.npat * KT;
    for (int i = tid; i < sd.npat * KT; i += kEmThreads) s_ck[i] = cks[i];
    for (int i = tid; i < min(TILE, nt); i += kEmThreads) s_pat[i] = psrc[i];
    // classes that can be active under a pattern (finite constant); the others have gamma == 0 exactly
    for (int p = tid; p < sd.npat; p += kEmThreads) {
      unsigned m = 0;
      for (int k = 0; k < KT; ++k)
        if (cks[p * KT + k] != -CUDART_INF_F) m |= 1u << k;
      s_amask[p] = (unsigned char)m;
    }
  }

  const int lane = tid & 31, warp = tid >> 5;
  const int g = LM::g_of(lane), slot = warp * LM::SPW + LM::slot_of(lane);
  {
    const float* cp = a.coef + sd.coef_off + (long long)f * L * (KT * NDOF);
    for (int i = tid; i < L * KT * NDOFP; i += kEmThreads) {
      const int j = i % NDOFP, gk = i / NDOFP;
      s_coef[(gk / KT) * Cfg::COEF_G + (gk % KT) * NDOFP + j] = j < NDOF ? cp[gk * NDOF + j] : 0.f;
    }
  }
  const ulonglong2* c4 = reinterpret_cast<const ulonglong2*>(s_coef + g * Cfg::COEF_G);
  constexpr int NP = NDOF / 2;            // packed pairs of dofs
  constexpr bool ODD = (NDOF & 1) != 0;   // + one scalar dof
  f32x2 acc2[NA][NP > 0 ? NP : 1];
  float acc1[NA];
  float mass[KT];
#pragma unroll
  for (int k = 0; k < KT; ++k) mass[k] = 0.f;
#pragma unroll
  for (int n = 0; n < NA; ++n) {
    acc1[n] = 0.f;
#pragma unroll
    for (int j = 0; j < NP; ++j) acc2[n][j] = 0ull;
  }
  double ll = 0.0;
  FramePlan<M, L> plan;
  plan.init(g);
  float* gout = MODE != kSweepEM && a.gamma != nullptr && sd.g_off >= 0
                    ? a.gamma + sd.g_off + ((long long)f * sd.T + t0) * sd.K
                    : nullptr;
  const int target = sd.target;
  const bool normalize = a.normalize != 0;

  for (int tile = 0; tile < ntiles; ++tile) {
    const int buf = tile & 1;
    // prefetch the next tile (data by cp.async, pattern ids through registers)
    unsigned char pnext[TILE / kEmThreads];
    const bool more = tile + 1 < ntiles;
    if (more) {
      issue_tile(tile + 1, buf ^ 1);
      const int nn = min(TILE, nt - (tile + 1) * TILE);
#pragma unroll
      for (int i = 0; i < TILE / kEmThreads; ++i) {
        const int idx = tid + i * kEmThreads;
        pnext[i] = idx < nn ? psrc[(tile + 1) * TILE + idx] : (unsigned char)0;
      }
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    const int nin = min(TILE, nt - tile * TILE);
    const float2* sl = slab + buf * TILE * FS;
    const unsigned char* sp = s_pat + buf * TILE;
    // The activity pattern of an iteration's frames (and the classes it can activate) is fetched one
    // iteration ahead: the LDS -> LDS -> REDUX chain is off the critical path.
    int pid_n = (int)sp[min(slot, nin - 1)];
    unsigned am_n = __reduce_or_sync(0xffffffffu, (unsigned)s_amask[pid_n]);
    float llf = 0.f;  // this tile's log-likelihood terms (<= TILE / SLOTS of them) in float, folded into ll per tile
#pragma unroll 1
    for (int fb = slot; fb < TILE; fb += SLOTS) {
      if (fb - slot >= nin) break;  // whole stripe of slots is past the data (block-uniform per warp row)
      const bool valid = fb < nin;
      const int fbc = valid ? fb : nin - 1;
      const int pid = pid_n;
      const unsigned am = am_n;
      {
        const int fbn = min(fb + SLOTS, nin - 1);
        pid_n = (int)sp[fbn];
        am_n = __reduce_or_sync(0xffffffffu, (unsigned)s_amask[pid_n]);
      }
      float pv[NDOF];
      plan.dofs(sl + fbc * FS, pv);
      f32x2 pv2[NP > 0 ? NP : 1];
#pragma unroll
      for (int j = 0; j < NP; ++j) pv2[j] = pack2(pv[2 * j], pv[2 * j + 1]);
      // Classes that are inactive for every frame this warp holds are skipped (warp-uniform branches):
      // speakers talk in long runs, so a warp's frames usually share one activity pattern.
      float q[KT];
#pragma unroll
      for (int k = 0; k < KT; ++k) {
        if (am & (1u << k)) {
          // even dofs accumulate in the low half, odd dofs in the high half (two chains)
          f32x2 s2 = 0ull;
          float s1 = 0.f;
#pragma unroll
          for (int j4 = 0; j4 < NDOFP / 4; ++j4) {
            const ulonglong2 c = c4[k * (NDOFP / 4) + j4];
            if (2 * j4 < NP) s2 = ffma2(c.x, pv2[2 * j4 < NP ? 2 * j4 : 0], s2);
            if (2 * j4 + 1 < NP) s2 = ffma2(c.y, pv2[2 * j4 + 1 < NP ? 2 * j4 + 1 : 0], s2);
            if (ODD && (NDOF - 1) / 4 == j4) {  // the scalar tail dof sits in this quad
              float c0, c1;
              unpack2(((NDOF - 1) & 2) ? c.y : c.x, c0, c1);
              s1 = c0 * pv[NDOF - 1];
            }
          }
          float sa, sb;
          unpack2(s2, sa, sb);
          q[k] = NP > 0 ? (sa + sb) + s1 : s1;
        } else {
          q[k] = 0.f;  // its constant is -inf: the posterior is exactly 0 whatever q is (floored below)
        }
      }
      // One joint butterfly over the frame's L lanes for |y|^2 and every class's partial quadratic form:
      // the KT + 1 shuffles of a stage are independent, so their latencies overlap.
      float n2 = 0.f;
      if (normalize) {
#pragma unroll
        for (int i = 0; i < Lay::RPL; ++i) n2 = fmaf(plan.rowmask[i], pv[i * M], n2);
      }
#pragma unroll
      for (int o = LM::G_LO; o < LM::G_HI; o <<= 1) {
        if (normalize) n2 += __shfl_xor_sync(0xffffffffu, n2, o);
#pragma unroll
        for (int k = 0; k < KT; ++k) q[k] += __shfl_xor_sync(0xffffffffu, q[k], o);
      }
      // Unit normalisation y/(|y|+1e-10) (wpe.hpp:135) scales every class's quadratic form by the same
      // s^2 = 1/nr2, which cancels in the posteriors and in gamma/q * s^2; only the floor and the likelihood
      // see it: max(q_raw s^2, 1e-10) = s^2 max(q_raw, 1e-10 nr2).
      float nr2 = 1.f;
      if (normalize) {
        const float nr = sqrt_approx(n2) + 1e-10f;
        nr2 = nr * nr;
      }
      const float qfloor = kQuadFloor * nr2;

      const float* ckp = s_ck + pid * KT;
      float u[KT];
      float mx = -CUDART_INF_F;
#pragma unroll
      for (int k = 0; k < KT; ++k) {
        q[k] = fmaxf(q[k], qfloor);                           // cacgmm.hpp:170-171, in raw units
        // log2 domain: the table holds ck * log2(e); inactive classes carry ck = -inf
        u[k] = fmaf(-(float)M, lg2_approx(q[k]), ckp[k]);
        mx = fmaxf(mx, u[k]);
      }
      float se = 0.f;
#pragma unroll
      for (int k = 0; k < KT; ++k) {
        u[k] = ex2_approx(u[k] - mx);
        se += u[k];
      }
      const float rinv = valid ? rcp_approx(se) : 0.f;
      // log2 units, scaled once at the end; the common s^2 factor comes back here: -M log2(s^2) = +M log2(nr2)
      if (valid && g == 0) llf += mx + lg2_approx(se) + (float)M * lg2_approx(nr2);
      float gam[KT];
#pragma unroll
      for (int k = 0; k < KT; ++k) {
        gam[k] = u[k] * rinv;  // exactly 0 for inactive classes
        mass[k] += gam[k];
        if (MODE != kSweepEM) {
          if (gout != nullptr && valid && (k % L) == g && k < sd.K)
            gout[(long long)(tile * TILE + fb) * sd.K + k] = gam[k];
        }
      }
      if (FINAL) {
        float wt = 0.f, wb = 0.f;
#pragma unroll
        for (int k = 0; k < KT; ++k) {
          wt += (k == target) ? gam[k] : 0.f;
          wb += (k == target) ? 0.f : gam[k];
        }
        const f32x2 wt2 = pack2(wt, wt), wb2 = pack2(wb, wb);
#pragma unroll
        for (int j = 0; j < NP; ++j) {
          acc2[0][j] = ffma2(wt2, pv2[j], acc2[0][j]);
          acc2[NA - 1][j] = ffma2(wb2, pv2[j], acc2[NA - 1][j]);
        }
        if (ODD) {
          acc1[0] = fmaf(wt, pv[NDOF - 1], acc1[0]);
          acc1[NA - 1] = fmaf(wb, pv[NDOF - 1], acc1[NA - 1]);
        }
      } else {
#pragma unroll
        for (int k = 0; k < NA; ++k) {
          if (am & (1u << k)) {
            const float w = gam[k] * rcp_approx(q[k]);  // (gamma / q s^2) on the raw frame
            const f32x2 w2 = pack2(w, w);
#pragma unroll
            for (int j = 0; j < NP; ++j) acc2[k][j] = ffma2(w2, pv2[j], acc2[k][j]);
            if (ODD) acc1[k] = fmaf(w, pv[NDOF - 1], acc1[k]);
          }
        }
      }
    }
    ll += (double)llf;
    __syncthreads();  // everyone is done with buffer `buf` (and with s_pat[buf])
    if (more) {
#pragma unroll
      for (int i = 0; i < TILE / kEmThreads; ++i) s_pat[(buf ^ 1) * TILE + tid + i * kEmThreads] = pnext[i];
    }
  }

  // ---- reduce: frame slots within the warp, then warps through shared memory
  ll = g != 0 ? 0.0 : ll * 0.69314718055994530942;  // back to natural-log units
  float acc[NA][NDOF];
#pragma unroll
  for (int n = 0; n < NA; ++n) {
#pragma unroll
    for (int j = 0; j < NP; ++j) unpack2(acc2[n][j], acc[n][2 * j], acc[n][2 * j + 1]);
    if (ODD) acc[n][NDOF - 1] = acc1[n];
  }
#pragma unroll
  for (int o = LM::S_LO; o < LM::S_HI; o <<= 1) {
#pragma unroll
    for (int k = 0; k < KT; ++k) mass[k] += __shfl_xor_sync(0xffffffffu, mass[k], o);
#pragma unroll
    for (int n = 0; n < NA; ++n)
#pragma unroll
      for (int j = 0; j < NDOF; ++j) acc[n][j] += __shfl_xor_sync(0xffffffffu, acc[n][j], o);
  }
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) ll += __shfl_xor_sync(0xffffffffu, ll, o);
  __syncthreads();  // pipeline buffers are free
  float* red = reinterpret_cast<float*>(smem_f4);
  double* redll = reinterpret_cast<double*>(red + NW * PL::CELL + (NW * PL::CELL & 1));
  if (LM::slot_of(lane) == 0) {
    float* r = red + (warp * L + g) * PL::STRIDE;
#pragma unroll
    for (int n = 0; n < NA; ++n)
#pragma unroll
      for (int j = 0; j < NDOF; ++j) r[n * NDOF + j] = acc[n][j];
#pragma unroll
    for (int k = 0; k < KT; ++k) r[PL::ACC + k] = mass[k];
  }
  if (lane == 0) redll[warp] = ll;
  __syncthreads();
  const long long cell = sd.cell_off + (long long)f * sd.nchunks + wi.chunk;
  float* out = a.part + cell * a.cell_stride;
  for (int i = tid; i < PL::CELL; i += kEmThreads) {
    float s = 0.f;
#pragma unroll
    for (int w = 0; w < NW; ++w) s += red[w * PL::CELL + i];
    out[i] = s;
  }
  if (tid == 0) {
    double s = 0.0;
#pragma unroll
    for (int w = 0; w < NW; ++w) s += redll[w];
    a.cell_ll[cell] = s;
  }
}

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

/// inv <- (L L^H)^-1, lane c solves column c (forward then backward substitution).
template <int M>
__device__ __forceinline__ void warp_cholesky_inverse(const cdbl* l, cdbl* inv, int lane) {
  if (lane < M) {
    const int c = lane;
    for (int i = 0; i < M; ++i) {
      cdbl s = cd_make(i == c ? 1.0 : 0.0, 0.0);
      for (int j = 0; j < i; ++j) s = cd_sub(s, cd_mul(l[i * M + j], inv[j * M + c]));
      inv[i * M + c] = cd_scale(s, 1.0 / l[i * M + i].re);
    }
    for (int i = M - 1; i >= 0; --i) {
      cdbl s = inv[i * M + c];
      for (int j = i + 1; j < M; ++j) s = cd_sub(s, cd_cmul(l[j * M + i], inv[j * M + c]));
      inv[i * M + c] = cd_scale(s, 1.0 / l[i * M + i].re);
    }
  }
  __syncwarp();
}

template <int M, int L, int KT>
__global__ void __launch_bounds__(KT * 32) em_update_kernel(EmUpdateArgs a) {
  using Lay = EmLayout<M, L>;
  using PL = PartLayout<M, L, KT, KT>;
  constexpr int NDOF = Lay::NDOF;
  constexpr int MM = M * M;
  __shared__ cdbl s_b[KT][MM], s_f[KT][MM], s_inv[KT][MM];
  __shared__ double s_pi[KT], s_ld[KT];

  const int k = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int f = blockIdx.x, seg = blockIdx.y;
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
      } else {
        // rare path, one lane: eigenvalue-floor fallback, then the retry on regularize(B)
        // (numerics.hpp:103-122, cacgmm.hpp:134-140)
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
