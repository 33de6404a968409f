// cacgmm_pass2.cuh -- the cACGMM sweep (E-step + M-step / MVDR accumulation), second design.
//
// Reference semantics: cacgmm.hpp:156-174 (quad_forms), :189-257 (estep_bin), :308-329 (M-step Gram),
// wpe.hpp:124-140 (unit_normalize, folded in), beamform.hpp:35-85 (accumulate_stats, last sweep).
//
// Why two phases. The first sweep of this repository gave every frame to L lanes for the whole iteration;
// each of them repeated the frame's soft-max, pattern lookup and loop control, and at M = 7, K = 4 only 46 %
// of its issued instructions were FP32 math (25.0 ms per cfg2 step against 16.3 ms for this one; DESIGN.md
// section 3). Here a warp works on groups of 32 frames in two phases with different lane maps:
//
//   phase A  lane = frame. The lane forms the M^2 Hermitian degrees of freedom ("dofs") of P = y y^H once,
//            feeds each into the K quadratic forms (coefficients are warp-uniform shared-memory broadcasts),
//            runs the guide-masked soft-max ONCE per frame without any shuffle, and parks the dofs (float4
//            chunks, XOR-swizzled) and the K accumulation weights in the warp's shared-memory scratch.
//   phase B  lane = (frame slot, dof slice g of L), the register layout of the accumulators (em_layout.cuh).
//            Per frame a lane fetches its NDOF dofs as float4s and the weights, and does K * NDOF FMAs.
//
// No block-wide barrier in the main loop: each warp streams its own groups of frames (one contiguous run of
// 32 * M * 8 bytes) through a private two-stage cp.async buffer, and the scratch is private to the warp.
// Cells (PartLayout) are what em_update_kernel and mvdr_stats_final_kernel read.
#pragma once

#include "cacgmm_kernels.cuh"

namespace gssb {

constexpr int pow2_ceil(int x) {
  int p = 1;
  while (p < x) p <<= 1;
  return p;
}

/// 8-byte async copy; `valid == false` writes zeros without reading the source (src-size 0).
__device__ __forceinline__ void cp_async8_zfill(void* smem_dst, const void* gsrc, bool valid) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(smem_dst);
  const int n = valid ? 8 : 0;
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(d), "l"(gsrc), "r"(n) : "memory");
}

template <int M, int L, int KT, bool FINAL>
struct EmPass2Cfg {
  using Lay = EmLayout<M, L>;
  static constexpr int NDOF = Lay::NDOF;
  static constexpr int NDOFP = (NDOF + 3) & ~3;
  static constexpr int CPG = NDOFP / 4;            // float4 chunks per lane slice g
  static constexpr int NCH = L * CPG;              // chunks per frame
  static constexpr int NCHP = pow2_ceil(NCH);      // frame stride of the dof scratch (float4 units)
  static constexpr int KTP = KT <= 2 ? 2 : KT <= 4 ? 4 : 8;  // padded class count of the tables
  static constexpr int NA = FINAL ? 2 : KT;
  static constexpr int WS = FINAL ? 2 : KTP;       // weights parked per frame
  static constexpr int SPW = 32 / L;               // frames per phase-B step
  /// Column swizzle of the dof scratch. SPW >= 8: a phase-B quarter-warp is 8 frames of one slice, the identity
  /// does it. SPW = 4 (L = 8): a quarter-warp is 4 frames x 2 slices whose chunk numbers differ in bit 1 (CPG = 2),
  /// so the frame's bit 1 must land elsewhere: bits (0, 1, 2) -> (0, 2, 1). With the identity these loads were
  /// 2-way conflicted (41 M conflict cycles per cfg3 sweep).
  static constexpr int FPL = NCHP < 8 ? 8 / NCHP : 1;  // frames per 128-byte line of a narrow scratch
  __host__ __device__ static constexpr unsigned swz(unsigned fr) {
    if (L == 8 && NDOFP == 8) return ((fr & 1u) | ((fr & 2u) << 1) | ((fr & 4u) >> 1) | (fr & ~7u)) & (unsigned)(NCHP - 1);
    // narrow scratch rows (NCHP < 8: M <= 4): 8 / NCHP frames share one 128-byte line, and the 8 frames of a
    // quarter-warp must land in 8 different 16-byte columns of it, so the XOR term advances once per line, not
    // once per frame (with fr % NCHP, frames fr and fr + NCHP collided: 29 % excess wavefronts at M = 4)
    if (NCHP < 8) return (fr / (unsigned)FPL) & (unsigned)(NCHP - 1);
    return fr & (unsigned)(NCHP - 1);
  }
  static constexpr int NW = kEmThreads / 32;
  // coefficient table of one lane slice: [dof][class] packed (no class padding), rounded up to whole float4s
  static constexpr int CS = NDOFP * KT;  // NDOFP is a multiple of 4
  static constexpr int COEF_FLOATS = L * CS;
  // one group of frames (cp.async landing zone). Frame stride in float2 units: odd, so that the 16 lanes of a
  // half-warp reading channel m of their own frame (LDS.64) fall into 16 different bank pairs. With the natural
  // stride M = 8 they fell into two (8-way conflict: 72 M conflict cycles per cfg3 sweep, profiles/ncu_full_r02.md)
  static constexpr int SY = (M % 2 == 0) ? M + 1 : M;
  static constexpr int YSTAGE_FLOATS = 32 * SY * 2;
  // per warp: dof scratch [32][NCHP] float4 | weights [32][WS] | frame landing zone | sums; a multiple of 256 bytes
  static constexpr int SUMS = KT + 1;  // per frame lane: class masses and the log-likelihood, kept out of registers
  // ONE landing zone: a group's frames are in registers a few instructions into its turn, and the next group's copy
  // is issued into the same zone right after (it has the whole turn to land). A second zone cost 18 KB per block
  // and, at M = 8, the second resident block with it.
  static constexpr int WARP_SCRATCH_FLOATS = (32 * NCHP * 4 + 32 * WS + YSTAGE_FLOATS + 32 * SUMS + 63) & ~63;
  // epilogue dump: every thread parks its accumulators, stride chosen odd in float4 units (conflict-free)
  static constexpr int DUMP_STRIDE = ((NA * NDOF + 3) / 4 | 1) * 4;
  // accumulators + two groups of frames in flight must fit the register file at this occupancy
#ifdef GSS_EXP_MINB
  static constexpr int MINB = GSS_EXP_MINB;
#else
  static constexpr int MINB = (NA * NDOF + 4 * M <= 88) ? 2 : 1;
#endif
};

template <int M, int L, int KT, int MODE>
__global__ void __launch_bounds__(kEmThreads, EmPass2Cfg<M, L, KT, MODE == kSweepFinal>::MINB)
    em_pass2_kernel(EmPassArgs a) {
  constexpr bool FINAL = MODE == kSweepFinal;
  using Cfg = EmPass2Cfg<M, L, KT, FINAL>;
  using Lay = EmLayout<M, L>;
  constexpr int NDOF = Cfg::NDOF, NDOFP = Cfg::NDOFP, CPG = Cfg::CPG, NCHP = Cfg::NCHP, KTP = Cfg::KTP;
  constexpr int NA = Cfg::NA, WS = Cfg::WS, SPW = Cfg::SPW, NW = Cfg::NW;
  constexpr bool CPG_POW2 = (CPG & (CPG - 1)) == 0;
  using PL = PartLayout<M, L, KT, NA>;
  extern __shared__ float4 smem_f4[];
  float* s_coef = reinterpret_cast<float*>(smem_f4);          // [g][idx * KT + k], CS floats per g
  float* s_ck = s_coef + Cfg::COEF_FLOATS;                    // [pattern][KTP]
  const int ck_floats = (a.npat_max * KTP + 3) & ~3;
  float* s_scratch = s_ck + ck_floats;                        // NW x WARP_SCRATCH_FLOATS, 256-byte aligned:
  s_scratch += ((256u - ((unsigned)__cvta_generic_to_shared(s_scratch) & 255u)) & 255u) >> 2;  // XOR addressing
  unsigned char* s_amask = reinterpret_cast<unsigned char*>(s_scratch + NW * Cfg::WARP_SCRATCH_FLOATS);

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const WorkItem wi = a.work[blockIdx.x];
  const int f = blockIdx.y;
  const SegDev sd = a.segs[wi.seg];
  const int t0 = wi.chunk * sd.TC;
  const int nt = min(sd.TC, sd.T - t0);
  const int ngroups = (nt + 31) >> 5;
  const float2* src = a.y + sd.y_off + ((long long)f * sd.T + t0) * M;
  const unsigned char* psrc = a.pat + sd.pat_off + t0;

  // ---- tables of this (segment, bin)
  {
    const float* cp = a.coef + sd.coef_off + (long long)f * L * (KT * NDOF);  // [g][k][j]
    for (int i = tid; i < Cfg::COEF_FLOATS; i += kEmThreads) {
      const int g = i / Cfg::CS, r = i - g * Cfg::CS, j = r / KT, k = r - j * KT;
      s_coef[i] = j < NDOF ? cp[(g * KT + k) * NDOF + j] : 0.f;
    }
    const float* cks = a.ck + sd.tab_off + (long long)f * sd.npat * KT;
    for (int i = tid; i < sd.npat * KTP; i += kEmThreads) {
      const int k = i % KTP, p = i / KTP;
      s_ck[i] = k < KT ? cks[p * KT + k] : -CUDART_INF_F;
    }
    // classes that can be active under a pattern (finite constant); the others have gamma == 0 exactly
    for (int p = tid; p < sd.npat; p += kEmThreads) {
      unsigned m = 0;
      for (int k = 0; k < KT; ++k)
        if (cks[p * KT + k] != -CUDART_INF_F) m |= 1u << k;
      s_amask[p] = (unsigned char)m;
    }
  }
  __syncthreads();

  float* wscr = s_scratch + warp * Cfg::WARP_SCRATCH_FLOATS;
  float* wbuf = wscr + 32 * NCHP * 4;                                     // [32][WS]
  float2* ybuf = reinterpret_cast<float2*>(wbuf + 32 * WS);               // [32][SY]
  float* sums = reinterpret_cast<float*>(ybuf + 32 * Cfg::SY) + lane;      // [SUMS][32], this lane's column
#pragma unroll
  for (int k = 0; k < Cfg::SUMS; ++k) sums[32 * k] = 0.f;
  const int g = lane / SPW, slot = lane % SPW;  // phase-B role
  // Dof scratch addressing: chunk c of frame fr lives at float4 position fr * NCHP + (c ^ swz(fr)); with the
  // scratch aligned to the frame stride that is (address of chunk 0's home) XOR (c * 16): one LOP3. swz is a
  // permutation of the frame number's low bits (Cfg::swz) chosen so that the 8 lanes of a quarter-warp hit 8
  // different 16-byte columns in phase A (8 frames, one chunk) AND in phase B (SPW frames x 8 / SPW slices).
  const unsigned pbase = (unsigned)__cvta_generic_to_shared(wscr);
  const unsigned pa_store = pbase + (unsigned)lane * (NCHP * 16) + Cfg::swz((unsigned)lane) * 16;

  float acc[NA][NDOF];
#pragma unroll
  for (int n = 0; n < NA; ++n)
#pragma unroll
    for (int j = 0; j < NDOF; ++j) acc[n][j] = 0.f;
  float* gout = MODE != kSweepEM && a.gamma != nullptr && sd.g_off >= 0
                    ? a.gamma + sd.g_off + ((long long)f * sd.T + t0) * sd.K
                    : nullptr;
  const int target = sd.target;
  const bool normalize = a.normalize != 0;

  // frames of group `grp` -> this warp's landing zone; frames past the end are zero
  auto issue_group = [&](int grp) {
    const float2* gs = src + (long long)grp * 32 * M;
    const int n = (nt - grp * 32) * M;  // valid elements (may exceed 32 * M)
#pragma unroll
    for (int j = 0; j < M; ++j) {
      const int i = lane + 32 * j;
      cp_async8_zfill(ybuf + i + (Cfg::SY - M) * (i / M), gs + (i < n ? i : 0), i < n);
    }
    cp_async_commit();
  };
  int pid = 0;
  if (warp < ngroups) {
    issue_group(warp);
    pid = (int)psrc[min(warp * 32 + lane, nt - 1)];
  }

#pragma unroll 1
  for (int grp = warp; grp < ngroups; grp += NW) {
    const int t = grp * 32 + lane;
    const bool valid = t < nt;
    cp_async_wait<0>();
    __syncwarp();
    float2 y[M];
    {
      const float2* ys = ybuf + lane * Cfg::SY;
#pragma unroll
      for (int m = 0; m < M; ++m) y[m] = ys[m];
    }
    __syncwarp();  // every lane has taken its frame: the zone may be overwritten
    // the next group of this warp is fetched while this one is processed
    int pidn = 0;
    if (grp + NW < ngroups) {
      issue_group(grp + NW);
      pidn = (int)psrc[min((grp + NW) * 32 + lane, nt - 1)];
    }

    // ================= phase A: lane = frame =================
    float q[KT];
#pragma unroll
    for (int k = 0; k < KT; ++k) q[k] = 0.f;
    float n2 = 0.f;
#pragma unroll
    for (int gg = 0; gg < L; ++gg) {
      float pg[NDOFP];
#pragma unroll
      for (int j = 0; j < NDOFP; ++j) pg[j] = 0.f;
      float4 cc = make_float4(0.f, 0.f, 0.f, 0.f);
      int have = -1;
#pragma unroll
      for (int i = 0; i < Lay::RPL; ++i) {
        const int row = gg + i * L;
        if (row < M) {
          const float2 x = y[row];
#pragma unroll
          for (int jr = 0; jr < M; ++jr) {
            float p;
            if (jr == 0) {
              p = fmaf(x.x, x.x, x.y * x.y);
              n2 += p;
            } else if (jr <= 2 * Lay::D) {
              const float2 z = y[(row + (jr + 1) / 2) % M];
              p = (jr & 1) ? fmaf(x.x, z.x, x.y * z.y) : fmaf(x.y, z.x, -(x.x * z.y));
            } else {  // half diagonal (M even)
              const float2 z = y[(row + M / 2) % M];
              p = row < M / 2 ? fmaf(x.x, z.x, x.y * z.y) : fmaf(x.y, z.x, -(x.x * z.y));
            }
            pg[i * M + jr] = p;
            // packed coefficients: element e = dof * KT + k of this slice, fetched as whole float4s through a
            // warp-uniform (broadcast) address; `have` and every select below fold at compile time
#pragma unroll
            for (int k = 0; k < KT; ++k) {
              const int e = (i * M + jr) * KT + k;
              if ((e >> 2) != have) {
                cc = reinterpret_cast<const float4*>(s_coef + gg * Cfg::CS)[e >> 2];
                have = e >> 2;
              }
              const float cv = (e & 3) == 0 ? cc.x : (e & 3) == 1 ? cc.y : (e & 3) == 2 ? cc.z : cc.w;
              q[k] = fmaf(cv, p, q[k]);
            }
          }
        }
      }
      // park this slice's dofs: chunk (gg, c) of frame `lane` at swizzled position (conflict-free both ways)
#pragma unroll
      for (int c = 0; c < CPG; ++c)
        asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(pa_store ^ (unsigned)((gg * CPG + c) * 16)),
                     "f"(pg[4 * c]), "f"(pg[4 * c + 1]), "f"(pg[4 * c + 2]), "f"(pg[4 * c + 3])
                     : "memory");
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
    const float* ckp = s_ck + pid * KTP;
    const unsigned am = __reduce_or_sync(0xffffffffu, (unsigned)s_amask[pid]);
    float u[KT];
    float mx = -CUDART_INF_F;
#pragma unroll
    for (int k = 0; k < KT; ++k) {
      q[k] = fmaxf(q[k], qfloor);                            // cacgmm.hpp:170-171, in raw units
      // log2 domain: the table holds ck * log2(e); inactive classes carry ck = -inf
      u[k] = fmaf(-(float)M, lg2_approx(q[k]), ckp[k]);
      mx = fmaxf(mx, u[k]);
    }
#ifdef GSS_ACCURATE_MATH
    double sed = 0.0, ud[KT];
#pragma unroll
    for (int k = 0; k < KT; ++k) {
      ud[k] = exp2((double)u[k] - (double)mx);
      sed += ud[k];
    }
    const double rinvd = valid ? 1.0 / sed : 0.0;
    const float se = (float)sed, rinv = 1.f;
#pragma unroll
    for (int k = 0; k < KT; ++k) u[k] = (float)(ud[k] * rinvd);
#else
    float se = 0.f;
#pragma unroll
    for (int k = 0; k < KT; ++k) {
      u[k] = ex2_approx(u[k] - mx);
      se += u[k];
    }
    const float rinv = valid ? rcp_approx(se) : 0.f;
#endif
    // log2 units, scaled once at the end; the common s^2 factor comes back here: -M log2(s^2) = +M log2(nr2)
    // (a lane sums at most T / 256 such terms in float; lanes and chunks are then summed in double)
    if (valid) sums[32 * KT] += mx + lg2_approx(se) + (float)M * lg2_approx(nr2);
    float gam[KT];
#pragma unroll
    for (int k = 0; k < KT; ++k) {
      gam[k] = u[k] * rinv;  // exactly 0 for inactive classes and for lanes past the end
      sums[32 * k] += gam[k];
    }
    if (MODE != kSweepEM) {
      if (gout != nullptr && valid) {
        float* go = gout + (long long)t * sd.K;
#pragma unroll
        for (int k = 0; k < KT; ++k)
          if (k < sd.K) go[k] = gam[k];
      }
    }
    if (FINAL) {
      float wt = 0.f, wb = 0.f;
#pragma unroll
      for (int k = 0; k < KT; ++k) {
        wt += (k == target) ? gam[k] : 0.f;
        wb += (k == target) ? 0.f : gam[k];
      }
      *reinterpret_cast<float2*>(wbuf + lane * WS) = make_float2(wt, wb);
    } else {
      float w[KTP];
#pragma unroll
      for (int k = 0; k < KTP; ++k) w[k] = k < KT ? gam[k < KT ? k : 0] * rcp_approx(q[k < KT ? k : 0]) : 0.f;  // gamma / (q s^2)
      if (KTP == 2) {
        *reinterpret_cast<float2*>(wbuf + lane * WS) = make_float2(w[0], w[1]);
      } else {
#pragma unroll
        for (int k4 = 0; k4 < KTP / 4; ++k4)
          reinterpret_cast<float4*>(wbuf + lane * WS)[k4] = make_float4(w[4 * k4], w[4 * k4 + 1], w[4 * k4 + 2], w[4 * k4 + 3]);
      }
    }
    __syncwarp();

    // ================= phase B: lane = (frame slot, dof slice g) =================
    // Register double buffering: the dofs and weights of step + 1 are requested before the FMAs of step. The loads
    // are volatile asm on purpose: as plain loads the compiler sank each class's weight into that class's
    // conditional block, and every block then began with a shared-memory round trip (short-scoreboard stalls were
    // 58 % of this phase's samples on cfg3, profiles/ncu_full_r02.md).
    auto load_step = [&](int step, float (&pv)[NDOFP], float (&w)[WS]) {
      const int fr = step * SPW + slot;
      const unsigned pa_load =
          (pbase + (unsigned)fr * (NCHP * 16) + Cfg::swz((unsigned)fr) * 16) ^ (unsigned)(g * CPG * 16);
#pragma unroll
      for (int c = 0; c < CPG; ++c)  // (g * CPG + c) ^ x == (g * CPG) ^ c ^ x when CPG is a power of two ...
        asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                     : "=f"(pv[4 * c]), "=f"(pv[4 * c + 1]), "=f"(pv[4 * c + 2]), "=f"(pv[4 * c + 3])
                     : "r"(CPG_POW2 ? (pa_load ^ (unsigned)(c * 16))
                                    : ((pbase + (unsigned)fr * (NCHP * 16) + Cfg::swz((unsigned)fr) * 16) ^
                                       (unsigned)((g * CPG + c) * 16)))
                     : "memory");
      const unsigned wa = pbase + (unsigned)(32 * NCHP * 16) + (unsigned)fr * (WS * 4);
      if (WS == 2) {
        asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(w[0]), "=f"(w[WS > 1 ? 1 : 0]) : "r"(wa) : "memory");
      } else {
#pragma unroll
        for (int k4 = 0; k4 < WS / 4; ++k4)
          asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                       : "=f"(w[WS >= 4 ? 4 * k4 : 0]), "=f"(w[WS >= 4 ? 4 * k4 + 1 : 0]),
                         "=f"(w[WS >= 4 ? 4 * k4 + 2 : 0]), "=f"(w[WS >= 4 ? 4 * k4 + 3 : 0])
                       : "r"(wa + (unsigned)(16 * k4))
                       : "memory");
      }
    };
    float pvb[2][NDOFP], wb[2][WS];
    load_step(0, pvb[0], wb[0]);
#pragma unroll
    for (int step = 0; step < L; ++step) {
      const float(&pv)[NDOFP] = pvb[step & 1];
      const float(&w)[WS] = wb[step & 1];
      if (step + 1 < L) load_step(step + 1, pvb[(step + 1) & 1], wb[(step + 1) & 1]);
      if (FINAL) {
#pragma unroll
        for (int j = 0; j < NDOF; ++j) {
          acc[0][j] = fmaf(w[0], pv[j], acc[0][j]);
          acc[NA - 1][j] = fmaf(w[1], pv[j], acc[NA - 1][j]);
        }
      } else {
#pragma unroll
        for (int k = 0; k < NA; ++k) {
          if (am & (1u << k)) {  // warp-uniform: classes inactive for all 32 frames are skipped
#pragma unroll
            for (int j = 0; j < NDOF; ++j) acc[k][j] = fmaf(w[k], pv[j], acc[k][j]);
          }
        }
      }
    }
    __syncwarp();  // the scratch is rewritten by the next group's phase A
    pid = pidn;
  }

  // ---- reduce. Masses and the likelihood: butterfly over the warp's 32 frame lanes. Accumulators: every
  // thread parks its tile in shared memory and cell element (g, e) is the sum over the NW * SPW threads that
  // own slice g, in fixed order.
  float mass[KT];
#pragma unroll
  for (int k = 0; k < KT; ++k) mass[k] = sums[32 * k];
  double ll = (double)sums[32 * KT];
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
#pragma unroll
    for (int k = 0; k < KT; ++k) mass[k] += __shfl_xor_sync(0xffffffffu, mass[k], o);
    ll += __shfl_xor_sync(0xffffffffu, ll, o);
  }
  ll *= 0.69314718055994530942;  // back to natural-log units
  __syncthreads();               // every warp is done with its scratch
  constexpr int DS = Cfg::DUMP_STRIDE;
  float* dump = s_scratch;                                     // [NW * 32][DS]
  float* redm = dump + NW * 32 * DS;                           // [NW][KT]
  double* redll = reinterpret_cast<double*>(redm + ((NW * KT + 1) & ~1));
  {
    float* d = dump + tid * DS;
#pragma unroll
    for (int e4 = 0; e4 < (NA * NDOF + 3) / 4; ++e4) {
      float v[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int e = 4 * e4 + i;
        v[i] = e < NA * NDOF ? acc[e < NA * NDOF ? e / NDOF : 0][e < NA * NDOF ? e % NDOF : 0] : 0.f;
      }
      reinterpret_cast<float4*>(d)[e4] = make_float4(v[0], v[1], v[2], v[3]);
    }
  }
  if (lane == 0) {
#pragma unroll
    for (int k = 0; k < KT; ++k) redm[warp * KT + k] = mass[k];
    redll[warp] = ll;
  }
  __syncthreads();
  const long long cell = sd.cell_off + (long long)f * sd.nchunks + wi.chunk;
  float* out = a.part + cell * a.cell_stride;
  for (int i = tid; i < PL::CELL; i += kEmThreads) {
    const int gg = i / PL::STRIDE, e = i - gg * PL::STRIDE;
    float s = 0.f;
    if (e < PL::ACC) {
      for (int w = 0; w < NW; ++w)
#pragma unroll
        for (int sl = 0; sl < SPW; ++sl) s += dump[(w * 32 + gg * SPW + sl) * DS + e];
    } else {
#pragma unroll
      for (int w = 0; w < NW; ++w) s += redm[w * KT + (e - PL::ACC)];
    }
    out[i] = s;
  }
  if (tid == 0) {
    double s = 0.0;
#pragma unroll
    for (int w = 0; w < NW; ++w) s += redll[w];
    a.cell_ll[cell] = s;
  }
}

}  // namespace gssb
