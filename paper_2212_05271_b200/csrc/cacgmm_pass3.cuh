// cacgmm_pass3.cuh -- the cACGMM sweep for the wide arrays (M = 7, 8): third design, "row owner".
//
// Reference semantics (unchanged): cacgmm.hpp:156-174 (quad_forms), :189-257 (estep_bin), :308-329 (M-step Gram),
// wpe.hpp:124-140 (unit_normalize, folded in), beamform.hpp:35-85 (accumulate_stats, last sweep).
//
// Why a third design. ncu on the two-phase sweep (cacgmm_pass2.cuh) at M = 8, K = 5 shows the SHARED-MEMORY PIPE at
// 0.91 wavefronts per cycle, not the FP32 pipe, as the bound: 415 wavefronts per group of 32 frames, of which 160
// are the warp-uniform coefficient loads of phase A (a uniform LDS.128 still costs two wavefronts) and 128 park
// and re-read the Hermitian dofs between the phases, against 192 cycles of FFMA issue (profiles/ncu_full_r02.md).
// Here a lane keeps ONE ROW of P = y y^H for good:
//
//   lane = (frame slot, row g), 8 lanes per frame, 4 frames per step, 8 steps per group of 32 frames.
//   phase 1  per step: the row's M dofs from the frame's channels (kept in registers for phase 3), and the row's
//            share of the K quadratic forms with the coefficients held in REGISTERS for the whole (segment, bin):
//            no coefficient traffic at all. The K partial forms (+ the row's |y_g|^2) go to a swizzled exchange
//            buffer.
//   phase 2  lane = frame: adds the 8 partial forms, runs the guide-masked soft-max once per frame (same code as
//            the two-phase sweep), writes the K accumulation weights.
//   phase 3  lane = (slot, row) again: weights of its 8 frames in registers, then class-outer accumulation
//            acc[k][j] += w[s][k] * P[s][j] over the 8 steps: one warp-uniform branch per class and GROUP.
//
// Shared-memory wavefronts per group: 80 (frames) + 64 + 64 (exchange) + 8 + 32 (weights) + 16 (landing) ~ 265,
// against 415; the dofs never leave the register file. Cost: ~190 registers per thread, one block of 8 warps per SM.
// Cells, coefficient and table layouts are those of EmLayout<M, 8>, so em_update_kernel and the MVDR finaliser
// read the result unchanged.
#pragma once

#include "cacgmm_pass2.cuh"

namespace gssb {

// 8 warps: at 10 or 12 the 168 registers left per thread spill (26.2 / 22.7 vs 20.4 ms per 16-segment cfg3 step)
constexpr int kEm3Threads = 256;

template <int M, int KT, bool FINAL>
struct EmPass3Cfg {
  static constexpr int L = 8;
  using Lay = EmLayout<M, L>;
  static_assert(Lay::RPL == 1, "row-owner sweep: one row per lane (M <= 8)");
  static constexpr int NDOF = M;
  static constexpr int KTP = KT <= 2 ? 2 : KT <= 4 ? 4 : 8;  // padded class count of the constant table
  static constexpr int NA = FINAL ? 2 : KT;
  static constexpr int WS = FINAL ? 2 : KT;                  // weights per frame
  static constexpr int SPW = 4, NSTEP = 8;                   // frames per step, steps per group
  static constexpr int NW = kEm3Threads / 32;
  static constexpr int NQ = KT + 1;                          // exchanged per (frame, row): K partial forms + |y_g|^2
  static constexpr int WPL = (WS + 3) / 4;                   // float4 planes of the weight buffer
  static constexpr int EXCH_BYTES = NQ * 32 * 8 * 4;         // [quantity][frame][row] float: one 1 KB plane per class
  static constexpr int W_BYTES = WPL * 32 * 16;              // [plane][frame] float4
  static constexpr int Y_BYTES = 32 * M * 8;                 // [frame][channel] float2, natural stride
  static constexpr int WARP_SCRATCH_BYTES = (EXCH_BYTES + W_BYTES + Y_BYTES + 127) & ~127;
  static constexpr int DUMP_STRIDE = ((NA * NDOF + 3) / 4 | 1) * 4;
};

template <int M, int KT, int MODE>
__global__ void __launch_bounds__(kEm3Threads, 1) em_pass3_kernel(EmPassArgs a) {
  constexpr bool FINAL = MODE == kSweepFinal;
  using Cfg = EmPass3Cfg<M, KT, FINAL>;
  using Lay = EmLayout<M, 8>;
  constexpr int L = 8, NDOF = Cfg::NDOF, KTP = Cfg::KTP, NA = Cfg::NA, NW = Cfg::NW;
  constexpr int NSTEP = Cfg::NSTEP, SPW = Cfg::SPW, WPL = Cfg::WPL;
  constexpr int D = Lay::D, HALF = Lay::HALF;
  using PL = PartLayout<M, L, KT, NA>;
  extern __shared__ float4 smem_f4[];
  float* s_ck = reinterpret_cast<float*>(smem_f4);            // [pattern][KTP]
  const int ck_floats = (a.npat_max * KTP + 3) & ~3;
  unsigned char* s_amask = reinterpret_cast<unsigned char*>(s_ck + ck_floats);
  unsigned char* s_scr = s_amask + ((a.npat_max + 15) & ~15);
  s_scr += (128u - ((unsigned)__cvta_generic_to_shared(s_scr) & 127u)) & 127u;  // XOR addressing of the exchange

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
    const float* cks = a.ck + sd.tab_off + (long long)f * sd.npat * KT;
    for (int i = tid; i < sd.npat * KTP; i += kEm3Threads) {
      const int k = i % KTP, p = i / KTP;
      s_ck[i] = k < KT ? cks[p * KT + k] : -CUDART_INF_F;
    }
    for (int p = tid; p < sd.npat; p += kEm3Threads) {
      unsigned m = 0;
      for (int k = 0; k < KT; ++k)
        if (cks[p * KT + k] != -CUDART_INF_F) m |= 1u << k;
      s_amask[p] = (unsigned char)m;
    }
  }
  // phase-1/3 role: lane = slot * 8 + g (row fastest: the 8 lanes of a frame read its 8 channels side by side)
  const int slot = lane >> 3, g = lane & 7;
  const bool owner = g < M;                 // M = 7: lane 7 of every frame idles (zero coefficients)
  const int row = owner ? g : 0;
  // quadratic-form coefficients of this row, all classes: registers for the life of the block
  float cf[KT][NDOF];
  {
    const float* cp = a.coef + sd.coef_off + ((long long)f * L + g) * (KT * NDOF);  // [k][j]
#pragma unroll
    for (int k = 0; k < KT; ++k)
#pragma unroll
      for (int j = 0; j < NDOF; ++j) cf[k][j] = cp[k * NDOF + j];
  }
  __syncthreads();

  const unsigned wbase = (unsigned)__cvta_generic_to_shared(s_scr) + (unsigned)warp * Cfg::WARP_SCRATCH_BYTES;
  const unsigned wofs = wbase + Cfg::EXCH_BYTES;                 // weights [plane][frame] float4
  const unsigned yofs = wofs + Cfg::W_BYTES;                     // frames  [frame][channel] float2
  float2* ybuf = reinterpret_cast<float2*>(s_scr + (size_t)warp * Cfg::WARP_SCRATCH_BYTES + Cfg::EXCH_BYTES + Cfg::W_BYTES);
  // exchange addressing: plane q (class, or the norm) holds [frame][row] floats, 32 bytes per frame. A phase-1 store
  // (one class, one step) is 32 lanes x 4 bytes = 128 contiguous bytes; phase 2 (lane = frame) reads its frame's two
  // 16-byte halves, and the halves of frames 4..7 (mod 8) are swapped so that a quarter-warp covers all 32 banks:
  // row g of frame fr sits at float (g ^ 4 ((fr >> 2) & 1)); in phase 1 fr >> 2 is the step number.
  const unsigned ex_st0 = wbase + (unsigned)(slot * 32 + g * 4), ex_st1 = wbase + (unsigned)(slot * 32 + (g ^ 4) * 4);
  const unsigned ex_ld = wbase + (unsigned)(lane * 32 + ((lane >> 2) & 1) * 16);
  // channel addresses of this row and of its partners (frame `slot` of a step)
  const unsigned y_x = yofs + (unsigned)(slot * M + row) * 8u;
  unsigned y_z[D + HALF > 0 ? D + HALF : 1];
#pragma unroll
  for (int d = 1; d <= D; ++d) y_z[d - 1] = yofs + (unsigned)(slot * M + (row + d) % M) * 8u;
  if (HALF) y_z[D] = yofs + (unsigned)(slot * M + (row + M / 2) % M) * 8u;
  const bool lo_half = row < M / 2;

  float acc[NA][NDOF];
#pragma unroll
  for (int n = 0; n < NA; ++n)
#pragma unroll
    for (int j = 0; j < NDOF; ++j) acc[n][j] = 0.f;
  float mass[KT];
#pragma unroll
  for (int k = 0; k < KT; ++k) mass[k] = 0.f;
  float llacc = 0.f;
  float* gout = MODE != kSweepEM && a.gamma != nullptr && sd.g_off >= 0
                    ? a.gamma + sd.g_off + ((long long)f * sd.T + t0) * sd.K
                    : nullptr;
  const int target = sd.target;
  const bool normalize = a.normalize != 0;

  auto issue_group = [&](int grp) {
    const float2* gs = src + (long long)grp * 32 * M;
    const int n = (nt - grp * 32) * M;  // valid elements (may exceed 32 * M)
#pragma unroll
    for (int j = 0; j < M; ++j) {
      const int i = lane + 32 * j;
      cp_async8_zfill(ybuf + i, gs + (i < n ? i : 0), i < n);
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

    // classes that are active in at least one of the group's 32 frames: the others have gamma == 0 throughout, so
    // neither their quadratic forms (phase 1) nor their accumulation (phase 3) is evaluated
    const unsigned am = __reduce_or_sync(0xffffffffu, (unsigned)s_amask[pid]);

    // ================= phase 1: lane = (slot, row) =================
    // 1a: the row's dofs of the 8 steps (the channels of step s + 1 are requested before the arithmetic of step s)
    float P[NSTEP][NDOF];
    constexpr int NZ = D + HALF > 0 ? D + HALF : 1;
    float2 xb[2], zb[2][NZ];
    auto load_frame = [&](int s, float2& x, float2 (&z)[NZ]) {
      const unsigned so = (unsigned)(s * SPW * M * 8);
      asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(x.x), "=f"(x.y) : "r"(y_x + so));
#pragma unroll
      for (int d = 0; d < D + HALF; ++d)
        asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(z[d].x), "=f"(z[d].y) : "r"(y_z[d] + so));
    };
    load_frame(0, xb[0], zb[0]);
#pragma unroll
    for (int s = 0; s < NSTEP; ++s) {
      if (s + 1 < NSTEP) load_frame(s + 1, xb[(s + 1) & 1], zb[(s + 1) & 1]);
      const float2 x = xb[s & 1];
      const float2(&z)[NZ] = zb[s & 1];
      P[s][0] = fmaf(x.x, x.x, x.y * x.y);
#pragma unroll
      for (int d = 1; d <= D; ++d) {
        P[s][2 * d - 1] = fmaf(x.x, z[d - 1].x, x.y * z[d - 1].y);
        P[s][2 * d] = fmaf(x.y, z[d - 1].x, -(x.x * z[d - 1].y));
      }
      if (HALF) {
        const float a1 = lo_half ? x.x : x.y, a2 = lo_half ? x.y : -x.x;
        P[s][M - 1] = fmaf(a1, z[D].x, a2 * z[D].y);
      }
      // this row's share of |y|^2 (plane KT)
      asm volatile("st.shared.f32 [%0], %1;" ::"r"(((s & 1) ? ex_st1 : ex_st0) + (unsigned)(KT * 1024 + s * 128)),
                   "f"(owner ? P[s][0] : 0.f)
                   : "memory");
    }
    // 1b: class-outer partial forms: 8 independent chains (one per step) per active class
#pragma unroll
    for (int k = 0; k < KT; ++k) {
      if (am & (1u << k)) {  // warp-uniform
        float v[NSTEP];
#pragma unroll
        for (int s = 0; s < NSTEP; ++s) v[s] = cf[k][0] * P[s][0];
#pragma unroll
        for (int j = 1; j < NDOF; ++j)
#pragma unroll
          for (int s = 0; s < NSTEP; ++s) v[s] = fmaf(cf[k][j], P[s][j], v[s]);
#pragma unroll
        for (int s = 0; s < NSTEP; ++s)
          asm volatile("st.shared.f32 [%0], %1;" ::"r"(((s & 1) ? ex_st1 : ex_st0) + (unsigned)(k * 1024 + s * 128)),
                       "f"(v[s])
                       : "memory");
      }
    }
    __syncwarp();  // partial forms visible; every lane has taken its channels: the landing zone may be overwritten
    int pidn = 0;
    if (grp + NW < ngroups) {
      issue_group(grp + NW);
      pidn = (int)psrc[min((grp + NW) * 32 + lane, nt - 1)];
    }

    // ================= phase 2: lane = frame =================
    auto row_sum = [&](int plane) {  // the 8 rows' shares of one quantity for this lane's frame
      float4 u0, u1;
      asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                   : "=f"(u0.x), "=f"(u0.y), "=f"(u0.z), "=f"(u0.w)
                   : "r"(ex_ld + (unsigned)(plane * 1024))
                   : "memory");
      asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                   : "=f"(u1.x), "=f"(u1.y), "=f"(u1.z), "=f"(u1.w)
                   : "r"((ex_ld ^ 16u) + (unsigned)(plane * 1024))
                   : "memory");
      return ((u0.x + u0.y) + (u0.z + u0.w)) + ((u1.x + u1.y) + (u1.z + u1.w));
    };
    float q[KT];
#pragma unroll
    for (int k = 0; k < KT; ++k) q[k] = (am & (1u << k)) ? row_sum(k) : 1.f;  // inactive: any positive value, ck = -inf
    const float n2 = row_sum(KT);
    // Unit normalisation y/(|y|+1e-10) (wpe.hpp:135): see cacgmm_pass2.cuh; only the floor and the likelihood see it
    float nr2 = 1.f;
    if (normalize) {
      const float nr = sqrt_approx(n2) + 1e-10f;
      nr2 = nr * nr;
    }
    const float qfloor = kQuadFloor * nr2;
    const float* ckp = s_ck + pid * KTP;
    float u[KT];
    float mx = -CUDART_INF_F;
#pragma unroll
    for (int k = 0; k < KT; ++k) {
      q[k] = fmaxf(q[k], qfloor);                            // cacgmm.hpp:170-171, in raw units
      u[k] = fmaf(-(float)M, lg2_approx(q[k]), ckp[k]);      // log2 domain; inactive classes carry ck = -inf
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
    if (valid) llacc += mx + lg2_approx(se) + (float)M * lg2_approx(nr2);
    float gam[KT];
#pragma unroll
    for (int k = 0; k < KT; ++k) {
      gam[k] = u[k] * rinv;  // exactly 0 for inactive classes and for lanes past the end
      mass[k] += gam[k];
    }
    if (MODE != kSweepEM) {
      if (gout != nullptr && valid) {
        float* go = gout + (long long)t * sd.K;
#pragma unroll
        for (int k = 0; k < KT; ++k)
          if (k < sd.K) go[k] = gam[k];
      }
    }
    {
      float wv[4 * WPL];
#pragma unroll
      for (int k = 0; k < 4 * WPL; ++k) wv[k] = 0.f;
      if (FINAL) {
        float wt = 0.f, wbk = 0.f;
#pragma unroll
        for (int k = 0; k < KT; ++k) {
          wt += (k == target) ? gam[k] : 0.f;
          wbk += (k == target) ? 0.f : gam[k];
        }
        wv[0] = wt;
        wv[1] = wbk;
      } else {
#pragma unroll
        for (int k = 0; k < KT; ++k) wv[k] = gam[k] * rcp_approx(q[k]);  // gamma / (q s^2)
      }
#pragma unroll
      for (int p = 0; p < WPL; ++p)
        asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(wofs + (unsigned)(p * 512 + lane * 16)),
                     "f"(wv[4 * p]), "f"(wv[4 * p + 1]), "f"(wv[4 * p + 2]), "f"(wv[4 * p + 3])
                     : "memory");
    }
    __syncwarp();

    // ================= phase 3: lane = (slot, row) =================
    // in PH passes of NSTEP / PH steps each: the pass's weights in registers, then class-outer accumulation
    constexpr int PH = 1;  // (two passes of four steps: 20.2 vs 20.4 ms, within noise)
    constexpr int HS = NSTEP / PH;
#pragma unroll
    for (int h = 0; h < PH; ++h) {
      float w[HS][4 * WPL];
#pragma unroll
      for (int s = 0; s < HS; ++s)
#pragma unroll
        for (int p = 0; p < WPL; ++p)
          asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                       : "=f"(w[s][4 * p]), "=f"(w[s][4 * p + 1]), "=f"(w[s][4 * p + 2]), "=f"(w[s][4 * p + 3])
                       : "r"(wofs + (unsigned)(p * 512 + ((h * HS + s) * SPW + slot) * 16))
                       : "memory");
      if (FINAL) {
#pragma unroll
        for (int s = 0; s < HS; ++s)
#pragma unroll
          for (int j = 0; j < NDOF; ++j) {
            acc[0][j] = fmaf(w[s][0], P[h * HS + s][j], acc[0][j]);
            acc[NA - 1][j] = fmaf(w[s][1], P[h * HS + s][j], acc[NA - 1][j]);
          }
      } else {
#pragma unroll
        for (int k = 0; k < NA; ++k) {
          if (am & (1u << k)) {  // warp-uniform: classes inactive for all 32 frames are skipped
#pragma unroll
            for (int s = 0; s < HS; ++s)
#pragma unroll
              for (int j = 0; j < NDOF; ++j) acc[k][j] = fmaf(w[s][k], P[h * HS + s][j], acc[k][j]);
          }
        }
      }
    }
    __syncwarp();  // exchange and weight buffers are rewritten by the next group
    pid = pidn;
  }

  // ---- reduce. Masses and the likelihood: butterfly over the warp's 32 frame lanes. Accumulators: every thread
  // parks its tile in shared memory and cell element (g, e) is the sum over the NW * SPW threads that own row g,
  // in fixed order.
  double ll = (double)llacc;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
#pragma unroll
    for (int k = 0; k < KT; ++k) mass[k] += __shfl_xor_sync(0xffffffffu, mass[k], o);
    ll += __shfl_xor_sync(0xffffffffu, ll, o);
  }
  ll *= 0.69314718055994530942;  // back to natural-log units
  __syncthreads();               // every warp is done with its scratch
  constexpr int DS = Cfg::DUMP_STRIDE;
  float* dump = reinterpret_cast<float*>(s_scr);               // [NW * 32][DS]
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
  for (int i = tid; i < PL::CELL; i += kEm3Threads) {
    const int gg = i / PL::STRIDE, e = i - gg * PL::STRIDE;
    float s = 0.f;
    if (e < PL::ACC) {
      for (int w = 0; w < NW; ++w)
#pragma unroll
        for (int sl = 0; sl < SPW; ++sl) s += dump[(w * 32 + sl * 8 + gg) * DS + e];  // lane = slot * 8 + row
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
