// kernels.h -- argument blocks and launchers of the stage kernels (internal).
#pragma once

#include "gss_internal.cuh"

namespace gssb {

// ---- STFT / iSTFT / apply (stft_kernels.cu) --------------------------------
struct StftArgs {
  const float* audio;
  float2* y;
  const SegDev* segs;
  const double2* tw_d;  // exp(-2 pi i k / n), k < n/2
  const double* win_d;  // analysis window, n doubles
  StftParams p;
  int M, TB, fft_warps;
};
struct ApplyArgs {
  const float2* y;
  const float2* hconj;  // (f, M): conj(h) rounded to cfloat
  float2* x;            // (T, F) per segment (frame_major) or (F, T)
  const SegDev* segs;
  int M, F;
  int frame_major;
};
struct IstftArgs {
  const float2* x;
  float* wave;
  const SegDev* segs;
  const float2* tw;
  const float* win;
  StftParams p;
  int HB;
};
cudaError_t launch_stft(const StftArgs& a, int nseg, int max_frames, cudaStream_t st);
cudaError_t launch_apply(const ApplyArgs& a, int nseg, int max_frames, cudaStream_t st);
cudaError_t launch_istft(const IstftArgs& a, int nseg, long long max_out_len, cudaStream_t st);

// ---- WPE (wpe_kernels.cu) ---------------------------------------------------
struct WpeArgs {
  const float2* yobs;   // observed spectrogram
  const float2* ycur;   // current estimate (power source)
  float2* yout;         // next estimate
  float* w;             // (F,T) weights
  float2* gram;         // tiles (FP32 path)
  float* gram_raw;      // raw real accumulators (tensor-core path): (F, 128, NCT) per segment
  float2* gconj;        // (F, km, M)
  const SegDev* segs;
  status_t* status;
  double regularization;
  int M, taps, delay, psd_context;
  cdbl* fb_scratch;     // eigenvalue-floor fallback: fb_slots slots of wpe_fallback_slot_elems cdbl
  int* fb_ticket;
  int fb_slots;
  cdbl* debug_rp;       // non-null: the solve kernel only dumps hermitized R (km x km) and P (km x M) per bin
  int use_tc;           // 1: the Gram of this iteration came from wpe_gram_tc_kernel
  int gram_f16;         // tensor-core Gram: 1 = FP16 hi / lo split (K = 16 per MMA), 0 = TF32 split (K = 8)
  int apply_tc;         // 1: the prediction runs on the tensor cores (wpe_apply_tc_kernel)
  int apply_f16;        // tensor-core prediction: 1 = FP16 hi / lo split (one MMA pair per tap), 0 = TF32 split (two)
  float* w_next;        // tensor-core prediction only: also write the NEXT iteration's Gram weights (psd_context 0)
};
/// cdbl elements of one scratch slot of the WPE solve's eigenvalue-floor fallback: A, two work matrices, B, eigenvalues
__host__ __device__ inline int wpe_fallback_slot_elems(int km, int M) { return 3 * km * km + km * M + km / 2 + 1; }
/// cfloat elements of one (segment, bin, chunk) Gram cell
int wpe_gram_cell_elems(int km, int M);
/// tensor-core Gram (wpe_gram_tc.cu)
/// Rows of the staged operand = columns of the accumulator D1: [Re a | Im a] (each padded to 8) + 16 current-frame rows,
/// rounded up to 16; up to one 128-row tile it is rounded to 32 so that a quarter of the columns is a whole number of
/// 8-column tensor-memory loads (M = 1, 3 at 10 taps).
__host__ __device__ inline int wpe_tc_operand_rows(int km) {
  const int kmp = (km + 7) & ~7, nr = ((2 * kmp + 16 + 15) / 16) * 16;
  return nr < 128 ? (nr + 31) & ~31 : nr;
}
int wpe_tc_supported(int km, int M);
int wpe_tc_cell_floats(int km, int M);
int wpe_tc_rows(int km, int M);
cudaError_t launch_wpe_gram_tc(const WpeArgs& a, int nseg, int F, cudaStream_t st);
/// tensor-core prediction (wpe_apply_tc.cu)
int wpe_apply_tc_supported(int taps, int delay, int M);
cudaError_t launch_wpe_apply_tc(const WpeArgs& a, int nseg, int F, cudaStream_t st);
/// one kernel of a WPE iteration; step: 0 power, 1 gram, 2 solve, 3 apply
cudaError_t launch_wpe_step(int step, const WpeArgs& a, int nseg, int F, int max_frames, int max_wchunks,
                            cudaStream_t st);

// ---- cACGMM EM + MVDR statistics (cacgmm_kernels.cuh, cacgmm_m*.cu) -----------
enum EmUpdateMode { kEmInit = 0, kEmMstep = 1, kEmFinal = 2, kEmFromState = 3 };

struct EmPassArgs {
  const float2* y;
  const SegDev* segs;
  const WorkItem* work;
  const unsigned char* pat;
  const float* ck;
  const float* coef;
  float* part;
  double* cell_ll;
  float* gamma;       // nullable: posteriors of this sweep
  int cell_stride;    // floats per partial cell
  int npat_max;
  int normalize;      // 1: frames are unit-normalised on the fly (wpe.hpp:124-140)
};
struct EmUpdateArgs {
  const SegDev* segs;
  const uint32_t* masks;
  const float* part;
  const double* cell_ll;
  cdbl* bstate;     // (fk, M*M) shape matrices B
  double* pi;       // (fk)
  double* logdet;   // (fk)
  float* coef;
  float* ck;
  double* bin_ll;   // (f) slot of this sweep
  status_t* status; // per segment of the group
  double c0;        // -M log(2 pi) + lgamma(M) (cacgmm.hpp:196)
  int cell_stride;
  int mode;
  int F;
};
struct StatsPassArgs {
  const float2* y;
  const float* gamma;
  const SegDev* segs;
  const WorkItem* work;
  float* part;
  int cell_stride;
};
struct StatsFinalArgs {
  const SegDev* segs;
  const float* part;
  cdbl* phi_t;     // (f, M*M)
  cdbl* phi_b;     // (f, M*M)
  double* tmass;   // (f)
  int cell_stride;
  int F;
};

/// Lanes cooperating on one frame, chosen so the per-thread register tiles
/// (2 * KT * NDOF floats) stay in registers.
constexpr int em_lanes(int M, int KT) {
#ifdef GSS_EXP_EM_LANES
  if (M >= 5) return GSS_EXP_EM_LANES;
#endif
  if (M == 1) return 1;
  if (M <= 4) return 2;
  if (M == 5) return KT <= 5 ? 2 : 4;
  if (M == 6) return 4;  // (the row-owner sweep with two idle lanes per frame: 13.0 vs 11.7 ms, tools/shape_bench.py 6 2)
  // M = 7, 8 run the row-owner sweep (cacgmm_pass3.cuh), one row of the outer product per lane: 8 lanes per frame
  // (at M = 7 the eighth lane of a frame idles; still 14.9 vs 15.4 ms per cfg2 step against the two-phase sweep once
  // the inactive classes are skipped; at M = 8 it wins for every class count: 14.5 vs 17.1 ms at K = 3).
  return 8;
}
/// Class count the kernels are instantiated for (>= K).
constexpr int em_class_tier(int K) { return K <= 2 ? 2 : K <= 3 ? 3 : K <= 4 ? 4 : K <= 5 ? 5 : K <= 6 ? 6 : 8; }
constexpr int em_ndof(int M, int L) { return ((M + L - 1) / L) * M; }
/// floats per partial cell (covers both sweep flavours)
constexpr int em_cell_floats(int M, int KT) {
  return em_lanes(M, KT) * ((KT > 2 ? KT : 2) * em_ndof(M, em_lanes(M, KT)) + KT);
}

struct EmShape {
  int M, KT;
};
cudaError_t launch_em_pass(EmShape s, bool final_sweep, const EmPassArgs& a, int nwork, int F, cudaStream_t st);
cudaError_t launch_em_update(EmShape s, const EmUpdateArgs& a, int nseg, cudaStream_t st);
cudaError_t launch_mvdr_stats(EmShape s, const StatsPassArgs& a, int nwork, int F, cudaStream_t st);
cudaError_t launch_mvdr_stats_final(EmShape s, const StatsFinalArgs& a, int nseg, cudaStream_t st);

// ---- beamformer design + misc (beamform_kernels.cu) -------------------------------
struct MvdrArgs {
  const SegDev* segs;
  const cdbl* phi_t;
  const cdbl* phi_b;
  const double* tmass;
  int* ref;            // per segment (in/out)
  int* zeroed;         // per segment
  cdbl* h;             // (f, M)
  float2* hconj;       // (f, M)
  status_t* status;
  int M, F;
  int fixed_ref;       // >= 0: use this reference channel instead of selecting
};
cudaError_t launch_select_reference(const MvdrArgs& a, int nseg, cudaStream_t st);
cudaError_t launch_mvdr_solve(const MvdrArgs& a, int nseg, cudaStream_t st);
cudaError_t launch_unit_normalize(const float2* in, float2* out, long long frames_total, int M, cudaStream_t st);
/// 256 * iters FMAs per thread, 256 threads per CTA
cudaError_t launch_fma_peak(float* scratch, int ctas, int iters, cudaStream_t st);
cudaError_t launch_sum_ll(const double* bin_ll, double* out, const SegDev* segs, int nseg, int F, cudaStream_t st);

}  // namespace gssb
