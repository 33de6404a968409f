// gss_internal.cuh -- structures shared between the stage kernels and the
// batch orchestrator (api.cu). Not part of the public C ABI.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "em_layout.cuh"
#include "linalg.cuh"

namespace gssb {

constexpr int kMaxChannels = 8;   // M limit of the specialised kernels
constexpr int kMaxClasses = 8;    // K limit of the specialised kernels
constexpr int kEmThreads = 256;
constexpr int kEmLanes = 4;       // lanes cooperating on one frame in the EM sweep
constexpr int kEmTileFrames = 512;  // frames per shared-memory pipeline stage
constexpr float kQuadFloor = 1e-10f;   // cacgmm.hpp:17
constexpr double kWeightFloor = 1e-10; // cacgmm.hpp:18
constexpr double kPowerFloor = 1e-10;  // wpe.hpp:37

// Status word written by kernels: kStatusOk, else (code << 32 | frequency); the
// smallest value wins (atomicMin) so the report is deterministic.
typedef unsigned long long status_t;
constexpr status_t kStatusOk = ~0ull;
__host__ __device__ inline status_t make_status(int code, int f) {
  return ((status_t)(unsigned)code << 32) | (unsigned)f;
}

/// One enhancement problem (one SuperSegment) as the kernels see it. Offsets
/// index batch-wide device arrays (element units of the named type); arrays
/// whose size depends on T are ragged.
struct SegDev {
  long long audio_off;  // float  : M x N channel-major audio
  long long y_off;      // cfloat : (F,T,M) spectrogram (same offset in Y and Yd)
  long long g_off;      // float  : (F,T,K) posteriors (-1: not kept)
  long long x_off;      // cfloat : (T,F) beamformed spectrum, frame-major
  long long wave_off;   // float  : N output samples
  long long pat_off;    // uint8  : T activity-pattern ids
  long long mask_off;   // uint32 : npat class bit-masks
  long long tab_off;    // float  : (F,npat,KT) E-step constants
  long long coef_off;   // float  : (F,L,KT,NDOF) quadratic-form coefficients
  long long cell_off;   // EM / MVDR partial cells: F x nchunks
  long long fk_off;     // per-(f,k) state arrays: F x KT
  long long f_off;      // per-f arrays: F
  long long w_off;      // float  : (F,T) WPE weights
  long long wcell_off;  // WPE gram tiles: F x wchunks
  long long g_wpe_off;  // cfloat : (F, km, M) conj(G)
  int N, T, K, target, noise, npat;
  int TC, nchunks;      // EM frame chunking
  int WTC, wchunks;     // WPE frame chunking
  int wpe_active;       // 0 when T <= taps+delay (pass-through, wpe.hpp:108-112)
  int index;            // position in the caller's batch
};

struct WorkItem {
  int seg;    // index into the group's SegDev array
  int chunk;
};

struct StftParams {
  int fft_size, shift, window, F, log2n;
};

inline int ilog2(int n) {
  int b = 0;
  while ((1 << b) < n) ++b;
  return b;
}

}  // namespace gssb
