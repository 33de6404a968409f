/* gss_b200.h -- C ABI of libgss_b200.so: the B200 (sm_100a) implementation of the
 * guided-source-separation hot path `scheduler::enhance_batch` and the stage
 * operators it calls (reference: /root/reference/proj/include/gss/, cited per
 * entry point as file:line).
 *
 * Conventions
 *  - Plain C types only. Every pointer is a HOST pointer owned by the caller
 *    (pageable or pinned -- see gss_b200_host_alloc); the library owns device
 *    memory, streams and workspaces through `gss_b200_ctx`.
 *  - Complex tensors are interleaved (re, im) pairs: `float[2]` per cfloat,
 *    `double[2]` per cdouble. Tensor layouts are the reference's:
 *      spectrogram (F,T,M) row-major, index (f*T+t)*M+m      (stft.hpp:52-80)
 *      posteriors  (F,T,K) row-major float                   (cacgmm.hpp:52-62)
 *      activity    (T,K)   frame-major uint8                 (manifests.hpp:58-68)
 *      audio       (M,N)   channel-major float               (stft.hpp:39-47)
 *      small matrices row-major.
 *  - Every call returns a gss_status. 0 = ok; 1..9 mirror the reference's
 *    exception classes (common.hpp:17-79). The message (and, for
 *    GSS_SINGULAR_MATRIX_ERROR, the frequency bin) of the last failure of a
 *    context is available from gss_b200_last_error*().
 *  - One context per (host thread, device). Calls on one context are serialised
 *    by the caller; different contexts may run concurrently.
 *  - There is NO CPU fallback: without a CUDA device gss_b200_create fails with
 *    GSS_CUDA_ERROR and nothing else can be called. The host-only helpers at
 *    the end (index arithmetic, scalar known-answer forms) need no context.
 */
#ifndef GSS_B200_H_
#define GSS_B200_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum gss_status {
  GSS_OK = 0,
  GSS_SHAPE_ERROR = 1,            /* common.hpp:28  ShapeError */
  GSS_CONFIG_ERROR = 2,           /* common.hpp:33  ConfigError */
  GSS_PARSE_ERROR = 3,            /* common.hpp:38  ParseError (unused on this path) */
  GSS_IO_ERROR = 4,               /* common.hpp:43  IoError (unused on this path) */
  GSS_SINGULAR_MATRIX_ERROR = 5,  /* common.hpp:48  SingularMatrixError(frequency) */
  GSS_INPUT_TOO_SHORT_ERROR = 6,  /* common.hpp:58  InputTooShortError */
  GSS_EMPTY_TARGET_ERROR = 7,     /* common.hpp:63  EmptyTargetError */
  GSS_DEGENERATE_STATS_ERROR = 8, /* common.hpp:68  DegenerateStatsError */
  GSS_SPEC_ERROR = 9,             /* common.hpp:73  SpecError */
  GSS_INTERNAL_ERROR = 100,
  GSS_CUDA_ERROR = 101,
  GSS_UNSUPPORTED = 102 /* shape outside the compiled kernel range (M, K <= 8) */
} gss_status;

/* stft.hpp:16-36 StftConfig. window: 0 = hann, 1 = sqrt-hann. */
typedef struct gss_stft_config {
  int32_t fft_size;    /* default 1024 */
  int32_t shift;       /* default 256  */
  int32_t window;      /* default 0    */
  int32_t sample_rate; /* default 16000 */
} gss_stft_config;

/* wpe.hpp:15-30 WpeConfig */
typedef struct gss_wpe_config {
  int32_t taps;           /* default 10 */
  int32_t delay;          /* default 2  */
  int32_t iterations;     /* default 3  */
  int32_t psd_context;    /* default 0  */
  double regularization;  /* default 1e-10 */
} gss_wpe_config;

/* The fields of scheduler.hpp:30-44 PipelineConfig that enhance_batch reads. */
typedef struct gss_pipeline_config {
  gss_stft_config stft;
  gss_wpe_config wpe;
  int32_t enable_wpe;     /* default 1  */
  int32_t bss_iterations; /* default 20 */
} gss_pipeline_config;

void gss_b200_default_stft_config(gss_stft_config* c);
void gss_b200_default_wpe_config(gss_wpe_config* c);
void gss_b200_default_pipeline_config(gss_pipeline_config* c);

typedef struct gss_b200_ctx gss_b200_ctx;

/* ---- context ------------------------------------------------------------ */
gss_status gss_b200_create(int device, gss_b200_ctx** out);
void gss_b200_destroy(gss_b200_ctx* ctx);
/* Message / frequency bin of the last failed call on ctx (ctx == NULL: of the
 * last failed context-free call on this thread). */
const char* gss_b200_last_error(const gss_b200_ctx* ctx);
int64_t gss_b200_last_error_frequency(const gss_b200_ctx* ctx);
/* cudaStream_t all kernels of this context are launched on. */
void* gss_b200_stream(gss_b200_ctx* ctx);
/* Kernels launched by this context since creation (monotonic). */
int64_t gss_b200_launch_count(const gss_b200_ctx* ctx);
/* Bytes of device memory currently held by the context's workspaces. */
int64_t gss_b200_device_bytes(const gss_b200_ctx* ctx);
/* High-water mark of the same since creation (or since the last call with reset != 0): the peak device
 * footprint of a batch, the number BASELINE configs[3] ("1 GPU memory-bound sizing") asks for. */
int64_t gss_b200_device_bytes_peak(gss_b200_ctx* ctx, int32_t reset);
/* Pinned host memory for fast, asynchronous transfers (optional). */
gss_status gss_b200_host_alloc(int64_t bytes, void** out);
void gss_b200_host_free(void* p);

/* ---- stage operators (one tensor per call; host in, host out) ------------ */

/* stft::analyze (stft.hpp:131-175). audio (M,N); out (F,T,M) cfloat with
 * F = fft_size/2+1, T = gss_b200_frame_count(N). signal_rate 0 = unspecified. */
gss_status gss_b200_stft(gss_b200_ctx* ctx, const float* audio, int32_t channels, int64_t num_samples,
                         int32_t signal_rate, const gss_stft_config* cfg, float* out_ftm);

/* stft::synthesize (stft.hpp:179-229). spec (F,T,M) cfloat; out (M,out_len),
 * out_len = num_samples > 0 ? num_samples : (T-1)*shift. */
gss_status gss_b200_istft(gss_b200_ctx* ctx, const float* spec_ftm, int32_t bins, int64_t frames,
                          int32_t channels, int64_t num_samples, const gss_stft_config* cfg, float* out);

/* wpe::dereverberate (wpe.hpp:105-120). frames <= taps+delay: bit-identical
 * pass-through (wpe.hpp:108-112). */
gss_status gss_b200_wpe(gss_b200_ctx* ctx, const float* in_ftm, int32_t bins, int64_t frames,
                        int32_t channels, const gss_wpe_config* cfg, float* out_ftm);

/* wpe::unit_normalize (wpe.hpp:124-140). */
gss_status gss_b200_unit_normalize(gss_b200_ctx* ctx, const float* in_ftm, int32_t bins, int64_t frames,
                                   int32_t channels, float* out_ftm);

/* cacgmm::em_fit (cacgmm.hpp:264-340) on an already unit-normalised tensor.
 * Outputs (each nullable): gamma (F,T,K) float; pi (F,K) double; shapes
 * (F,K,M,M) cdouble; trace[iterations+1] double. */
gss_status gss_b200_em_fit(gss_b200_ctx* ctx, const float* yn_ftm, int32_t bins, int64_t frames,
                           int32_t channels, const uint8_t* activity_tk, int64_t activity_frames,
                           int32_t classes, int32_t noise_index, int32_t iterations, float* gamma_ftk,
                           double* pi_fk, double* shapes_fkmm, double* trace);

/* cacgmm::log_likelihood (cacgmm.hpp:343-370). */
gss_status gss_b200_log_likelihood(gss_b200_ctx* ctx, const float* yn_ftm, int32_t bins, int64_t frames,
                                   int32_t channels, const uint8_t* activity_tk, int32_t classes,
                                   int32_t noise_index, const double* pi_fk, const double* shapes_fkmm,
                                   double* out);

/* beamform::accumulate_stats (beamform.hpp:35-85). target/background (F,M,M) cdouble. */
gss_status gss_b200_mvdr_stats(gss_b200_ctx* ctx, const float* y_ftm, const float* gamma_ftk,
                               int32_t bins, int64_t frames, int32_t channels, int32_t classes,
                               int32_t target_index, double* target_fmm, double* background_fmm);

/* beamform::select_reference (beamform.hpp:89-107). */
gss_status gss_b200_select_reference(gss_b200_ctx* ctx, const double* target_fmm,
                                     const double* background_fmm, int32_t bins, int32_t channels,
                                     int32_t* ref_channel);

/* beamform::mvdr (beamform.hpp:111-135). h (F,M) cdouble. */
gss_status gss_b200_mvdr(gss_b200_ctx* ctx, const double* target_fmm, const double* background_fmm,
                         int32_t bins, int32_t channels, int32_t ref_channel, double* h_fm,
                         int64_t* zeroed_bins);

/* beamform::apply (beamform.hpp:138-165). out (F,T,1) cfloat. */
gss_status gss_b200_apply(gss_b200_ctx* ctx, const double* h_fm, int32_t h_bins, int32_t h_channels,
                          const float* y_ftm, int32_t bins, int64_t frames, int32_t channels,
                          float* out_ft);

/* ---- the hot path: scheduler::enhance_batch over a batch of SuperSegments -- */

/* One SuperSegment (scheduler.hpp:165-180) as plain arrays. */
typedef struct gss_segment_desc {
  const float* audio;        /* (M,N) channel-major */
  int32_t channels;          /* M */
  int32_t sample_rate;       /* 0 = unspecified */
  int64_t num_samples;       /* N */
  const uint8_t* activity;   /* (T,K), T must equal frame_count(N) */
  int64_t activity_frames;   /* T */
  int32_t num_classes;       /* K */
  int32_t target_index;
  int32_t noise_index;       /* -1 = no noise class */
  int32_t num_parts;
  const int64_t* part_begin; /* SuperSegment::Part::sample_begin */
  const int64_t* part_end;   /* SuperSegment::Part::sample_end */
  /* outputs (caller-allocated) */
  float* out_wave;           /* concatenated cuts, capacity sum(min(end,N)-begin) */
  int64_t* out_lengths;      /* [num_parts] */
  float* mono_out;           /* nullable: full synthesis window, N floats */
  float* gamma_out;          /* nullable: (F,T,K) posteriors of the last E-step */
  double* h_out;             /* nullable: (F,M) cdouble beamformer */
} gss_segment_desc;

/* EnhancementResult diagnostics (scheduler.hpp:283-294) + per-segment status. */
typedef struct gss_segment_diag {
  int32_t status;            /* gss_status of this segment */
  int32_t ref_channel;
  int64_t error_frequency;   /* bin for GSS_SINGULAR_MATRIX_ERROR, else -1 */
  int64_t zeroed_bins;
  int64_t frames;
  double ll_final;
} gss_segment_diag;

/* Device time per stage of the last batch run on ctx, milliseconds (CUDA events):
 * [0] stft [1] wpe [2] mask (unit-norm + EM) [3] beamform [4] istft [5] h2d [6] d2h */
#define GSS_B200_NUM_STAGES 7

/* scheduler::enhance_batch (scheduler.hpp:314-365) for n_segments independent
 * SuperSegments in one call (the size-1 case is the reference's signature).
 * Returns non-zero only for call-level failures (bad config, CUDA error); a
 * failing segment reports through diags[i].status and does not affect the
 * others (the reference fails one batch at a time, scheduler.hpp:565-575). */
gss_status gss_b200_enhance_batch(gss_b200_ctx* ctx, int32_t n_segments, const gss_segment_desc* segments,
                                  const gss_pipeline_config* cfg, gss_segment_diag* diags);

/* The same work split in three, so that callers can keep a batch resident in
 * HBM: upload (H2D) -> run (kernels only, asynchronous on the context stream)
 * -> fetch (D2H + synchronise). enhance_batch == upload + run + fetch + free. */
typedef struct gss_b200_batch gss_b200_batch;
gss_status gss_b200_batch_upload(gss_b200_ctx* ctx, int32_t n_segments, const gss_segment_desc* segments,
                                 const gss_pipeline_config* cfg, gss_b200_batch** out);
gss_status gss_b200_batch_run(gss_b200_ctx* ctx, gss_b200_batch* batch);
gss_status gss_b200_batch_fetch(gss_b200_ctx* ctx, gss_b200_batch* batch, gss_segment_diag* diags);
void gss_b200_batch_free(gss_b200_ctx* ctx, gss_b200_batch* batch);
gss_status gss_b200_stage_ms(gss_b200_ctx* ctx, double* ms /* [GSS_B200_NUM_STAGES] */);

/* Per-kernel device clocks. gss_b200_profile(ctx, 1) resets the counters and brackets every launch with
 * CUDA events on the context stream; gss_b200_kernel_ms synchronises and returns, per kernel class, the
 * summed duration (ms) and the number of launches since then. Classes:
 * 0 stft, 1 wpe_power, 2 wpe_gram, 3 wpe_solve, 4 wpe_apply, 5 em_pass, 6 em_update, 7 mvdr, 8 apply,
 * 9 istft, 10 misc. Launch counts are maintained even when event timing is off. */
/* Measured FP32 FMA throughput of the device (TFLOP/s, FMA = 2 flop): the roofline denominator of the
 * FP32-bound kernels (WPE Gram, EM sweep). Bench harness use. */
gss_status gss_b200_fp32_peak(gss_b200_ctx* ctx, double* tflops);
#define GSS_B200_NUM_KERNELS 11
gss_status gss_b200_profile(gss_b200_ctx* ctx, int32_t enable);
gss_status gss_b200_kernel_ms(gss_b200_ctx* ctx, double* ms /* [GSS_B200_NUM_KERNELS] */,
                              int64_t* launches /* [GSS_B200_NUM_KERNELS] */);

/* ---- device-pointer variants ("All pointers are host pointers unless the _dev variant is used") --
 * For callers whose tensors already live in HBM (a loader that decodes on the GPU, a downstream ASR front end).
 * Every tensor argument is a DEVICE pointer on the context's device; small control arrays stay on the host where
 * noted. `stream` is the caller's cudaStream_t (NULL = legacy default stream): the operator is ordered after the
 * work already queued on it, and the stream waits for the operator's results -- the stage operators below do not
 * synchronise with the host (gss_b200_wpe_dev reads back one status word, a solve can fail). Same return codes,
 * same kernels, same bits as the host variants. */
gss_status gss_b200_stft_dev(gss_b200_ctx* ctx, const float* audio_dev, int32_t channels, int64_t num_samples,
                             int32_t signal_rate, const gss_stft_config* cfg, float* out_ftm_dev, void* stream);
gss_status gss_b200_istft_dev(gss_b200_ctx* ctx, const float* spec_ftm_dev, int32_t bins, int64_t frames,
                              int32_t channels, int64_t num_samples, const gss_stft_config* cfg, float* out_dev,
                              void* stream);
gss_status gss_b200_wpe_dev(gss_b200_ctx* ctx, const float* in_ftm_dev, int32_t bins, int64_t frames,
                            int32_t channels, const gss_wpe_config* cfg, float* out_ftm_dev, void* stream);
gss_status gss_b200_unit_normalize_dev(gss_b200_ctx* ctx, const float* in_ftm_dev, int32_t bins, int64_t frames,
                                       int32_t channels, float* out_ftm_dev, void* stream);
/* h_fm is a HOST array (F x M cdouble, the value mvdr returned); y and out are device tensors. */
gss_status gss_b200_apply_dev(gss_b200_ctx* ctx, const double* h_fm, int32_t h_bins, int32_t h_channels,
                              const float* y_ftm_dev, int32_t bins, int64_t frames, int32_t channels,
                              float* out_ft_dev, void* stream);
/* scheduler::enhance_batch with the audio and the outputs in HBM: in every gss_segment_desc `audio`, `out_wave`
 * and the optional `mono_out` / `gamma_out` / `h_out` are DEVICE pointers; `activity`, `part_begin`, `part_end`
 * and `out_lengths` stay HOST arrays (a few KB of integers the host planner produced). Per-segment status comes
 * back in `diags`, so the call returns after the batch has finished. */
gss_status gss_b200_enhance_batch_dev(gss_b200_ctx* ctx, int32_t n_segments, const gss_segment_desc* segments,
                                      const gss_pipeline_config* cfg, gss_segment_diag* diags, void* stream);

/* NVTX: every stage of enhance_batch is enqueued inside a host-side range named after the reference's stage keys
 * ("gss.stft", "gss.wpe", "gss.mask", "gss.beamform", "gss.istft", "gss.d2h", all inside "gss.enhance_batch"), so
 * a profiler attributes the launches to the stage. Returns how many ranges this context has opened. */
int64_t gss_b200_nvtx_range_count(const gss_b200_ctx* ctx);

/* ---- host-only helpers (bit-exact integer / scalar forms; no context) ---- */

/* stft::frame_count (stft.hpp:120-124) */
int64_t gss_b200_frame_count(int64_t num_samples, int32_t fft_size, int32_t shift);

/* manifests::build_activity_at (manifests.hpp:372-414). classes_out receives
 * the '\n'-joined class labels (sorted speakers, target included, "noise" last). */
gss_status gss_b200_build_activity_at(int32_t n_segments, const char* const* speakers, const double* starts,
                                      const double* durations, const int64_t* centers, int64_t n_centers,
                                      int32_t sample_rate, const char* target, int32_t noise_class,
                                      uint8_t* grid, int64_t grid_capacity, int32_t* num_classes,
                                      int32_t* target_index, int32_t* noise_index, char* classes_out,
                                      int32_t classes_capacity);

/* The integer half of scheduler::assemble (scheduler.hpp:196-266): span list,
 * part offsets inside the assembled audio, frame-centre -> source-sample map. */
gss_status gss_b200_assemble_indices(int32_t n_parts, const double* starts, const double* durations,
                                     int32_t sample_rate, int64_t rec_samples, double context_duration,
                                     int32_t fft_size, int32_t shift, int64_t* spans_out /* [2*(n_parts+2)] */,
                                     int32_t* n_spans, int64_t* part_begin, int64_t* part_end, int64_t* total,
                                     int64_t* centers_out, int64_t centers_capacity, int64_t* n_centers,
                                     double* context_left, double* context_right);

/* cacgmm::cacg_log_pdf (cacgmm.hpp:66-82), y[M] cdouble, b (M,M) cdouble. */
gss_status gss_b200_cacg_log_pdf(int32_t channels, const double* y, const double* b, double* out);
/* cacgmm::time_varying_weights (cacgmm.hpp:87-112). */
gss_status gss_b200_time_varying_weights(int32_t classes, const double* pi, const uint8_t* activity,
                                         int32_t noise_index, double* out);

#ifdef __cplusplus
}
#endif
#endif /* GSS_B200_H_ */
