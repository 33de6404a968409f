// api.cu -- the C ABI of libgss_b200.so (include/gss_b200.h): context, batch
// orchestration of scheduler::enhance_batch (scheduler.hpp:314-365) over many
// independent SuperSegments, and the stage entry points. Host code only; every
// numerical step is a kernel launch on the context's stream. There is no CPU
// implementation of any stage in this library.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <chrono>
#include <cstring>
#include <map>
#include <memory>
#include <string>
#include <vector>

#include "../../include/gss_b200.h"
#include <nvtx3/nvToolsExt.h>

#include "kernels.h"

namespace gssb {

namespace {
thread_local std::string t_err;
thread_local long long t_err_freq = -1;
}  // namespace

void set_thread_error(int code, const std::string& msg, long long freq) {
  (void)code;
  t_err = msg;
  t_err_freq = freq;
}

struct Tables {
  float2* tw = nullptr;
  float* win = nullptr;
  double2* tw_d = nullptr;
  double* win_d = nullptr;
};

struct Fail {
  gss_status code;
  std::string msg;
  long long freq;
};

}  // namespace gssb

using namespace gssb;

struct gss_b200_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  cudaStream_t copy_stream = nullptr;  // audio uploads, wave by wave, under the previous wave's kernels
  int waves = 3;                       // GSS_B200_WAVES
  double wave_first_frac = 0.0;        // GSS_B200_WAVE_FIRST_PCT: share of the audio in the first wave (0: from the growth)
  double wave_growth = 4.0;            // GSS_B200_WAVE_GROWTH: each wave this many times the previous one
  long long wave_min_floats = 2 << 20; // GSS_B200_WAVE_MIN_FLOATS: no wave smaller than this (8 MB)
  std::string err;
  long long err_freq = -1;
  long long launches = 0;
  long long device_bytes = 0;
  long long device_bytes_peak = 0;
  std::map<std::pair<int, int>, Tables> tables;
  double stage_ms[GSS_B200_NUM_STAGES] = {0, 0, 0, 0, 0, 0, 0};
  // optional per-kernel device clocks (gss_b200_profile)
  bool prof_on = false;
  struct ProfRec {
    int id;
    cudaEvent_t a, b;
  };
  std::vector<ProfRec> prof_recs;
  double kernel_ms[GSS_B200_NUM_KERNELS] = {0};
  long long kernel_launches[GSS_B200_NUM_KERNELS] = {0};
  // WPE kernel choice: 2 = by shape (default), 1 = tcgen05 wherever it is supported (GSS_B200_WPE_GRAM / _APPLY = tc),
  // 0 = the FP32-FMA kernels (= fp32). By shape, with the FP16 kinds (tools/shape_bench.py, 16 segments, ms per step):
  // both from 4 channels. Gram: 6.6 against 16.9 at M = 4. At M = 2, 3 the tensor kernel is faster too (5.56 against
  // 6.85, 6.62 against 9.95) but the split's 1e-6 Gram error -- against 1e-7 of an FP32 sum -- tips a few barely
  // positive-definite bins of those more-sources-than-channels shapes into the solve's eigenvalue-floor fallback in the
  // third iteration (2.0 instead of 0.28 ms for that launch), so they keep the FP32 kernel. Prediction: 1.59 and the
  // fused power pass against 1.98 + 0.33 at M = 4; a tie at M = 3; 1.54 against 0.78 at M = 2.
  int wpe_gram_tc = 2;
  int wpe_gram_f16 = 1;      // tensor-core Gram operand split: 1 = FP16 (K = 16 per MMA), 0 = TF32 (GSS_B200_WPE_GRAM_KIND = tf32)
  int wpe_apply_tc = 2;
  int wpe_apply_f16 = 1;     // tensor-core prediction operand split, as wpe_gram_f16 (GSS_B200_WPE_APPLY_KIND = tf32)
  int em_chunk_frames = 0;   // debug knob: force the EM frame chunk (0 = automatic)
  int wpe_chunk_frames = 0;  // debug knob: force the WPE frame chunk (0 = one chunk)
  // Shape groups of one batch (segments sharing channel count and class tier) are independent: they are enqueued
  // on up to kGroupStreams streams so that one group's latency-bound kernels (FP64 update / solve, small grids)
  // run beside another group's sweeps. GSS_B200_GROUP_STREAMS=1 puts everything back on `stream`.
  static constexpr int kGroupStreams = 4;
  cudaStream_t side[kGroupStreams - 1] = {nullptr, nullptr, nullptr};
  cudaEvent_t fork_ev = nullptr, join_ev[kGroupStreams - 1] = {nullptr, nullptr, nullptr};
  int group_streams = kGroupStreams;
  cudaStream_t active = nullptr;  // stream the stage drivers launch on (null: `stream`)
  bool dev_call = false;     // inside a *_dev entry point: tensors are device memory, completion is an event
  long long nvtx_ranges = 0; // NVTX ranges opened by this context (gss_b200_nvtx_range_count)
};

namespace {

/// Stream the stage drivers (and the per-kernel clocks) enqueue on.
inline cudaStream_t S(gss_b200_ctx* c) { return c->active ? c->active : c->stream; }

gss_status fail(gss_b200_ctx* c, gss_status code, const std::string& msg, long long freq = -1) {
  if (c) {
    c->err = msg;
    c->err_freq = freq;
  }
  set_thread_error(code, msg, freq);
  return code;
}

/// Brackets one kernel launch with events when profiling is on, and counts it.
struct KClock {
  gss_b200_ctx* c;
  int id;
  cudaEvent_t b = nullptr;
  KClock(gss_b200_ctx* ctx, int kid) : c(ctx), id(kid) {
    ++c->launches;
    ++c->kernel_launches[id];
    if (!c->prof_on) return;
    cudaEvent_t a;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a, S(c));
    c->prof_recs.push_back({id, a, b});
  }
  ~KClock() {
    if (b) cudaEventRecord(b, S(c));
  }
};
/// NVTX range on the calling host thread, named after the reference's stage keys ("gss.stft", "gss.wpe", ...):
/// a profiler attributes the launches enqueued inside it to the stage. No tool attached = two empty calls.
struct NvtxRange {
  NvtxRange(gss_b200_ctx* c, const char* name) {
    if (c) ++c->nvtx_ranges;
    nvtxRangePushA(name);
  }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};

/// End of a stage entry point: the host variants return finished results; the *_dev variants return as soon as
/// the work is queued (DevCall makes the caller's stream wait for it).
inline cudaError_t finish_call(gss_b200_ctx* c) { return c->dev_call ? cudaSuccess : cudaStreamSynchronize(c->stream); }

/// Scope of a *_dev entry point: the context stream first waits for everything queued on the caller's stream,
/// and on exit the caller's stream waits for everything the call queued. No host synchronisation.
struct DevCall {
  gss_b200_ctx* c;
  cudaStream_t user;
  cudaEvent_t ev = nullptr;
  DevCall(gss_b200_ctx* ctx, void* stream) : c(ctx), user(reinterpret_cast<cudaStream_t>(stream)) {
    if (!c) return;
    cudaSetDevice(c->device);
    c->dev_call = true;
    if (cudaEventCreateWithFlags(&ev, cudaEventDisableTiming) != cudaSuccess) {
      ev = nullptr;
      return;
    }
    cudaEventRecord(ev, user);
    cudaStreamWaitEvent(c->stream, ev, 0);
    cudaStreamWaitEvent(c->copy_stream, ev, 0);  // enhance_batch moves the audio on its copy stream
  }
  ~DevCall() {
    if (!c) return;
    c->dev_call = false;
    if (ev) {
      cudaEventRecord(ev, c->stream);
      cudaStreamWaitEvent(user, ev, 0);
      cudaEventDestroy(ev);
    } else {
      cudaStreamSynchronize(c->stream);  // no event: fall back to a host wait, never to unordered work
    }
  }
};

/// A pair of timing events destroyed on every exit path.
struct EventPair {
  cudaEvent_t a = nullptr, b = nullptr;
  cudaError_t create() {
    cudaError_t e = cudaEventCreate(&a);
    return e != cudaSuccess ? e : cudaEventCreate(&b);
  }
  ~EventPair() {
    if (a) cudaEventDestroy(a);
    if (b) cudaEventDestroy(b);
  }
  EventPair() = default;
  EventPair(const EventPair&) = delete;
  EventPair& operator=(const EventPair&) = delete;
};
constexpr int kWpeFallbackSlots = 32;  // concurrent eigenvalue-floor repairs per WPE launch; further bins wait for a slot
enum KernelId { kK_stft = 0, kK_wpe_power, kK_wpe_gram, kK_wpe_solve, kK_wpe_apply, kK_em_pass, kK_em_update,
                kK_mvdr, kK_apply, kK_istft, kK_misc };

#define CU_TRY(ctx, expr)                                                                          \
  do {                                                                                             \
    cudaError_t e__ = (expr);                                                                      \
    if (e__ != cudaSuccess)                                                                        \
      return fail(ctx, GSS_CUDA_ERROR, std::string(#expr) + ": " + cudaGetErrorString(e__));      \
  } while (0)

const char* status_name(int code) {
  switch (code) {
    case GSS_SHAPE_ERROR: return "ShapeError";
    case GSS_CONFIG_ERROR: return "ConfigError";
    case GSS_SINGULAR_MATRIX_ERROR: return "SingularMatrixError";
    case GSS_INPUT_TOO_SHORT_ERROR: return "InputTooShortError";
    case GSS_EMPTY_TARGET_ERROR: return "EmptyTargetError";
    case GSS_DEGENERATE_STATS_ERROR: return "DegenerateStatsError";
    default: return "Error";
  }
}

// ---- configuration validation (stft.hpp:25-35, wpe.hpp:22-29, scheduler.hpp:46-57)
bool validate_stft(const gss_stft_config& s, std::string& why) {
  if (s.fft_size <= 0 || s.shift <= 0) return why = "stft: fft_size and shift must be positive", false;
  if (s.fft_size % s.shift != 0) return why = "stft: shift must divide fft_size for overlap-add", false;
  if (s.sample_rate <= 0) return why = "stft: sample_rate must be positive", false;
  return true;
}
bool validate_wpe(const gss_wpe_config& w, std::string& why) {
  if (w.taps < 1 || w.delay < 1 || w.iterations < 1)
    return why = "wpe: taps, delay and iterations must be >= 1", false;
  if (w.psd_context < 0 || w.regularization < 0.0)
    return why = "wpe: psd_context and regularization must be >= 0", false;
  return true;
}
bool kernel_fft_supported(const gss_stft_config& s, std::string& why) {
  const int n = s.fft_size;
  if ((n & (n - 1)) != 0 || n < 32 || n > 2048)
    return why = "fft_size must be a power of two in [32, 2048] on this device path", false;
  if (s.window != 0 && s.window != 1) return why = "stft: unknown window", false;
  return true;
}

// ---- device memory (stream-ordered pool; freed blocks are reused across batches)
struct DevMem {
  gss_b200_ctx* c = nullptr;
  std::vector<std::pair<void*, size_t>> blocks;
  cudaError_t last = cudaSuccess;
  template <typename T>
  T* get(size_t count) {
    if (last != cudaSuccess) return nullptr;
    size_t bytes = std::max<size_t>(count, 1) * sizeof(T) + 64;  // slack for aligned over-reads
    void* p = nullptr;
    last = cudaMallocAsync(&p, bytes, c->stream);
    if (last != cudaSuccess) return nullptr;
    blocks.emplace_back(p, bytes);
    c->device_bytes += (long long)bytes;
    c->device_bytes_peak = std::max(c->device_bytes_peak, c->device_bytes);
    return reinterpret_cast<T*>(p);
  }
  void release() {
    for (auto& b : blocks) {
      cudaFreeAsync(b.first, c->stream);
      c->device_bytes -= (long long)b.second;
    }
    blocks.clear();
  }
};

gss_status get_tables(gss_b200_ctx* c, const gss_stft_config& s, Tables& out) {
  const auto key = std::make_pair(s.fft_size, s.window);
  auto it = c->tables.find(key);
  if (it != c->tables.end()) {
    out = it->second;
    return GSS_OK;
  }
  const int n = s.fft_size;
  std::vector<float2> tw(n / 2);
  std::vector<float> win(n);
  std::vector<double2> tw_d(n / 2);
  std::vector<double> win_d(n);
  for (int k = 0; k < n / 2; ++k) {
    const double ang = -2.0 * M_PI * k / n;
    tw_d[k] = make_double2(std::cos(ang), std::sin(ang));
    tw[k] = make_float2((float)tw_d[k].x, (float)tw_d[k].y);
  }
  for (int i = 0; i < n; ++i) {  // stft.hpp:89-97
    const double h = 0.5 * (1.0 - std::cos(2.0 * M_PI * i / n));
    win_d[i] = s.window == 0 ? h : std::sqrt(h);
    win[i] = (float)win_d[i];
  }
  Tables t;
  CU_TRY(c, cudaMalloc(&t.tw, sizeof(float2) * (n / 2)));
  CU_TRY(c, cudaMalloc(&t.win, sizeof(float) * n));
  CU_TRY(c, cudaMalloc(&t.tw_d, sizeof(double2) * (n / 2)));
  CU_TRY(c, cudaMalloc(&t.win_d, sizeof(double) * n));
  CU_TRY(c, cudaMemcpyAsync(t.tw, tw.data(), sizeof(float2) * (n / 2), cudaMemcpyDefault, c->stream));
  CU_TRY(c, cudaMemcpyAsync(t.win, win.data(), sizeof(float) * n, cudaMemcpyDefault, c->stream));
  CU_TRY(c, cudaMemcpyAsync(t.tw_d, tw_d.data(), sizeof(double2) * (n / 2), cudaMemcpyDefault, c->stream));
  CU_TRY(c, cudaMemcpyAsync(t.win_d, win_d.data(), sizeof(double) * n, cudaMemcpyDefault, c->stream));
  CU_TRY(c, cudaStreamSynchronize(c->stream));
  c->tables[key] = t;
  out = t;
  return GSS_OK;
}

StftParams stft_params(const gss_stft_config& s) {
  StftParams p;
  p.fft_size = s.fft_size;
  p.shift = s.shift;
  p.window = s.window;
  p.F = s.fft_size / 2 + 1;
  p.log2n = ilog2(s.fft_size);
  return p;
}

// ---- one (M, KT) group of segments and its device arrays -----------------------
struct SegSpec {  // what the group builder needs to know about one segment
  long long N = 0;  // audio samples (or output length for synthesis-only groups)
  int T = 0, K = 1, target = 0, noise = -1;
  const uint8_t* activity = nullptr;  // (T,K) or null
  bool keep_gamma = false;
  int index = 0;
};

struct Needs {
  bool audio = false, y = false, yd = false, gamma = false, x = false, wave = false, em = false, wpe = false,
       mvdr = false;
};

struct Group {
  int M = 0, KT = 2, L = 1, F = 0, nseg = 0;
  int max_T = 0, npat_max = 1, cell_stride = 0, max_wchunks = 1, nwork = 0, iterations = 0;
  long long max_N = 0, nF = 0;
  std::vector<SegDev> segs;
  std::vector<int> members;  // caller indices
  DevMem mem;
  SegDev* d_segs = nullptr;
  WorkItem* d_work = nullptr;
  float* audio = nullptr;
  float2 *Y = nullptr, *Yd = nullptr, *X = nullptr;
  float *gamma = nullptr, *wave = nullptr;
  unsigned char* pat = nullptr;
  uint32_t* masks = nullptr;
  float *ck = nullptr, *coef = nullptr, *part = nullptr;
  double* cell_ll = nullptr;
  cdbl* bstate = nullptr;
  double *pi = nullptr, *logdet = nullptr, *bin_ll = nullptr, *seg_ll = nullptr;
  cdbl *phi_t = nullptr, *phi_b = nullptr, *h = nullptr;
  double* tmass = nullptr;
  float2* hconj = nullptr;
  float* w = nullptr;
  float2 *gram = nullptr, *gconj = nullptr;
  float* gram_raw = nullptr;
  int use_tc = 0;
  cdbl* fb_scratch = nullptr;
  int* fb_ticket = nullptr;
  status_t* status = nullptr;
  int *ref = nullptr, *zeroed = nullptr;
  long long tot_audio = 0, tot_y = 0, tot_g = 0, tot_x = 0, tot_wave = 0, tot_pat = 0, tot_mask = 0;
  // upload waves: segments [wave_first[w], wave_first[w + 1]) are copied together; the STFT and the WPE of wave w
  // run while wave w + 1 is still on the bus (everything after the WPE runs on the whole group)
  std::vector<int> wave_first;
  std::vector<cudaEvent_t> wave_ev;  // audio of wave w is in HBM
  std::vector<cudaEvent_t> marks;    // 2 per wave: after its STFT, after its WPE (stage clocks)
  int waves_copied = 0, waves_run = 0;
  int num_waves() const { return (int)wave_ev.size(); }
};

int pick_chunks(gss_b200_ctx* c, int T, long long ctas_one_chunk) {
  const int slots_mult = 256;  // 8 warps x 32-frame groups of the sweep (cacgmm_pass2.cuh)
  int nch = 1;
  if (c->em_chunk_frames > 0) {
    nch = (T + c->em_chunk_frames - 1) / c->em_chunk_frames;
  } else if (ctas_one_chunk < 148) {
    // one segment alone should still put a block on each of the 148 SMs; every extra chunk costs a sweep
    // prologue and a cell reduction per (segment, bin) (two half-length blocks per SM take as long as one)
    const int want = (int)((148 + ctas_one_chunk - 1) / ctas_one_chunk);
    nch = std::max(1, std::min(want, (T + 255) / 256));
  }
  int TC = (T + nch - 1) / nch;
  TC = ((TC + slots_mult - 1) / slots_mult) * slots_mult;
  return std::max(TC, slots_mult);
}

gss_status build_group(gss_b200_ctx* c, Group& g, int M, int K_for_tier, int F, const std::vector<SegSpec>& specs,
                       const Needs& need, const gss_wpe_config* wpe, int iterations) {
  g.M = M;
  g.KT = em_class_tier(K_for_tier);
  g.L = em_lanes(M, g.KT);
  g.F = F;
  g.nseg = (int)specs.size();
  g.iterations = iterations;
  g.mem.c = c;
  g.cell_stride = em_cell_floats(M, g.KT);
  const int ndof = em_ndof(M, g.L);
  const int km = wpe ? wpe->taps * M : 0;
  const int wcell = wpe ? wpe_gram_cell_elems(km, M) : 0;
  std::vector<unsigned char> h_pat;
  std::vector<uint32_t> h_masks;
  long long o_audio = 0, o_y = 0, o_g = 0, o_x = 0, o_wave = 0, o_tab = 0, o_coef = 0, o_cell = 0, o_fk = 0, o_f = 0,
            o_w = 0, o_wcell = 0, o_gw = 0;
  for (const SegSpec& s : specs) {
    SegDev d;
    std::memset(&d, 0, sizeof(d));
    d.N = (int)s.N;
    d.T = s.T;
    d.K = s.K;
    d.target = s.target;
    d.noise = s.noise;
    d.index = s.index;
    d.audio_off = o_audio;
    d.y_off = o_y;
    d.g_off = s.keep_gamma ? o_g : -1;
    d.x_off = o_x;
    d.wave_off = o_wave;
    d.pat_off = (long long)h_pat.size();
    d.mask_off = (long long)h_masks.size();
    // activity rows -> pattern ids (first-appearance order) + class bit masks
    if (s.activity != nullptr) {
      // K <= 8 classes: a row is one of at most 256 bit masks, so the id table is a flat array
      int id_of[256];
      std::fill(id_of, id_of + 256, -1);
      int nseen = 0;
      const size_t base = h_pat.size();
      h_pat.resize(base + (size_t)s.T);
      unsigned char* out_ids = h_pat.data() + base;
      const uint8_t* act = s.activity;
      for (int t = 0; t < s.T; ++t, act += s.K) {
        uint32_t m = 0;
        for (int k = 0; k < s.K; ++k) m |= (act[k] ? 1u : 0u) << k;
        int id = id_of[m];
        if (id < 0) {
          id = id_of[m] = nseen++;
          h_masks.push_back(m);
        }
        out_ids[t] = (unsigned char)id;
      }
      d.npat = nseen;
    } else {
      d.npat = 0;
    }
    g.npat_max = std::max(g.npat_max, d.npat);
    d.tab_off = o_tab;
    d.coef_off = o_coef;
    d.cell_off = o_cell;
    d.fk_off = o_fk;
    d.f_off = o_f;
    d.w_off = o_w;
    d.wcell_off = o_wcell;
    d.g_wpe_off = o_gw;
    d.TC = pick_chunks(c, s.T, F);  // a function of the segment alone: results do not depend on batch composition
    d.nchunks = (s.T + d.TC - 1) / d.TC;
    d.WTC = c->wpe_chunk_frames > 0 ? c->wpe_chunk_frames : std::max(s.T, 1);
    d.wchunks = (s.T + d.WTC - 1) / d.WTC;
    d.wpe_active = (wpe != nullptr && s.T > wpe->taps + wpe->delay) ? 1 : 0;
    g.max_wchunks = std::max(g.max_wchunks, d.wchunks);
    g.max_T = std::max(g.max_T, s.T);
    g.max_N = std::max(g.max_N, s.N);
    o_audio += (long long)M * s.N;
    o_y += (long long)F * s.T * M;
    if (s.keep_gamma) o_g += (long long)F * s.T * s.K;
    o_x += (long long)s.T * F;
    o_wave += s.N;
    o_tab += (long long)F * std::max(d.npat, 1) * g.KT;
    o_coef += (long long)F * g.L * g.KT * ndof;
    o_cell += (long long)F * d.nchunks;
    o_fk += (long long)F * g.KT;
    o_f += F;
    o_w += (long long)F * s.T;
    o_wcell += (long long)F * d.wchunks;
    o_gw += (long long)F * km * M;
    g.segs.push_back(d);
    g.members.push_back(s.index);
  }
  g.nF = o_f;
  g.tot_audio = o_audio;
  g.tot_y = o_y;
  g.tot_g = o_g;
  g.tot_x = o_x;
  g.tot_wave = o_wave;
  g.tot_pat = (long long)h_pat.size();
  g.tot_mask = (long long)h_masks.size();
  std::vector<WorkItem> work;
  for (int i = 0; i < g.nseg; ++i)
    for (int ch = 0; ch < g.segs[i].nchunks; ++ch) work.push_back(WorkItem{i, ch});
  g.nwork = (int)work.size();

  DevMem& m = g.mem;
  g.d_segs = m.get<SegDev>(g.nseg);
  g.d_work = m.get<WorkItem>(work.size());
  g.status = m.get<status_t>(g.nseg);
  g.ref = m.get<int>(g.nseg);
  g.zeroed = m.get<int>(g.nseg);
  g.seg_ll = m.get<double>((size_t)g.nseg * (iterations + 1));
  if (need.audio) g.audio = m.get<float>(o_audio);
  if (need.y) g.Y = m.get<float2>(o_y);
  if (need.yd) g.Yd = m.get<float2>(o_y);
  if (need.gamma && o_g > 0) g.gamma = m.get<float>(o_g);
  if (need.x) g.X = m.get<float2>(o_x);
  if (need.wave) g.wave = m.get<float>(o_wave);
  if (need.em) {
    g.pat = m.get<unsigned char>(h_pat.size());
    g.masks = m.get<uint32_t>(h_masks.size());
    g.ck = m.get<float>(o_tab);
    g.coef = m.get<float>(o_coef);
    g.bstate = m.get<cdbl>((size_t)o_fk * M * M);
    g.pi = m.get<double>(o_fk);
    g.logdet = m.get<double>(o_fk);
    g.bin_ll = m.get<double>((size_t)o_f * (iterations + 1));
  }
  if (need.em || need.mvdr) {
    g.part = m.get<float>((size_t)o_cell * g.cell_stride);
    g.cell_ll = m.get<double>(o_cell);
  }
  if (need.mvdr) {
    g.phi_t = m.get<cdbl>((size_t)o_f * M * M);
    g.phi_b = m.get<cdbl>((size_t)o_f * M * M);
    g.tmass = m.get<double>(o_f);
    g.h = m.get<cdbl>((size_t)o_f * M);
    g.hconj = m.get<float2>((size_t)o_f * M);
  }
  if (need.wpe) {
    g.w = m.get<float>(o_w);
    g.use_tc = (c->wpe_gram_tc == 1 || (c->wpe_gram_tc == 2 && M >= 4)) && wpe_tc_supported(km, M) && g.max_wchunks == 1;
    if (g.use_tc)
      g.gram_raw = m.get<float>((size_t)o_f * wpe_tc_cell_floats(km, M));
    else
      g.gram = m.get<float2>((size_t)o_wcell * wcell);
    g.gconj = m.get<float2>(o_gw);
    g.fb_scratch = m.get<cdbl>((size_t)kWpeFallbackSlots * wpe_fallback_slot_elems(km, M));
    g.fb_ticket = m.get<int>(kWpeFallbackSlots);  // one busy flag per slot
  }
  if (m.last != cudaSuccess) {
    const std::string why = std::string("device allocation failed: ") + cudaGetErrorString(m.last);
    m.release();
    return fail(c, GSS_CUDA_ERROR, why);
  }
  cudaStream_t st = c->stream;
  CU_TRY(c, cudaMemcpyAsync(g.d_segs, g.segs.data(), sizeof(SegDev) * g.nseg, cudaMemcpyDefault, st));
  if (!work.empty())
    CU_TRY(c, cudaMemcpyAsync(g.d_work, work.data(), sizeof(WorkItem) * work.size(), cudaMemcpyDefault, st));
  CU_TRY(c, cudaMemsetAsync(g.status, 0xFF, sizeof(status_t) * g.nseg, st));
  CU_TRY(c, cudaMemsetAsync(g.zeroed, 0, sizeof(int) * g.nseg, st));
  CU_TRY(c, cudaMemsetAsync(g.ref, 0, sizeof(int) * g.nseg, st));
  if (need.em && !h_pat.empty()) {
    CU_TRY(c, cudaMemcpyAsync(g.pat, h_pat.data(), h_pat.size(), cudaMemcpyDefault, st));
    CU_TRY(c, cudaMemcpyAsync(g.masks, h_masks.data(), sizeof(uint32_t) * h_masks.size(), cudaMemcpyDefault, st));
  }
  // pageable sources above (std::vector) are consumed synchronously by cudaMemcpyAsync's
  // staging, so they may go out of scope on return.
  return GSS_OK;
}

// ---- stage drivers (device side only) ---------------------------------------------
gss_status run_wpe(gss_b200_ctx* c, Group& g, const gss_wpe_config& w, int first = 0, int count = -1) {
  if (count < 0) count = g.nseg - first;
  bool any = false;
  for (int j = first; j < first + count; ++j) {
    const SegDev& d = g.segs[j];
    if (d.wpe_active) {
      any = true;
    } else {  // pass-through (wpe.hpp:108-112)
      CU_TRY(c, cudaMemcpyAsync(g.Yd + d.y_off, g.Y + d.y_off, sizeof(float2) * (size_t)g.F * d.T * g.M,
                                cudaMemcpyDeviceToDevice, S(c)));
    }
  }
  if (!any) return GSS_OK;
  WpeArgs a;
  a.yobs = g.Y;
  a.yout = g.Yd;
  a.w = g.w;
  a.gram = g.gram;
  a.gram_raw = g.gram_raw;
  a.use_tc = g.use_tc;
  a.gram_f16 = c->wpe_gram_f16;
  a.apply_f16 = c->wpe_apply_f16;
  a.apply_tc = (c->wpe_apply_tc == 1 || (c->wpe_apply_tc == 2 && g.M >= 4)) &&
               wpe_apply_tc_supported(w.taps, w.delay, g.M);
  a.debug_rp = nullptr;
  a.w_next = nullptr;
  a.fb_scratch = g.fb_scratch;
  a.fb_ticket = g.fb_ticket;
  a.fb_slots = kWpeFallbackSlots;
  a.gconj = g.gconj;
  a.segs = g.d_segs + first;  // kernels index segments and their status from the launch's first one
  a.status = g.status + first;
  a.regularization = w.regularization;
  a.M = g.M;
  a.taps = w.taps;
  a.delay = w.delay;
  a.psd_context = w.psd_context;
  // With psd_context 0 the next iteration's weights are the power of the frames the prediction kernel has just
  // written: the tensor-core kernel emits them and the power pass runs for the first iteration only.
  const bool fuse_power = a.apply_tc && w.psd_context == 0;
  bool w_ready = false;
  for (int it = 0; it < w.iterations; ++it) {
    a.ycur = it == 0 ? g.Y : g.Yd;
    a.w_next = fuse_power && it + 1 < w.iterations ? g.w : nullptr;
    CU_TRY(c, cudaMemsetAsync(g.fb_ticket, 0, sizeof(int) * kWpeFallbackSlots, S(c)));
    for (int step = 0; step < 4; ++step) {
      if (step == 0 && w_ready) continue;
      KClock k(c, kK_wpe_power + step);
      CU_TRY(c, launch_wpe_step(step, a, count, g.F, g.max_T, g.max_wchunks, S(c)));
    }
    w_ready = a.w_next != nullptr;
  }
  return GSS_OK;
}

struct EmRun {
  const float2* tensor;
  int normalize;
  bool final_stats;
  bool from_state;
  bool all_ll;  // reduce every sweep's likelihood (stage API) instead of only the last
};

gss_status run_em(gss_b200_ctx* c, Group& g, const EmRun& r) {
  const EmShape shape{g.M, g.KT};
  const int I = g.iterations;
  EmUpdateArgs u;
  u.segs = g.d_segs;
  u.masks = g.masks;
  u.part = g.part;
  u.cell_ll = g.cell_ll;
  u.bstate = g.bstate;
  u.pi = g.pi;
  u.logdet = g.logdet;
  u.coef = g.coef;
  u.ck = g.ck;
  u.bin_ll = g.bin_ll;
  u.status = g.status;
  u.c0 = -(double)g.M * std::log(2.0 * M_PI) + std::lgamma((double)g.M);
  u.cell_stride = g.cell_stride;
  u.F = g.F;
  u.mode = r.from_state ? kEmFromState : kEmInit;
  {
    KClock k(c, kK_em_update);
    CU_TRY(c, launch_em_update(shape, u, g.nseg, S(c)));
  }
  EmPassArgs p;
  p.y = r.tensor;
  p.segs = g.d_segs;
  p.work = g.d_work;
  p.pat = g.pat;
  p.ck = g.ck;
  p.coef = g.coef;
  p.part = g.part;
  p.cell_ll = g.cell_ll;
  p.gamma = nullptr;
  p.cell_stride = g.cell_stride;
  p.npat_max = g.npat_max;
  p.normalize = r.normalize;
  for (int it = 0; it < I; ++it) {
    {
      KClock k(c, kK_em_pass);
      CU_TRY(c, launch_em_pass(shape, false, p, g.nwork, g.F, S(c)));
    }
    u.mode = kEmMstep;
    u.bin_ll = g.bin_ll + (long long)it * g.nF;
    {
      KClock k(c, kK_em_update);
      CU_TRY(c, launch_em_update(shape, u, g.nseg, S(c)));
    }
  }
  p.gamma = g.gamma;
  {
    KClock k(c, kK_em_pass);
    CU_TRY(c, launch_em_pass(shape, r.final_stats, p, g.nwork, g.F, S(c)));
  }
  u.mode = kEmFinal;
  u.bin_ll = g.bin_ll + (long long)I * g.nF;
  {
    KClock k(c, kK_em_update);
    CU_TRY(c, launch_em_update(shape, u, g.nseg, S(c)));
  }
  for (int it = r.all_ll ? 0 : I; it <= I; ++it) {
    KClock k(c, kK_misc);
    CU_TRY(c, launch_sum_ll(g.bin_ll + (long long)it * g.nF, g.seg_ll + (long long)it * g.nseg, g.d_segs, g.nseg,
                            g.F, S(c)));
  }
  return GSS_OK;
}

gss_status run_mvdr_design(gss_b200_ctx* c, Group& g, int fixed_ref, bool have_tmass) {
  MvdrArgs a;
  a.segs = g.d_segs;
  a.phi_t = g.phi_t;
  a.phi_b = g.phi_b;
  a.tmass = have_tmass ? g.tmass : nullptr;
  a.ref = g.ref;
  a.zeroed = g.zeroed;
  a.h = g.h;
  a.hconj = g.hconj;
  a.status = g.status;
  a.M = g.M;
  a.F = g.F;
  a.fixed_ref = fixed_ref;
  {
    KClock k(c, kK_mvdr);
    CU_TRY(c, launch_select_reference(a, g.nseg, S(c)));
  }
  {
    KClock k(c, kK_mvdr);
    CU_TRY(c, launch_mvdr_solve(a, g.nseg, S(c)));
  }
  return GSS_OK;
}

}  // namespace

// ===========================================================================
// batch object
// ===========================================================================
struct gss_b200_batch {
  gss_pipeline_config cfg;
  int n = 0;
  std::vector<gss_segment_desc> desc;
  std::vector<std::vector<int64_t>> pb, pe;
  std::vector<Fail> fails;           // per segment host-side verdicts (code 0 = ok)
  std::vector<int> frames;
  std::vector<std::unique_ptr<Group>> groups;
  std::vector<cudaEvent_t> events;   // 6 per group + 2 around upload
  bool ran = false;
  Tables tables;
};

namespace {

void free_batch(gss_b200_ctx* c, gss_b200_batch* b) {
  if (!b) return;
  for (auto& g : b->groups) {
    // the copy stream may still be writing into the group's audio when a failed call is torn down
    if (c && g->waves_copied > 0) cudaStreamSynchronize(c->copy_stream);
    g->mem.release();
    for (cudaEvent_t e : g->wave_ev)
      if (e) cudaEventDestroy(e);
    for (cudaEvent_t e : g->marks)
      if (e) cudaEventDestroy(e);
  }
  for (cudaEvent_t e : b->events)
    if (e) cudaEventDestroy(e);
  delete b;
  (void)c;
}

/// Queues the host->device copies of wave w's audio on the copy stream and marks their end.
gss_status copy_wave(gss_b200_ctx* c, gss_b200_batch* b, Group& g, int w) {
  for (int j = g.wave_first[w]; j < g.wave_first[w + 1]; ++j) {
    const gss_segment_desc& d = b->desc[g.members[j]];
    CU_TRY(c, cudaMemcpyAsync(g.audio + g.segs[j].audio_off, d.audio,
                              sizeof(float) * (size_t)d.channels * d.num_samples, cudaMemcpyDefault,
                              c->copy_stream));
  }
  CU_TRY(c, cudaEventRecord(g.wave_ev[w], c->copy_stream));
  g.waves_copied = w + 1;
  return GSS_OK;
}

gss_status upload_impl(gss_b200_ctx* c, int32_t n, const gss_segment_desc* segs, const gss_pipeline_config* cfg,
                       bool copy_now, gss_b200_batch** out);
gss_status run_impl(gss_b200_ctx* c, gss_b200_batch* b);

}  // namespace

extern "C" {

void gss_b200_default_stft_config(gss_stft_config* c) {
  c->fft_size = 1024;
  c->shift = 256;
  c->window = 0;
  c->sample_rate = 16000;
}
void gss_b200_default_wpe_config(gss_wpe_config* c) {
  c->taps = 10;
  c->delay = 2;
  c->iterations = 3;
  c->psd_context = 0;
  c->regularization = 1e-10;
}
void gss_b200_default_pipeline_config(gss_pipeline_config* c) {
  gss_b200_default_stft_config(&c->stft);
  gss_b200_default_wpe_config(&c->wpe);
  c->enable_wpe = 1;
  c->bss_iterations = 20;
}

gss_status gss_b200_create(int device, gss_b200_ctx** out) {
  *out = nullptr;
  int count = 0;
  cudaError_t e = cudaGetDeviceCount(&count);
  if (e != cudaSuccess || count <= 0)
    return fail(nullptr, GSS_CUDA_ERROR,
                std::string("no CUDA device available (") + cudaGetErrorString(e) +
                    "); libgss_b200 has no CPU fallback");
  if (device < 0 || device >= count) return fail(nullptr, GSS_CUDA_ERROR, "device index out of range");
  CU_TRY(nullptr, cudaSetDevice(device));
  cudaDeviceProp prop;
  CU_TRY(nullptr, cudaGetDeviceProperties(&prop, device));
  if (prop.major < 10)
    return fail(nullptr, GSS_CUDA_ERROR, "libgss_b200 is built for sm_100a (B200) only");
  auto* c = new gss_b200_ctx();
  c->device = device;
  e = cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking);
  if (e != cudaSuccess) {
    delete c;
    return fail(nullptr, GSS_CUDA_ERROR, cudaGetErrorString(e));
  }
  e = cudaStreamCreateWithFlags(&c->copy_stream, cudaStreamNonBlocking);
  if (e != cudaSuccess) {
    cudaStreamDestroy(c->stream);
    delete c;
    return fail(nullptr, GSS_CUDA_ERROR, cudaGetErrorString(e));
  }
  if (const char* sg = std::getenv("GSS_B200_GROUP_STREAMS"))
    c->group_streams = std::min<int>(gss_b200_ctx::kGroupStreams, std::max(1, std::atoi(sg)));
  bool side_ok = cudaEventCreateWithFlags(&c->fork_ev, cudaEventDisableTiming) == cudaSuccess;
  for (int i = 0; i < gss_b200_ctx::kGroupStreams - 1 && side_ok; ++i)
    side_ok = cudaStreamCreateWithFlags(&c->side[i], cudaStreamNonBlocking) == cudaSuccess &&
              cudaEventCreateWithFlags(&c->join_ev[i], cudaEventDisableTiming) == cudaSuccess;
  if (!side_ok) c->group_streams = 1;  // the single-stream path needs none of them
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
    unsigned long long thr = ~0ull;  // keep freed blocks cached for the next batch
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
  }
  if (const char* s = std::getenv("GSS_B200_WPE_GRAM")) c->wpe_gram_tc = std::strcmp(s, "fp32") == 0 ? 0 : std::strcmp(s, "tc") == 0 ? 1 : 2;
  if (const char* s = std::getenv("GSS_B200_WPE_GRAM_KIND")) c->wpe_gram_f16 = std::strcmp(s, "tf32") == 0 ? 0 : 1;
  if (const char* s = std::getenv("GSS_B200_WPE_APPLY_KIND")) c->wpe_apply_f16 = std::strcmp(s, "tf32") == 0 ? 0 : 1;
  if (const char* s = std::getenv("GSS_B200_WPE_APPLY")) c->wpe_apply_tc = std::strcmp(s, "fp32") == 0 ? 0 : std::strcmp(s, "tc") == 0 ? 1 : 2;
  if (const char* s = std::getenv("GSS_B200_EM_CHUNK_FRAMES")) c->em_chunk_frames = std::atoi(s);
  if (const char* s = std::getenv("GSS_B200_WPE_CHUNK_FRAMES")) c->wpe_chunk_frames = std::atoi(s);
  if (const char* s = std::getenv("GSS_B200_WAVES")) c->waves = std::max(1, std::atoi(s));
  if (const char* s = std::getenv("GSS_B200_WAVE_MIN_FLOATS")) c->wave_min_floats = std::max(1LL, std::atoll(s));
  if (const char* s = std::getenv("GSS_B200_WAVE_FIRST_PCT"))
    c->wave_first_frac = std::min(100, std::max(1, std::atoi(s))) * 0.01;
  if (const char* s = std::getenv("GSS_B200_WAVE_GROWTH")) c->wave_growth = std::min(64.0, std::max(1.0, std::atof(s)));
  *out = c;
  return GSS_OK;
}

void gss_b200_destroy(gss_b200_ctx* c) {
  if (!c) return;
  cudaSetDevice(c->device);
  cudaStreamSynchronize(c->stream);
  cudaStreamSynchronize(c->copy_stream);
  cudaStreamDestroy(c->copy_stream);
  for (int i = 0; i < gss_b200_ctx::kGroupStreams - 1; ++i) {
    if (c->side[i]) {
      cudaStreamSynchronize(c->side[i]);
      cudaStreamDestroy(c->side[i]);
    }
    if (c->join_ev[i]) cudaEventDestroy(c->join_ev[i]);
  }
  if (c->fork_ev) cudaEventDestroy(c->fork_ev);
  for (auto& kv : c->tables) {
    cudaFree(kv.second.tw);
    cudaFree(kv.second.win);
    cudaFree(kv.second.tw_d);
    cudaFree(kv.second.win_d);
  }
  cudaStreamDestroy(c->stream);
  delete c;
}

const char* gss_b200_last_error(const gss_b200_ctx* c) { return c ? c->err.c_str() : t_err.c_str(); }
int64_t gss_b200_last_error_frequency(const gss_b200_ctx* c) { return c ? c->err_freq : t_err_freq; }
void* gss_b200_stream(gss_b200_ctx* c) { return c ? (void*)c->stream : nullptr; }
int64_t gss_b200_launch_count(const gss_b200_ctx* c) { return c ? c->launches : 0; }
int64_t gss_b200_device_bytes(const gss_b200_ctx* c) { return c ? c->device_bytes : 0; }
int64_t gss_b200_device_bytes_peak(gss_b200_ctx* c, int32_t reset) {
  if (!c) return 0;
  const long long peak = c->device_bytes_peak;
  if (reset) c->device_bytes_peak = c->device_bytes;
  return peak;
}

gss_status gss_b200_host_alloc(int64_t bytes, void** out) {
  *out = nullptr;
  cudaError_t e = cudaMallocHost(out, (size_t)std::max<int64_t>(bytes, 1));
  if (e != cudaSuccess) return fail(nullptr, GSS_CUDA_ERROR, cudaGetErrorString(e));
  return GSS_OK;
}
void gss_b200_host_free(void* p) {
  if (p) cudaFreeHost(p);
}

gss_status gss_b200_profile(gss_b200_ctx* c, int32_t enable) {
  cudaStreamSynchronize(c->stream);
  for (auto& r : c->prof_recs) {
    cudaEventDestroy(r.a);
    cudaEventDestroy(r.b);
  }
  c->prof_recs.clear();
  for (int i = 0; i < GSS_B200_NUM_KERNELS; ++i) {
    c->kernel_ms[i] = 0.0;
    c->kernel_launches[i] = 0;
  }
  c->prof_on = enable != 0;
  return GSS_OK;
}

gss_status gss_b200_kernel_ms(gss_b200_ctx* c, double* ms, int64_t* launches) {
  CU_TRY(c, cudaStreamSynchronize(c->stream));
  for (auto& r : c->prof_recs) {
    float t = 0.f;
    if (cudaEventElapsedTime(&t, r.a, r.b) == cudaSuccess) c->kernel_ms[r.id] += t;
    cudaEventDestroy(r.a);
    cudaEventDestroy(r.b);
  }
  c->prof_recs.clear();
  for (int i = 0; i < GSS_B200_NUM_KERNELS; ++i) {
    ms[i] = c->kernel_ms[i];
    launches[i] = c->kernel_launches[i];
  }
  return GSS_OK;
}

gss_status gss_b200_fp32_peak(gss_b200_ctx* c, double* tflops) {
  CU_TRY(c, cudaSetDevice(c->device));
  float* scratch = nullptr;
  CU_TRY(c, cudaMalloc(&scratch, 256));
  cudaDeviceProp prop;
  CU_TRY(c, cudaGetDeviceProperties(&prop, c->device));
  const int ctas = prop.multiProcessorCount * 8, iters = 2048;
  EventPair ev;
  CU_TRY(c, ev.create());
  cudaEvent_t a = ev.a, b = ev.b;
  double best = 0.0;
  for (int rep = 0; rep < 6; ++rep) {
    cudaEventRecord(a, c->stream);
    cudaError_t e = launch_fma_peak(scratch, ctas, iters, c->stream);
    cudaEventRecord(b, c->stream);
    cudaEventSynchronize(b);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, a, b);
    if (e == cudaSuccess && rep > 0 && ms > 0.f)
      best = std::max(best, 2.0 * 256.0 * iters * 256.0 * ctas / (ms * 1e-3) * 1e-12);
  }
  cudaFree(scratch);
  *tflops = best;
  return GSS_OK;
}

gss_status gss_b200_stage_ms(gss_b200_ctx* c, double* ms) {
  for (int i = 0; i < GSS_B200_NUM_STAGES; ++i) ms[i] = c->stage_ms[i];
  return GSS_OK;
}

// ---------------------------------------------------------------------------
// enhance_batch = upload + run + fetch
// ---------------------------------------------------------------------------
}  // extern "C"

namespace {

gss_status upload_impl(gss_b200_ctx* c, int32_t n, const gss_segment_desc* segs, const gss_pipeline_config* cfg,
                       bool copy_now, gss_b200_batch** out) {
  *out = nullptr;
  if (!c) return fail(nullptr, GSS_INTERNAL_ERROR, "null context");
  CU_TRY(c, cudaSetDevice(c->device));
  std::string why;
  // same order as PipelineConfig::validate (scheduler.hpp:46-57)
  if (cfg->bss_iterations < 1) return fail(c, GSS_CONFIG_ERROR, "scheduler: bss_iterations must be >= 1");
  if (!validate_wpe(cfg->wpe, why)) return fail(c, GSS_CONFIG_ERROR, why);
  if (!validate_stft(cfg->stft, why)) return fail(c, GSS_CONFIG_ERROR, why);
  if (!kernel_fft_supported(cfg->stft, why)) return fail(c, GSS_UNSUPPORTED, why);
  if (n < 0) return fail(c, GSS_SHAPE_ERROR, "negative segment count");
  auto* b = new gss_b200_batch();
  b->cfg = *cfg;
  b->n = n;
  b->desc.assign(segs, segs + n);
  b->pb.resize(n);
  b->pe.resize(n);
  b->fails.assign(n, Fail{GSS_OK, "", -1});
  b->frames.assign(n, 0);
  gss_status rc = get_tables(c, cfg->stft, b->tables);
  if (rc != GSS_OK) {
    delete b;
    return rc;
  }
  const int F = cfg->stft.fft_size / 2 + 1;
  // host-side validation per segment, in the order the reference would raise
  std::map<std::pair<int, int>, std::vector<SegSpec>> by_shape;
  for (int i = 0; i < n; ++i) {
    const gss_segment_desc& d = b->desc[i];
    Fail& fl = b->fails[i];
    b->pb[i].assign(d.part_begin, d.part_begin + std::max(d.num_parts, 0));
    b->pe[i].assign(d.part_end, d.part_end + std::max(d.num_parts, 0));
    if (d.channels < 1) {
      fl = Fail{GSS_SHAPE_ERROR, "stft.analyze: no channels", -1};
    } else if (d.num_samples < cfg->stft.fft_size) {
      fl = Fail{GSS_INPUT_TOO_SHORT_ERROR, "stft.analyze: fewer samples than fft_size", -1};
    } else if (d.sample_rate > 0 && d.sample_rate != cfg->stft.sample_rate) {
      fl = Fail{GSS_CONFIG_ERROR, "stft.analyze: signal/config sample rate mismatch", -1};
    } else if (d.channels > kMaxChannels || d.num_classes > kMaxClasses) {
      fl = Fail{GSS_UNSUPPORTED, "more than 8 channels or classes", -1};
    } else if (d.num_samples > 0x7fffffffLL) {
      fl = Fail{GSS_UNSUPPORTED, "segment longer than 2^31 samples", -1};
    }
    if (fl.code != GSS_OK) continue;
    const int64_t T = gss_b200_frame_count(d.num_samples, cfg->stft.fft_size, cfg->stft.shift);
    b->frames[i] = (int)T;
    if (d.activity_frames != T) {
      fl = Fail{GSS_SHAPE_ERROR, "cacgmm: activity frames do not match tensor", -1};
    } else if (d.num_classes < 1 || d.target_index < 0 || d.target_index >= d.num_classes) {
      fl = Fail{GSS_SHAPE_ERROR, "accumulate_stats: target class out of range", -1};
    } else {
      for (int p = 0; p < d.num_parts; ++p)
        if (b->pb[i][p] < 0 || b->pb[i][p] > std::min<int64_t>(b->pe[i][p], d.num_samples))
          fl = Fail{GSS_SHAPE_ERROR, "part offsets outside the assembled audio", -1};
    }
    if (fl.code != GSS_OK) continue;
    SegSpec s;
    s.N = d.num_samples;
    s.T = (int)T;
    s.K = d.num_classes;
    s.target = d.target_index;
    s.noise = d.noise_index;
    s.activity = d.activity;
    s.keep_gamma = d.gamma_out != nullptr;
    s.index = i;
    by_shape[std::make_pair(d.channels, em_class_tier(d.num_classes))].push_back(s);
  }
  b->events.assign(2 + 6 * by_shape.size(), nullptr);
  for (auto& e : b->events)
    if (cudaError_t ce = cudaEventCreate(&e); ce != cudaSuccess) {
      free_batch(c, b);
      return fail(c, GSS_CUDA_ERROR, std::string("cudaEventCreate: ") + cudaGetErrorString(ce));
    }
  cudaEventRecord(b->events[0], c->stream);
  Needs need;
  need.audio = need.y = need.x = need.wave = need.em = need.mvdr = true;
  need.yd = need.wpe = cfg->enable_wpe != 0;
  need.gamma = true;
  for (auto& kv : by_shape) {
    std::unique_ptr<Group> g(new Group());
    rc = build_group(c, *g, kv.first.first, kv.first.second, F, kv.second, need,
                     cfg->enable_wpe ? &cfg->wpe : nullptr, cfg->bss_iterations);
    if (rc != GSS_OK) {
      g->mem.release();
      free_batch(c, b);
      return rc;
    }
    // Waves of whole segments. Only the first wave's upload is exposed, so it is small; the STFT + WPE of a wave
    // take about 4x the bus time of its bytes on the headline shapes, so every wave may be ~4x the previous one and
    // still have its upload covered: three waves of 1 : 4 : 16 (5 % of the audio exposed). Small launches pay in
    // tail effects, so no wave is below ~8 MB.
    {
      long long floats = 0;
      for (int j = 0; j < g->nseg; ++j) floats += (long long)g->M * g->segs[j].N;
      const long long min_wave = c->wave_min_floats;
      double geo = 0.0, term = 1.0;
      for (int w = 0; w < c->waves; ++w, term *= c->wave_growth) geo += term;
      const double first_frac = c->wave_first_frac > 0.0 ? c->wave_first_frac : 1.0 / geo;
      long long acc = 0;
      double want = std::max<double>((double)floats * first_frac, (double)min_wave);
      long long target = c->waves > 1 ? (long long)want : floats + 1;
      g->wave_first.push_back(0);
      for (int j = 0; j < g->nseg; ++j) {
        acc += (long long)g->M * g->segs[j].N;
        if (acc >= target && j + 1 < g->nseg && (int)g->wave_first.size() < c->waves) {
          g->wave_first.push_back(j + 1);
          acc = 0;
          want = std::max<double>(want * c->wave_growth, (double)min_wave);
          target = (long long)want;
        }
      }
      g->wave_first.push_back(g->nseg);
      const int nw = (int)g->wave_first.size() - 1;
      g->wave_ev.assign(nw, nullptr);
      g->marks.assign(2 * nw, nullptr);
      cudaError_t ce = cudaSuccess;
      for (auto& e : g->wave_ev)
        if (ce == cudaSuccess) ce = cudaEventCreate(&e);
      for (auto& e : g->marks)
        if (ce == cudaSuccess) ce = cudaEventCreate(&e);
      if (ce != cudaSuccess) {
        b->groups.push_back(std::move(g));  // free_batch destroys what was created
        free_batch(c, b);
        return fail(c, GSS_CUDA_ERROR, std::string("cudaEventCreate: ") + cudaGetErrorString(ce));
      }
    }
    b->groups.push_back(std::move(g));
  }
  // the buffers are stream-ordered allocations of the compute stream: the copy stream starts behind them (and
  // behind whatever the compute stream was still doing with the pool's memory)
  cudaEventRecord(b->events[1], c->stream);
  cudaStreamWaitEvent(c->copy_stream, b->events[1], 0);
  if (copy_now)
    for (auto& g : b->groups)
      for (int w = 0; w < g->num_waves(); ++w) {
        rc = copy_wave(c, b, *g, w);
        if (rc != GSS_OK) {
          free_batch(c, b);
          return rc;
        }
      }
  *out = b;
  return GSS_OK;
}

gss_status run_impl(gss_b200_ctx* c, gss_b200_batch* b) {
  CU_TRY(c, cudaSetDevice(c->device));
  const gss_pipeline_config& cfg = b->cfg;
  const StftParams sp = stft_params(cfg.stft);
  int gi = 0;
  // fork: several shape groups -> several streams (see gss_b200_ctx::side); joined again below and on every exit
  // (per-kernel event clocks are only meaningful for serialised launches: profiling keeps everything on one stream)
  const int nstreams = c->prof_on ? 1 : std::min<int>((int)b->groups.size(), c->group_streams);
  struct Join {
    gss_b200_ctx* c;
    int n;
    ~Join() {
      c->active = nullptr;
      for (int i = 1; i < n; ++i) {
        cudaEventRecord(c->join_ev[i - 1], c->side[i - 1]);
        cudaStreamWaitEvent(c->stream, c->join_ev[i - 1], 0);
      }
    }
  } join{c, nstreams};
  if (nstreams > 1) {
    cudaEventRecord(c->fork_ev, c->stream);
    for (int i = 1; i < nstreams; ++i) cudaStreamWaitEvent(c->side[i - 1], c->fork_ev, 0);
  }
  for (auto& gp : b->groups) {
    Group& g = *gp;
    c->active = nstreams > 1 && gi % nstreams > 0 ? c->side[gi % nstreams - 1] : nullptr;
    cudaEvent_t* ev = &b->events[2 + 6 * gi++];
    cudaStream_t st = S(c);
    // device-side state that a previous run of the same batch may have touched
    CU_TRY(c, cudaMemsetAsync(g.status, 0xFF, sizeof(status_t) * g.nseg, st));
    CU_TRY(c, cudaMemsetAsync(g.zeroed, 0, sizeof(int) * g.nseg, st));
    cudaEventRecord(ev[0], st);
    const float2* tensor = cfg.enable_wpe ? g.Yd : g.Y;
    if (g.waves_copied == 0) {
      gss_status rc = copy_wave(c, b, g, 0);
      if (rc != GSS_OK) return rc;
    }
    // a batch whose audio was all queued at upload time (the resident form) runs as one wave
    const bool resident = g.waves_copied == g.num_waves();
    g.waves_run = resident ? 1 : g.num_waves();
    for (int w = 0; w < g.waves_run; ++w) {
      const int first = resident ? 0 : g.wave_first[w], count = resident ? g.nseg : g.wave_first[w + 1] - first;
      for (int v = resident ? 0 : w; v <= (resident ? g.num_waves() - 1 : w); ++v)
        CU_TRY(c, cudaStreamWaitEvent(st, g.wave_ev[v], 0));
      {
        NvtxRange nv(c, "gss.stft");
        StftArgs a;
        a.audio = g.audio;
        a.y = g.Y;
        a.segs = g.d_segs + first;
        a.tw_d = b->tables.tw_d;
        a.win_d = b->tables.win_d;
        a.p = sp;
        a.M = g.M;
        a.TB = 0;
        a.fft_warps = 0;
        KClock k(c, kK_stft);
        CU_TRY(c, launch_stft(a, count, g.max_T, st));
      }
      cudaEventRecord(g.marks[2 * w], st);
      if (cfg.enable_wpe) {
        NvtxRange nv(c, "gss.wpe");
        gss_status rc = run_wpe(c, g, cfg.wpe, first, count);
        if (rc != GSS_OK) return rc;
      }
      cudaEventRecord(g.marks[2 * w + 1], st);
      // the next wave's audio goes on the bus behind this wave's launches: with pageable host memory the copy
      // call blocks the host, and the device works through this wave meanwhile
      if (!resident && w + 1 < g.num_waves() && g.waves_copied <= w + 1) {
        gss_status rc = copy_wave(c, b, g, w + 1);
        if (rc != GSS_OK) return rc;
      }
    }
    cudaEventRecord(ev[1], st);
    cudaEventRecord(ev[2], st);
    {
      NvtxRange nv(c, "gss.mask");
      EmRun r{tensor, 1, true, false, false};
      gss_status rc = run_em(c, g, r);
      if (rc != GSS_OK) return rc;
    }
    cudaEventRecord(ev[3], st);
    {
      NvtxRange nv(c, "gss.beamform");
      StatsFinalArgs sf;
      sf.segs = g.d_segs;
      sf.part = g.part;
      sf.phi_t = g.phi_t;
      sf.phi_b = g.phi_b;
      sf.tmass = g.tmass;
      sf.cell_stride = g.cell_stride;
      sf.F = g.F;
      {
        KClock k(c, kK_mvdr);
        CU_TRY(c, launch_mvdr_stats_final(EmShape{g.M, g.KT}, sf, g.nseg, st));
      }
      gss_status rc = run_mvdr_design(c, g, -1, true);
      if (rc != GSS_OK) return rc;
      ApplyArgs aa;
      aa.y = tensor;
      aa.hconj = g.hconj;
      aa.x = g.X;
      aa.segs = g.d_segs;
      aa.M = g.M;
      aa.F = g.F;
      aa.frame_major = 1;
      KClock k(c, kK_apply);
      CU_TRY(c, launch_apply(aa, g.nseg, g.max_T, st));
    }
    cudaEventRecord(ev[4], st);
    {
      NvtxRange nv(c, "gss.istft");
      IstftArgs ia;
      ia.x = g.X;
      ia.wave = g.wave;
      ia.segs = g.d_segs;
      ia.tw = b->tables.tw;
      ia.win = b->tables.win;
      ia.p = sp;
      ia.HB = 0;
      KClock k(c, kK_istft);
      CU_TRY(c, launch_istft(ia, g.nseg, g.max_N, st));
    }
    cudaEventRecord(ev[5], st);
  }
  b->ran = true;
  return GSS_OK;
}

}  // namespace

extern "C" {

gss_status gss_b200_batch_upload(gss_b200_ctx* c, int32_t n, const gss_segment_desc* segs,
                                 const gss_pipeline_config* cfg, gss_b200_batch** out) {
  return upload_impl(c, n, segs, cfg, /*copy_now=*/true, out);
}

gss_status gss_b200_batch_run(gss_b200_ctx* c, gss_b200_batch* b) { return run_impl(c, b); }

gss_status gss_b200_batch_fetch(gss_b200_ctx* c, gss_b200_batch* b, gss_segment_diag* diags) {
  CU_TRY(c, cudaSetDevice(c->device));
  if (!b->ran) return fail(c, GSS_INTERNAL_ERROR, "batch_fetch before batch_run");
  NvtxRange nv(c, "gss.d2h");
  cudaStream_t st = c->stream;
  const int F = b->cfg.stft.fft_size / 2 + 1;
  const int I = b->cfg.bss_iterations;
  for (int i = 0; i < b->n; ++i) {
    diags[i].status = b->fails[i].code;
    diags[i].ref_channel = 0;
    diags[i].error_frequency = b->fails[i].freq;
    diags[i].zeroed_bins = 0;
    diags[i].frames = b->frames[i];
    diags[i].ll_final = 0.0;
    for (int p = 0; p < b->desc[i].num_parts; ++p) b->desc[i].out_lengths[p] = 0;
  }
  EventPair d2h;
  CU_TRY(c, d2h.create());
  cudaEvent_t d2h0 = d2h.a, d2h1 = d2h.b;
  cudaEventRecord(d2h0, st);
  // small per-segment results first (they decide which waveforms are copied)
  struct Small {
    std::vector<status_t> status;
    std::vector<int> ref, zeroed;
    std::vector<double> ll;
  };
  std::vector<Small> small(b->groups.size());
  for (size_t gi = 0; gi < b->groups.size(); ++gi) {
    Group& g = *b->groups[gi];
    Small& s = small[gi];
    s.status.resize(g.nseg);
    s.ref.resize(g.nseg);
    s.zeroed.resize(g.nseg);
    s.ll.resize(g.nseg);
    CU_TRY(c, cudaMemcpyAsync(s.status.data(), g.status, sizeof(status_t) * g.nseg, cudaMemcpyDefault, st));
    CU_TRY(c, cudaMemcpyAsync(s.ref.data(), g.ref, sizeof(int) * g.nseg, cudaMemcpyDefault, st));
    CU_TRY(c, cudaMemcpyAsync(s.zeroed.data(), g.zeroed, sizeof(int) * g.nseg, cudaMemcpyDefault, st));
    CU_TRY(c, cudaMemcpyAsync(s.ll.data(), g.seg_ll + (long long)I * g.nseg, sizeof(double) * g.nseg,
                              cudaMemcpyDefault, st));
  }
  CU_TRY(c, cudaStreamSynchronize(st));
  for (size_t gi = 0; gi < b->groups.size(); ++gi) {
    Group& g = *b->groups[gi];
    const Small& s = small[gi];
    for (int j = 0; j < g.nseg; ++j) {
      const int i = g.members[j];
      const gss_segment_desc& d = b->desc[i];
      gss_segment_diag& dg = diags[i];
      dg.ref_channel = s.ref[j];
      dg.zeroed_bins = s.zeroed[j];
      dg.ll_final = s.ll[j];
      if (s.status[j] != kStatusOk) {
        dg.status = (int)(s.status[j] >> 32);
        dg.error_frequency = dg.status == GSS_SINGULAR_MATRIX_ERROR ? (int64_t)(s.status[j] & 0xffffffffu) : -1;
        b->fails[i] = Fail{(gss_status)dg.status,
                           dg.status == GSS_DEGENERATE_STATS_ERROR ? "accumulate_stats: target mask is all zero"
                                                                   : "matrix has no positive eigenvalue",
                           dg.error_frequency};
        continue;
      }
      const SegDev& sd = g.segs[j];
      int64_t off = 0;
      for (int p = 0; p < d.num_parts; ++p) {
        const int64_t hi = std::min<int64_t>(b->pe[i][p], d.num_samples);  // scheduler.hpp:354-356
        const int64_t len = hi - b->pb[i][p];
        if (len > 0)
          CU_TRY(c, cudaMemcpyAsync(d.out_wave + off, g.wave + sd.wave_off + b->pb[i][p], sizeof(float) * len,
                                    cudaMemcpyDefault, st));
        d.out_lengths[p] = len;
        off += len;
      }
      if (d.mono_out)
        CU_TRY(c, cudaMemcpyAsync(d.mono_out, g.wave + sd.wave_off, sizeof(float) * d.num_samples,
                                  cudaMemcpyDefault, st));
      if (d.gamma_out && sd.g_off >= 0)
        CU_TRY(c, cudaMemcpyAsync(d.gamma_out, g.gamma + sd.g_off, sizeof(float) * (size_t)F * sd.T * sd.K,
                                  cudaMemcpyDefault, st));
      if (d.h_out)
        CU_TRY(c, cudaMemcpyAsync(d.h_out, g.h + sd.f_off * g.M, sizeof(cdbl) * (size_t)F * g.M,
                                  cudaMemcpyDefault, st));
    }
  }
  cudaEventRecord(d2h1, st);
  CU_TRY(c, cudaStreamSynchronize(st));
  // stage clocks
  for (double& v : c->stage_ms) v = 0.0;
  float ms = 0.f;
  if (cudaEventElapsedTime(&ms, d2h0, d2h1) == cudaSuccess) c->stage_ms[6] = ms;
  for (size_t gi = 0; gi < b->groups.size(); ++gi) {
    const Group& g = *b->groups[gi];
    // the STFT and the WPE alternate wave by wave: their stage clocks are sums over the waves (a wave's STFT
    // clock includes any wait for its audio); the upload that is NOT hidden is what the first wave waits for
    cudaEvent_t prev = b->events[2 + 6 * gi];
    for (int w = 0; w < g.waves_run; ++w) {
      if (cudaEventElapsedTime(&ms, prev, g.marks[2 * w]) == cudaSuccess) c->stage_ms[0] += ms;
      if (cudaEventElapsedTime(&ms, g.marks[2 * w], g.marks[2 * w + 1]) == cudaSuccess) c->stage_ms[1] += ms;
      prev = g.marks[2 * w + 1];
    }
    for (int s = 2; s < 5; ++s)
      if (cudaEventElapsedTime(&ms, b->events[2 + 6 * gi + s], b->events[2 + 6 * gi + s + 1]) == cudaSuccess)
        c->stage_ms[s] += ms;
  }
  // upload clock: from the first copy being allowed to start to the last wave being resident (most of it runs
  // under the earlier waves' kernels)
  if (!b->groups.empty() && !b->groups.back()->wave_ev.empty() &&
      cudaEventElapsedTime(&ms, b->events[1], b->groups.back()->wave_ev.back()) == cudaSuccess)
    c->stage_ms[5] = ms;
  // remember the first failure for gss_b200_last_error
  for (int i = 0; i < b->n; ++i)
    if (b->fails[i].code != GSS_OK) {
      c->err = std::string(status_name(b->fails[i].code)) + ": " + b->fails[i].msg + " (segment " +
               std::to_string(i) + ")";
      c->err_freq = b->fails[i].freq;
      break;
    }
  return GSS_OK;
}

void gss_b200_batch_free(gss_b200_ctx* c, gss_b200_batch* b) {
  if (c) cudaSetDevice(c->device);
  free_batch(c, b);
}

gss_status gss_b200_enhance_batch(gss_b200_ctx* c, int32_t n, const gss_segment_desc* segs,
                                  const gss_pipeline_config* cfg, gss_segment_diag* diags) {
  gss_b200_batch* b = nullptr;
  NvtxRange nv(c, "gss.enhance_batch");
  // the audio goes up wave by wave from inside the run, each wave behind the previous wave's launches
  static const bool trace = std::getenv("GSS_B200_TRACE") != nullptr;
  const auto t0 = std::chrono::steady_clock::now();
  gss_status rc = upload_impl(c, n, segs, cfg, /*copy_now=*/false, &b);
  if (rc != GSS_OK) return rc;
  const auto t1 = std::chrono::steady_clock::now();
  rc = run_impl(c, b);
  const auto t2 = std::chrono::steady_clock::now();
  if (rc == GSS_OK) rc = gss_b200_batch_fetch(c, b, diags);
  cudaStreamSynchronize(c->stream);
  const auto t3 = std::chrono::steady_clock::now();
  gss_b200_batch_free(c, b);
  if (trace) {
    const auto t4 = std::chrono::steady_clock::now();
    auto ms = [](auto a, auto b) { return std::chrono::duration<double, std::milli>(b - a).count(); };
    std::fprintf(stderr, "[gss_b200] enhance_batch host ms: prepare %.3f, enqueue %.3f, wait+fetch %.3f, free %.3f\n",
                 ms(t0, t1), ms(t1, t2), ms(t2, t3), ms(t3, t4));
  }
  return rc;
}

}  // extern "C"

// ===========================================================================
// stage entry points: one tensor per call, through the same kernels
// ===========================================================================
namespace {

struct StageGroup {
  gss_b200_ctx* c;
  Group g;
  explicit StageGroup(gss_b200_ctx* ctx) : c(ctx) {}
  ~StageGroup() {
    cudaStreamSynchronize(c->stream);
    g.mem.release();
  }
};

gss_status check_tensor(gss_b200_ctx* c, int bins, int64_t frames, int channels) {
  if (!c) return fail(nullptr, GSS_INTERNAL_ERROR, "null context");
  if (bins < 1 || frames < 1 || channels < 1) return fail(c, GSS_SHAPE_ERROR, "empty tensor");
  if (channels > kMaxChannels) return fail(c, GSS_UNSUPPORTED, "more than 8 channels");
  if (frames > 0x7fffffffLL / std::max(1, channels)) return fail(c, GSS_UNSUPPORTED, "too many frames");
  return GSS_OK;
}

gss_status device_status(gss_b200_ctx* c, Group& g) {
  status_t s = kStatusOk;
  CU_TRY(c, cudaMemcpyAsync(&s, g.status, sizeof(s), cudaMemcpyDefault, c->stream));
  CU_TRY(c, cudaStreamSynchronize(c->stream));
  if (s == kStatusOk) return GSS_OK;
  const int code = (int)(s >> 32);
  if (code == GSS_SINGULAR_MATRIX_ERROR)
    return fail(c, GSS_SINGULAR_MATRIX_ERROR, "matrix has no positive eigenvalue", (long long)(s & 0xffffffffu));
  if (code == GSS_DEGENERATE_STATS_ERROR)
    return fail(c, GSS_DEGENERATE_STATS_ERROR, "accumulate_stats: target mask is all zero");
  return fail(c, (gss_status)code, "device-side failure");
}

}  // namespace

extern "C" {

gss_status gss_b200_stft(gss_b200_ctx* c, const float* audio, int32_t M, int64_t N, int32_t signal_rate,
                         const gss_stft_config* cfg, float* out) {
  if (!c) return fail(nullptr, GSS_INTERNAL_ERROR, "null context");
  CU_TRY(c, cudaSetDevice(c->device));
  std::string why;
  if (!validate_stft(*cfg, why)) return fail(c, GSS_CONFIG_ERROR, why);
  if (M < 1) return fail(c, GSS_SHAPE_ERROR, "stft.analyze: no channels");
  if (N < cfg->fft_size) return fail(c, GSS_INPUT_TOO_SHORT_ERROR, "stft.analyze: fewer samples than fft_size");
  if (signal_rate > 0 && signal_rate != cfg->sample_rate)
    return fail(c, GSS_CONFIG_ERROR, "stft.analyze: signal/config sample rate mismatch");
  if (!kernel_fft_supported(*cfg, why)) return fail(c, GSS_UNSUPPORTED, why);
  if (M > kMaxChannels || N > 0x7fffffffLL) return fail(c, GSS_UNSUPPORTED, "more than 8 channels");
  Tables tb;
  gss_status rc = get_tables(c, *cfg, tb);
  if (rc != GSS_OK) return rc;
  const int F = cfg->fft_size / 2 + 1;
  const int64_t T = gss_b200_frame_count(N, cfg->fft_size, cfg->shift);
  StageGroup sg(c);
  SegSpec s;
  s.N = N;
  s.T = (int)T;
  Needs need;
  need.audio = need.y = true;
  rc = build_group(c, sg.g, M, 1, F, {s}, need, nullptr, 0);
  if (rc != GSS_OK) return rc;
  CU_TRY(c, cudaMemcpyAsync(sg.g.audio, audio, sizeof(float) * (size_t)M * N, cudaMemcpyDefault, c->stream));
  StftArgs a;
  a.audio = sg.g.audio;
  a.y = sg.g.Y;
  a.segs = sg.g.d_segs;
  a.tw_d = tb.tw_d;
  a.win_d = tb.win_d;
  a.p = stft_params(*cfg);
  a.M = M;
  a.TB = 0;
  a.fft_warps = 0;
  {
    KClock k(c, kK_stft);
    CU_TRY(c, launch_stft(a, 1, (int)T, c->stream));
  }
  CU_TRY(c, cudaMemcpyAsync(out, sg.g.Y, sizeof(float2) * (size_t)F * T * M, cudaMemcpyDefault, c->stream));
  CU_TRY(c, finish_call(c));
  return GSS_OK;
}

gss_status gss_b200_istft(gss_b200_ctx* c, const float* spec, int32_t bins, int64_t T, int32_t M,
                          int64_t num_samples, const gss_stft_config* cfg, float* out) {
  gss_status rc = check_tensor(c, bins, T, M);
  if (rc != GSS_OK) return rc;
  CU_TRY(c, cudaSetDevice(c->device));
  std::string why;
  if (!validate_stft(*cfg, why)) return fail(c, GSS_CONFIG_ERROR, why);
  if (bins != cfg->fft_size / 2 + 1) return fail(c, GSS_CONFIG_ERROR, "stft.synthesize: tensor bins do not match config");
  if (!kernel_fft_supported(*cfg, why)) return fail(c, GSS_UNSUPPORTED, why);
  Tables tb;
  rc = get_tables(c, *cfg, tb);
  if (rc != GSS_OK) return rc;
  const int F = bins;
  const int64_t padded_len = (T - 1) * cfg->shift + cfg->fft_size;
  const int64_t out_len = num_samples > 0 ? num_samples : std::max<int64_t>(0, padded_len - cfg->fft_size);
  if (out_len == 0) return GSS_OK;
  if (out_len > 0x7fffffffLL) return fail(c, GSS_UNSUPPORTED, "output longer than 2^31 samples");
  StageGroup sg(c);
  SegSpec s;
  s.N = out_len;
  s.T = (int)T;
  Needs need;
  need.y = need.x = need.wave = need.mvdr = true;
  rc = build_group(c, sg.g, M, 1, F, {s}, need, nullptr, 0);
  if (rc != GSS_OK) return rc;
  Group& g = sg.g;
  CU_TRY(c, cudaMemcpyAsync(g.Y, spec, sizeof(float2) * (size_t)F * T * M, cudaMemcpyDefault, c->stream));
  std::vector<float2> sel((size_t)F * M);
  for (int ch = 0; ch < M; ++ch) {
    // channel selection through the beamformer kernel: h = e_ch
    for (int f = 0; f < F; ++f)
      for (int m = 0; m < M; ++m) sel[(size_t)f * M + m] = make_float2(m == ch ? 1.f : 0.f, 0.f);
    CU_TRY(c, cudaMemcpyAsync(g.hconj, sel.data(), sizeof(float2) * sel.size(), cudaMemcpyDefault, c->stream));
    ApplyArgs aa;
    aa.y = g.Y;
    aa.hconj = g.hconj;
    aa.x = g.X;
    aa.segs = g.d_segs;
    aa.M = M;
    aa.F = F;
    aa.frame_major = 1;
    {
      KClock k(c, kK_apply);
      CU_TRY(c, launch_apply(aa, 1, (int)T, c->stream));
    }
    IstftArgs ia;
    ia.x = g.X;
    ia.wave = g.wave;
    ia.segs = g.d_segs;
    ia.tw = tb.tw;
    ia.win = tb.win;
    ia.p = stft_params(*cfg);
    ia.HB = 0;
    {
      KClock k(c, kK_istft);
      CU_TRY(c, launch_istft(ia, 1, out_len, c->stream));
    }
    CU_TRY(c, cudaMemcpyAsync(out + (size_t)ch * out_len, g.wave, sizeof(float) * out_len, cudaMemcpyDefault,
                              c->stream));
    CU_TRY(c, finish_call(c));
  }
  return GSS_OK;
}

gss_status gss_b200_wpe(gss_b200_ctx* c, const float* in, int32_t bins, int64_t T, int32_t M,
                        const gss_wpe_config* cfg, float* out) {
  gss_status rc = check_tensor(c, bins, T, M);
  if (rc != GSS_OK) return rc;
  CU_TRY(c, cudaSetDevice(c->device));
  std::string why;
  if (!validate_wpe(*cfg, why)) return fail(c, GSS_CONFIG_ERROR, why);
  const size_t bytes = sizeof(float2) * (size_t)bins * T * M;
  if (T <= cfg->taps + cfg->delay) {  // wpe.hpp:108-112: input returned unchanged
    if (out != in) std::memmove(out, in, bytes);
    return GSS_OK;
  }
  StageGroup sg(c);
  SegSpec s;
  s.T = (int)T;
  Needs need;
  need.y = need.yd = need.wpe = true;
  rc = build_group(c, sg.g, M, 1, bins, {s}, need, cfg, 0);
  if (rc != GSS_OK) return rc;
  CU_TRY(c, cudaMemcpyAsync(sg.g.Y, in, bytes, cudaMemcpyDefault, c->stream));
  rc = run_wpe(c, sg.g, *cfg);
  if (rc != GSS_OK) return rc;
  rc = device_status(c, sg.g);
  if (rc != GSS_OK) return rc;
  CU_TRY(c, cudaMemcpyAsync(out, sg.g.Yd, bytes, cudaMemcpyDefault, c->stream));
  CU_TRY(c, finish_call(c));
  return GSS_OK;
}

// Test hook (not in the public header): weights from `in`, one Gram pass, hermitized R and P per bin as cdouble.
gss_status gss_b200_debug_wpe_gram(gss_b200_ctx* c, const float* in, int32_t bins, int64_t T, int32_t M,
                                   const gss_wpe_config* cfg, double* out_rp) {
  gss_status rc = check_tensor(c, bins, T, M);
  if (rc != GSS_OK) return rc;
  CU_TRY(c, cudaSetDevice(c->device));
  StageGroup sg(c);
  SegSpec s;
  s.T = (int)T;
  Needs need;
  need.y = need.yd = need.wpe = true;
  rc = build_group(c, sg.g, M, 1, bins, {s}, need, cfg, 0);
  if (rc != GSS_OK) return rc;
  Group& g = sg.g;
  const int km = cfg->taps * M;
  const size_t per = (size_t)km * km + (size_t)km * M;
  cdbl* d_rp = g.mem.get<cdbl>(per * bins);
  if (!d_rp) return fail(c, GSS_CUDA_ERROR, "alloc");
  CU_TRY(c, cudaMemcpyAsync(g.Y, in, sizeof(float2) * (size_t)bins * T * M, cudaMemcpyDefault, c->stream));
  WpeArgs a;
  a.yobs = g.Y;
  a.ycur = g.Y;
  a.yout = g.Yd;
  a.w = g.w;
  a.gram = g.gram;
  a.gram_raw = g.gram_raw;
  a.use_tc = g.use_tc;
  a.gram_f16 = c->wpe_gram_f16;
  a.apply_f16 = c->wpe_apply_f16;
  a.apply_tc = 0;
  a.w_next = nullptr;
  a.debug_rp = d_rp;
  a.fb_scratch = g.fb_scratch;
  a.fb_ticket = g.fb_ticket;
  a.fb_slots = 0;
  a.gconj = g.gconj;
  a.segs = g.d_segs;
  a.status = g.status;
  a.regularization = cfg->regularization;
  a.M = M;
  a.taps = cfg->taps;
  a.delay = cfg->delay;
  a.psd_context = cfg->psd_context;
  for (int step = 0; step < 3; ++step) {
    KClock k(c, kK_wpe_power + step);
    CU_TRY(c, launch_wpe_step(step, a, 1, bins, (int)T, g.max_wchunks, c->stream));
  }
  CU_TRY(c, cudaMemcpyAsync(out_rp, d_rp, sizeof(cdbl) * per * bins, cudaMemcpyDefault, c->stream));
  CU_TRY(c, cudaStreamSynchronize(c->stream));
  return GSS_OK;
}

gss_status gss_b200_unit_normalize(gss_b200_ctx* c, const float* in, int32_t bins, int64_t T, int32_t M,
                                   float* out) {
  gss_status rc = check_tensor(c, bins, T, M);
  if (rc != GSS_OK) return rc;
  CU_TRY(c, cudaSetDevice(c->device));
  StageGroup sg(c);
  SegSpec s;
  s.T = (int)T;
  Needs need;
  need.y = need.yd = true;
  rc = build_group(c, sg.g, M, 1, bins, {s}, need, nullptr, 0);
  if (rc != GSS_OK) return rc;
  const size_t bytes = sizeof(float2) * (size_t)bins * T * M;
  CU_TRY(c, cudaMemcpyAsync(sg.g.Y, in, bytes, cudaMemcpyDefault, c->stream));
  {
    KClock k(c, kK_misc);
    CU_TRY(c, launch_unit_normalize(sg.g.Y, sg.g.Yd, (long long)bins * T, M, c->stream));
  }
  CU_TRY(c, cudaMemcpyAsync(out, sg.g.Yd, bytes, cudaMemcpyDefault, c->stream));
  CU_TRY(c, finish_call(c));
  return GSS_OK;
}

static gss_status em_common(gss_b200_ctx* c, const float* yn, int32_t bins, int64_t T, int32_t M,
                            const uint8_t* act, int64_t act_frames, int32_t K, int32_t noise, int32_t iterations,
                            const double* pi_in, const double* shapes_in, float* gamma, double* pi,
                            double* shapes, double* trace) {
  gss_status rc = check_tensor(c, bins, T, M);
  if (rc != GSS_OK) return rc;
  CU_TRY(c, cudaSetDevice(c->device));
  const bool from_state = pi_in != nullptr;
  if (!from_state && iterations < 1) return fail(c, GSS_CONFIG_ERROR, "cacgmm: iterations must be >= 1");
  if (act_frames != T) return fail(c, GSS_SHAPE_ERROR, "cacgmm: activity frames do not match tensor");
  if (K < 1) return fail(c, GSS_SHAPE_ERROR, "cacgmm: no classes");
  if (K > kMaxClasses) return fail(c, GSS_UNSUPPORTED, "more than 8 classes");
  StageGroup sg(c);
  SegSpec s;
  s.T = (int)T;
  s.K = K;
  s.noise = noise;
  s.activity = act;
  s.keep_gamma = gamma != nullptr;
  Needs need;
  need.y = need.em = need.gamma = true;
  rc = build_group(c, sg.g, M, K, bins, {s}, need, nullptr, from_state ? 0 : iterations);
  if (rc != GSS_OK) return rc;
  Group& g = sg.g;
  const int KT = g.KT, MM = M * M;
  CU_TRY(c, cudaMemcpyAsync(g.Y, yn, sizeof(float2) * (size_t)bins * T * M, cudaMemcpyDefault, c->stream));
  std::vector<double> h_pi;
  std::vector<cdbl> h_b;
  if (from_state) {
    h_pi.assign((size_t)bins * KT, 0.0);
    h_b.assign((size_t)bins * KT * MM, cd_make(0.0, 0.0));
    for (int f = 0; f < bins; ++f)
      for (int k = 0; k < K; ++k) {
        h_pi[(size_t)f * KT + k] = pi_in[(size_t)f * K + k];
        for (int i = 0; i < MM; ++i)
          h_b[((size_t)f * KT + k) * MM + i] = cd_make(shapes_in[2 * (((size_t)f * K + k) * MM + i)],
                                                        shapes_in[2 * (((size_t)f * K + k) * MM + i) + 1]);
      }
    CU_TRY(c, cudaMemcpyAsync(g.pi, h_pi.data(), sizeof(double) * h_pi.size(), cudaMemcpyDefault, c->stream));
    CU_TRY(c, cudaMemcpyAsync(g.bstate, h_b.data(), sizeof(cdbl) * h_b.size(), cudaMemcpyDefault, c->stream));
  }
  EmRun r{g.Y, 0, false, from_state, true};
  rc = run_em(c, g, r);
  if (rc != GSS_OK) return rc;
  rc = device_status(c, g);
  if (rc != GSS_OK) return rc;
  const int I = g.iterations;
  if (gamma)
    CU_TRY(c, cudaMemcpyAsync(gamma, g.gamma, sizeof(float) * (size_t)bins * T * K, cudaMemcpyDefault, c->stream));
  if (trace) CU_TRY(c, cudaMemcpyAsync(trace, g.seg_ll, sizeof(double) * (I + 1), cudaMemcpyDefault, c->stream));
  if (pi || shapes) {
    h_pi.resize((size_t)bins * KT);
    h_b.resize((size_t)bins * KT * MM);
    CU_TRY(c, cudaMemcpyAsync(h_pi.data(), g.pi, sizeof(double) * h_pi.size(), cudaMemcpyDefault, c->stream));
    CU_TRY(c, cudaMemcpyAsync(h_b.data(), g.bstate, sizeof(cdbl) * h_b.size(), cudaMemcpyDefault, c->stream));
  }
  CU_TRY(c, cudaStreamSynchronize(c->stream));
  if (pi || shapes)
    for (int f = 0; f < bins; ++f)
      for (int k = 0; k < K; ++k) {  // drop the class padding of the kernel tier
        if (pi) pi[(size_t)f * K + k] = h_pi[(size_t)f * KT + k];
        if (shapes)
          std::memcpy(shapes + 2 * (((size_t)f * K + k) * MM), &h_b[((size_t)f * KT + k) * MM], sizeof(cdbl) * MM);
      }
  return GSS_OK;
}

gss_status gss_b200_em_fit(gss_b200_ctx* c, const float* yn, int32_t bins, int64_t T, int32_t M,
                           const uint8_t* act, int64_t act_frames, int32_t K, int32_t noise, int32_t iterations,
                           float* gamma, double* pi, double* shapes, double* trace) {
  return em_common(c, yn, bins, T, M, act, act_frames, K, noise, iterations, nullptr, nullptr, gamma, pi, shapes,
                   trace);
}

gss_status gss_b200_log_likelihood(gss_b200_ctx* c, const float* yn, int32_t bins, int64_t T, int32_t M,
                                   const uint8_t* act, int32_t K, int32_t noise, const double* pi,
                                   const double* shapes, double* out) {
  if (!pi || !shapes) return fail(c, GSS_SHAPE_ERROR, "log_likelihood: inconsistent shapes");
  return em_common(c, yn, bins, T, M, act, T, K, noise, 0, pi, shapes, nullptr, nullptr, nullptr, out);
}

gss_status gss_b200_mvdr_stats(gss_b200_ctx* c, const float* y, const float* gamma, int32_t bins, int64_t T,
                               int32_t M, int32_t K, int32_t target, double* tgt, double* bg) {
  gss_status rc = check_tensor(c, bins, T, M);
  if (rc != GSS_OK) return rc;
  CU_TRY(c, cudaSetDevice(c->device));
  if (K < 1 || K > kMaxClasses) return fail(c, K < 1 ? GSS_SHAPE_ERROR : GSS_UNSUPPORTED, "class count out of range");
  if (target < 0 || target >= K) return fail(c, GSS_SHAPE_ERROR, "accumulate_stats: target class out of range");
  StageGroup sg(c);
  SegSpec s;
  s.T = (int)T;
  s.K = K;
  s.target = target;
  s.keep_gamma = true;
  Needs need;
  need.y = need.gamma = need.mvdr = true;
  rc = build_group(c, sg.g, M, K, bins, {s}, need, nullptr, 0);
  if (rc != GSS_OK) return rc;
  Group& g = sg.g;
  CU_TRY(c, cudaMemcpyAsync(g.Y, y, sizeof(float2) * (size_t)bins * T * M, cudaMemcpyDefault, c->stream));
  CU_TRY(c, cudaMemcpyAsync(g.gamma, gamma, sizeof(float) * (size_t)bins * T * K, cudaMemcpyDefault, c->stream));
  StatsPassArgs sp;
  sp.y = g.Y;
  sp.gamma = g.gamma;
  sp.segs = g.d_segs;
  sp.work = g.d_work;
  sp.part = g.part;
  sp.cell_stride = g.cell_stride;
  {
    KClock k(c, kK_mvdr);
    CU_TRY(c, launch_mvdr_stats(EmShape{g.M, g.KT}, sp, g.nwork, bins, c->stream));
  }
  StatsFinalArgs sf;
  sf.segs = g.d_segs;
  sf.part = g.part;
  sf.phi_t = g.phi_t;
  sf.phi_b = g.phi_b;
  sf.tmass = g.tmass;
  sf.cell_stride = g.cell_stride;
  sf.F = bins;
  {
    KClock k(c, kK_mvdr);
    CU_TRY(c, launch_mvdr_stats_final(EmShape{g.M, g.KT}, sf, 1, c->stream));
  }
  std::vector<double> tm(bins);
  CU_TRY(c, cudaMemcpyAsync(tm.data(), g.tmass, sizeof(double) * bins, cudaMemcpyDefault, c->stream));
  CU_TRY(c, cudaMemcpyAsync(tgt, g.phi_t, sizeof(cdbl) * (size_t)bins * M * M, cudaMemcpyDefault, c->stream));
  CU_TRY(c, cudaMemcpyAsync(bg, g.phi_b, sizeof(cdbl) * (size_t)bins * M * M, cudaMemcpyDefault, c->stream));
  CU_TRY(c, cudaStreamSynchronize(c->stream));
  double total = 0.0;
  for (double v : tm) total += v;
  if (total <= 0.0) return fail(c, GSS_DEGENERATE_STATS_ERROR, "accumulate_stats: target mask is all zero");
  return GSS_OK;
}

static gss_status mvdr_common(gss_b200_ctx* c, const double* tgt, const double* bg, int32_t bins, int32_t M,
                              int fixed_ref, int32_t* ref_out, double* h, int64_t* zeroed) {
  gss_status rc = check_tensor(c, bins, 1, M);
  if (rc != GSS_OK) return rc;
  CU_TRY(c, cudaSetDevice(c->device));
  StageGroup sg(c);
  SegSpec s;
  s.T = 1;
  Needs need;
  need.mvdr = true;
  rc = build_group(c, sg.g, M, 1, bins, {s}, need, nullptr, 0);
  if (rc != GSS_OK) return rc;
  Group& g = sg.g;
  const size_t mb = sizeof(cdbl) * (size_t)bins * M * M;
  CU_TRY(c, cudaMemcpyAsync(g.phi_t, tgt, mb, cudaMemcpyDefault, c->stream));
  CU_TRY(c, cudaMemcpyAsync(g.phi_b, bg, mb, cudaMemcpyDefault, c->stream));
  if (h) {
    rc = run_mvdr_design(c, g, fixed_ref, false);
    if (rc != GSS_OK) return rc;
    rc = device_status(c, g);
    if (rc != GSS_OK) return rc;
    int z = 0;
    CU_TRY(c, cudaMemcpyAsync(h, g.h, sizeof(cdbl) * (size_t)bins * M, cudaMemcpyDefault, c->stream));
    CU_TRY(c, cudaMemcpyAsync(&z, g.zeroed, sizeof(int), cudaMemcpyDefault, c->stream));
    CU_TRY(c, cudaStreamSynchronize(c->stream));
    if (zeroed) *zeroed = z;
  } else {
    MvdrArgs a;
    a.segs = g.d_segs;
    a.phi_t = g.phi_t;
    a.phi_b = g.phi_b;
    a.tmass = nullptr;
    a.ref = g.ref;
    a.zeroed = g.zeroed;
    a.h = g.h;
    a.hconj = g.hconj;
    a.status = g.status;
    a.M = M;
    a.F = bins;
    a.fixed_ref = -1;
    {
      KClock k(c, kK_mvdr);
      CU_TRY(c, launch_select_reference(a, 1, c->stream));
    }
    int r = 0;
    CU_TRY(c, cudaMemcpyAsync(&r, g.ref, sizeof(int), cudaMemcpyDefault, c->stream));
    CU_TRY(c, cudaStreamSynchronize(c->stream));
    *ref_out = r;
  }
  return GSS_OK;
}

gss_status gss_b200_select_reference(gss_b200_ctx* c, const double* tgt, const double* bg, int32_t bins,
                                     int32_t M, int32_t* ref) {
  return mvdr_common(c, tgt, bg, bins, M, -1, ref, nullptr, nullptr);
}

gss_status gss_b200_mvdr(gss_b200_ctx* c, const double* tgt, const double* bg, int32_t bins, int32_t M,
                         int32_t ref, double* h, int64_t* zeroed) {
  if (ref < 0 || ref >= M) return fail(c, GSS_SHAPE_ERROR, "mvdr: reference channel out of range");
  return mvdr_common(c, tgt, bg, bins, M, ref, nullptr, h, zeroed);
}

gss_status gss_b200_apply(gss_b200_ctx* c, const double* h, int32_t h_bins, int32_t h_channels, const float* y,
                          int32_t bins, int64_t T, int32_t M, float* out) {
  gss_status rc = check_tensor(c, bins, T, M);
  if (rc != GSS_OK) return rc;
  CU_TRY(c, cudaSetDevice(c->device));
  if (h_channels != M || h_bins != bins) return fail(c, GSS_SHAPE_ERROR, "beamform.apply: filter does not match tensor");
  StageGroup sg(c);
  SegSpec s;
  s.T = (int)T;
  Needs need;
  need.y = need.x = need.mvdr = true;
  rc = build_group(c, sg.g, M, 1, bins, {s}, need, nullptr, 0);
  if (rc != GSS_OK) return rc;
  Group& g = sg.g;
  std::vector<float2> hc((size_t)bins * M);
  for (size_t i = 0; i < hc.size(); ++i) hc[i] = make_float2((float)h[2 * i], -(float)h[2 * i + 1]);
  CU_TRY(c, cudaMemcpyAsync(g.Y, y, sizeof(float2) * (size_t)bins * T * M, cudaMemcpyDefault, c->stream));
  CU_TRY(c, cudaMemcpyAsync(g.hconj, hc.data(), sizeof(float2) * hc.size(), cudaMemcpyDefault, c->stream));
  ApplyArgs aa;
  aa.y = g.Y;
  aa.hconj = g.hconj;
  aa.x = g.X;
  aa.segs = g.d_segs;
  aa.M = M;
  aa.F = bins;
  aa.frame_major = 0;
  {
    KClock k(c, kK_apply);
    CU_TRY(c, launch_apply(aa, 1, (int)T, c->stream));
  }
  CU_TRY(c, cudaMemcpyAsync(out, g.X, sizeof(float2) * (size_t)bins * T, cudaMemcpyDefault, c->stream));
  CU_TRY(c, finish_call(c));
  return GSS_OK;
}


// ---- device-pointer variants: the same operators for callers whose tensors already live in HBM.
// Tensor arguments are DEVICE pointers on the context's device; `stream` is the caller's CUDA stream (0 = the
// legacy default stream): the call is ordered after the work already queued on it, and the stream waits for the
// call's results, so the caller never synchronises with the host. Copies are device-to-device.
gss_status gss_b200_stft_dev(gss_b200_ctx* c, const float* audio, int32_t M, int64_t N, int32_t signal_rate,
                             const gss_stft_config* cfg, float* out, void* stream) {
  DevCall scope(c, stream);
  return gss_b200_stft(c, audio, M, N, signal_rate, cfg, out);
}

gss_status gss_b200_istft_dev(gss_b200_ctx* c, const float* spec, int32_t bins, int64_t T, int32_t M,
                              int64_t num_samples, const gss_stft_config* cfg, float* out, void* stream) {
  DevCall scope(c, stream);
  return gss_b200_istft(c, spec, bins, T, M, num_samples, cfg, out);
}

gss_status gss_b200_wpe_dev(gss_b200_ctx* c, const float* in, int32_t bins, int64_t T, int32_t M,
                            const gss_wpe_config* cfg, float* out, void* stream) {
  DevCall scope(c, stream);
  return gss_b200_wpe(c, in, bins, T, M, cfg, out);  // reads the device status word: one host wait, as a solve can fail
}

gss_status gss_b200_unit_normalize_dev(gss_b200_ctx* c, const float* in, int32_t bins, int64_t T, int32_t M,
                                       float* out, void* stream) {
  DevCall scope(c, stream);
  return gss_b200_unit_normalize(c, in, bins, T, M, out);
}

gss_status gss_b200_apply_dev(gss_b200_ctx* c, const double* h, int32_t h_bins, int32_t h_channels, const float* y,
                              int32_t bins, int64_t T, int32_t M, float* out, void* stream) {
  DevCall scope(c, stream);
  return gss_b200_apply(c, h, h_bins, h_channels, y, bins, T, M, out);  // h (F x M cdouble) stays a HOST array
}

gss_status gss_b200_enhance_batch_dev(gss_b200_ctx* c, int32_t n, const gss_segment_desc* segs,
                                      const gss_pipeline_config* cfg, gss_segment_diag* diags, void* stream) {
  DevCall scope(c, stream);
  return gss_b200_enhance_batch(c, n, segs, cfg, diags);
}

int64_t gss_b200_nvtx_range_count(const gss_b200_ctx* c) { return c ? c->nvtx_ranges : 0; }

}  // extern "C"
