// oracle_capi.cpp -- flat C entry points over gss_oracle.hpp so tests and the
// cpu_baseline leg of bench.py can drive the CPU ORACLE through ctypes.
// TEST INFRASTRUCTURE ONLY; nothing in the product links against this.
// Matrices cross this boundary row-major (numpy default).
#include "gss_oracle.hpp"

#include <cstring>
#include <sstream>

using namespace gss_oracle;

namespace {
thread_local std::string g_err;
thread_local long g_err_freq = -1;

template <typename Fn>
int guarded(Fn&& fn) {
  try {
    fn();
    return kOk;
  } catch (const OracleError& e) {
    g_err = e.what();
    g_err_freq = e.frequency;
    return e.code;
  } catch (const std::exception& e) {
    g_err = e.what();
    g_err_freq = -1;
    return 100;
  }
}

CMat from_rowmajor(const cd* a, int r, int c) {
  CMat m(r, c);
  for (int i = 0; i < r; ++i)
    for (int j = 0; j < c; ++j) m(i, j) = a[i * c + j];
  return m;
}
void to_rowmajor(const CMat& m, cd* out) {
  for (int i = 0; i < m.r; ++i)
    for (int j = 0; j < m.c; ++j) out[i * m.c + j] = m(i, j);
}

Spec wrap_spec(const cf* data, int F, int64_t T, int M, const StftConfig* cfg, int64_t num_samples) {
  Spec s;
  if (cfg) s.config = *cfg;
  s.num_bins = F;
  s.num_frames = T;
  s.num_channels = M;
  s.num_samples = num_samples;
  s.origin_samples = cfg ? -cfg->fft_size / 2 : 0;
  s.data.assign(data, data + static_cast<size_t>(F) * T * M);
  return s;
}

Activity wrap_activity(const uint8_t* grid, int64_t T, int K, int target, int noise) {
  Activity a;
  a.frames = T;
  a.classes.resize(K);
  for (int k = 0; k < K; ++k) a.classes[k] = "c" + std::to_string(k);
  a.target_index = target;
  a.noise_index = noise;
  a.grid.assign(grid, grid + T * K);
  return a;
}
}  // namespace

extern "C" {

const char* oracle_last_error() { return g_err.c_str(); }
long oracle_last_error_frequency() { return g_err_freq; }
void oracle_set_threads(int n) { thread_override() = n; }
int oracle_hardware_threads() { return hardware_threads(); }

int oracle_hermitize(int n, int cols, const cd* a, cd* out) {
  return guarded([&] { to_rowmajor(hermitize(from_rowmajor(a, n, cols)), out); });
}
int oracle_regularize(int n, const cd* a, double eps, cd* out) {
  return guarded([&] { to_rowmajor(regularize(from_rowmajor(a, n, n), eps), out); });
}
int oracle_hermitian_solve(int n, int nrhs, const cd* a, const cd* b, long freq, cd* x) {
  return guarded(
      [&] { to_rowmajor(hermitian_solve(from_rowmajor(a, n, n), from_rowmajor(b, n, nrhs), freq), x); });
}
int oracle_hermitian_inverse_logdet(int n, const cd* a, cd* inv, double* logdet) {
  return guarded([&] {
    InverseLogDet r = hermitian_inverse_logdet(from_rowmajor(a, n, n));
    to_rowmajor(r.inverse, inv);
    *logdet = r.log_det;
  });
}
int oracle_hermitian_eig(int n, const cd* a, cd* vecs, double* vals) {
  return guarded([&] {
    CMat v;
    std::vector<double> w;
    if (!hermitian_eig(from_rowmajor(a, n, n), v, w))
      throw OracleError(kSingularMatrixError, "eig failed");
    to_rowmajor(v, vecs);
    std::copy(w.begin(), w.end(), vals);
  });
}
int oracle_weighted_gram(const cf* a, int64_t rows, int cols, const float* w, int64_t chunk, cd* out) {
  return guarded([&] { to_rowmajor(weighted_gram(a, rows, cols, w, chunk), out); });
}

int oracle_make_window(int fft_size, int window, double* out) {
  return guarded([&] {
    StftConfig c;
    c.fft_size = fft_size;
    c.window = window;
    auto w = make_window(c);
    std::copy(w.begin(), w.end(), out);
  });
}
int64_t oracle_frame_count(int64_t n, int fft_size, int shift) {
  StftConfig c;
  c.fft_size = fft_size;
  c.shift = shift;
  return frame_count(n, c);
}

// audio: M x N row-major. out: (F,T,M) cfloat with T = frame_count(N)
int oracle_stft(const float* audio, int M, int64_t N, int signal_rate, const StftConfig* cfg, cf* out) {
  return guarded([&] {
    Signal s;
    s.sample_rate = signal_rate;
    s.channels.resize(M);
    for (int m = 0; m < M; ++m) s.channels[m].assign(audio + m * N, audio + (m + 1) * N);
    Spec sp = analyze(s, *cfg);
    std::copy(sp.data.begin(), sp.data.end(), out);
  });
}
// spec: (F,T,M); out: M x out_len, out_len = num_samples>0 ? num_samples : (T-1)*shift
int oracle_istft(const cf* spec, int F, int64_t T, int M, int64_t num_samples, const StftConfig* cfg,
                 float* out) {
  return guarded([&] {
    Spec sp = wrap_spec(spec, F, T, M, cfg, num_samples);
    Signal s = synthesize(sp);
    for (int m = 0; m < M; ++m)
      std::copy(s.channels[m].begin(), s.channels[m].end(), out + m * s.num_samples());
  });
}
int oracle_wpe(const cf* in, int F, int64_t T, int M, const WpeConfig* cfg, cf* out) {
  return guarded([&] {
    Spec sp = wrap_spec(in, F, T, M, nullptr, 0);
    Spec o = dereverberate(sp, *cfg);
    std::copy(o.data.begin(), o.data.end(), out);
  });
}
int oracle_unit_normalize(const cf* in, int F, int64_t T, int M, cf* out) {
  return guarded([&] {
    Spec o = unit_normalize(wrap_spec(in, F, T, M, nullptr, 0));
    std::copy(o.data.begin(), o.data.end(), out);
  });
}

int oracle_cacg_log_pdf(int m, const cd* y, const cd* b, double* out) {
  return guarded([&] {
    std::vector<cd> yv(y, y + m);
    *out = cacg_log_pdf(yv, from_rowmajor(b, m, m));
  });
}
int oracle_time_varying_weights(int k, const double* pi, const uint8_t* act, int noise, double* out) {
  return guarded([&] {
    auto w = time_varying_weights(std::vector<double>(pi, pi + k), std::vector<uint8_t>(act, act + k), noise);
    std::copy(w.begin(), w.end(), out);
  });
}

// gamma (F,T,K) float; pi (F,K) double; shapes (F,K,M,M) cdouble row-major; trace iters+1
int oracle_em_fit(const cf* yn, int F, int64_t T, int M, const uint8_t* act, int64_t act_frames, int K,
                  int target, int noise, int iterations, int precise_quad, float* gamma, double* pi,
                  cd* shapes, double* trace) {
  return guarded([&] {
    Spec sp = wrap_spec(yn, F, T, M, nullptr, 0);
    Activity a = wrap_activity(act, act_frames, K, target, noise);
    EmResult r = em_fit(sp, a, iterations, precise_quad != 0);
    if (gamma) std::copy(r.gamma.begin(), r.gamma.end(), gamma);
    if (pi) std::copy(r.state.weights.begin(), r.state.weights.end(), pi);
    if (shapes)
      for (size_t i = 0; i < r.state.shapes.size(); ++i) to_rowmajor(r.state.shapes[i], shapes + i * M * M);
    if (trace) std::copy(r.likelihood_trace.begin(), r.likelihood_trace.end(), trace);
  });
}
int oracle_log_likelihood(const cf* yn, int F, int64_t T, int M, const uint8_t* act, int K, int noise,
                          const double* pi, const cd* shapes, double* out) {
  return guarded([&] {
    Spec sp = wrap_spec(yn, F, T, M, nullptr, 0);
    Activity a = wrap_activity(act, T, K, 0, noise);
    CacgmmState st = CacgmmState::uniform(F, K, M);
    std::copy(pi, pi + F * K, st.weights.begin());
    for (int i = 0; i < F * K; ++i) st.shapes[i] = from_rowmajor(shapes + (size_t)i * M * M, M, M);
    *out = log_likelihood(sp, st, a);
  });
}

int oracle_mvdr_stats(const cf* y, const float* gamma, int F, int64_t T, int M, int K, int target,
                      cd* tgt, cd* bg) {
  return guarded([&] {
    Spec sp = wrap_spec(y, F, T, M, nullptr, 0);
    std::vector<float> g(gamma, gamma + (size_t)F * T * K);
    BeamformerStats st = accumulate_stats(sp, g, K, target);
    for (int f = 0; f < F; ++f) {
      to_rowmajor(st.target[f], tgt + (size_t)f * M * M);
      to_rowmajor(st.background[f], bg + (size_t)f * M * M);
    }
  });
}
static BeamformerStats stats_from(const cd* tgt, const cd* bg, int F, int M) {
  BeamformerStats st;
  st.num_bins = F;
  st.num_channels = M;
  st.frame_count = 1;
  for (int f = 0; f < F; ++f) {
    st.target.push_back(from_rowmajor(tgt + (size_t)f * M * M, M, M));
    st.background.push_back(from_rowmajor(bg + (size_t)f * M * M, M, M));
  }
  return st;
}
int oracle_select_reference(const cd* tgt, const cd* bg, int F, int M, int* ref) {
  return guarded([&] { *ref = select_reference(stats_from(tgt, bg, F, M)); });
}
int oracle_mvdr(const cd* tgt, const cd* bg, int F, int M, int ref, cd* h, int64_t* zeroed) {
  return guarded([&] {
    BeamformerFilter flt = mvdr(stats_from(tgt, bg, F, M), ref);
    for (int f = 0; f < F; ++f) std::copy(flt.h[f].begin(), flt.h[f].end(), h + (size_t)f * M);
    *zeroed = flt.zeroed_bins;
  });
}
int oracle_apply(const cd* h, int hF, int hM, const cf* y, int F, int64_t T, int M, cf* out) {
  return guarded([&] {
    BeamformerFilter flt;
    flt.num_channels = hM;
    for (int f = 0; f < hF; ++f) flt.h.emplace_back(h + (size_t)f * hM, h + (size_t)(f + 1) * hM);
    Spec o = apply_filter(flt, wrap_spec(y, F, T, M, nullptr, 0));
    std::copy(o.data.begin(), o.data.end(), out);
  });
}

// speakers: n_seg C strings. classes_out receives '\n'-joined class labels.
int oracle_build_activity_at(int n_seg, const char* const* speakers, const double* starts,
                             const double* durations, const int64_t* centers, int64_t n_centers,
                             int sample_rate, const char* target, int noise_class, uint8_t* grid,
                             int64_t grid_capacity, int* num_classes, int* target_index, int* noise_index,
                             char* classes_out, int classes_capacity) {
  return guarded([&] {
    std::vector<Segment> segs(n_seg);
    for (int i = 0; i < n_seg; ++i) {
      segs[i].speaker = speakers[i];
      segs[i].start = starts[i];
      segs[i].duration = durations[i];
    }
    Activity a = build_activity_at(segs, std::vector<int64_t>(centers, centers + n_centers), sample_rate,
                                   target, noise_class != 0);
    *num_classes = a.num_classes();
    *target_index = a.target_index;
    *noise_index = a.noise_index;
    if ((int64_t)a.grid.size() > grid_capacity) throw OracleError(kShapeError, "grid buffer too small");
    std::copy(a.grid.begin(), a.grid.end(), grid);
    std::string joined;
    for (size_t i = 0; i < a.classes.size(); ++i) joined += (i ? "\n" : "") + a.classes[i];
    if ((int)joined.size() + 1 > classes_capacity) throw OracleError(kShapeError, "label buffer too small");
    std::memcpy(classes_out, joined.c_str(), joined.size() + 1);
  });
}

// spans_out: up to n_parts+2 pairs; returns counts through pointers
int oracle_assemble_indices(int n_parts, const double* starts, const double* durations, int sr,
                            int64_t rec_samples, double context, int fft_size, int shift,
                            int64_t* spans_out, int* n_spans, int64_t* part_begin, int64_t* part_end,
                            int64_t* total, int64_t* centers_out, int64_t centers_capacity,
                            int64_t* n_centers, double* ctx_left, double* ctx_right) {
  return guarded([&] {
    std::vector<std::pair<double, double>> parts;
    for (int i = 0; i < n_parts; ++i) parts.emplace_back(starts[i], durations[i]);
    StftConfig c;
    c.fft_size = fft_size;
    c.shift = shift;
    AssemblyPlan ap = assemble_indices(parts, sr, rec_samples, context, c);
    *n_spans = (int)ap.spans.size();
    for (size_t i = 0; i < ap.spans.size(); ++i) {
      spans_out[2 * i] = ap.spans[i].first;
      spans_out[2 * i + 1] = ap.spans[i].second;
    }
    for (int i = 0; i < n_parts; ++i) {
      part_begin[i] = ap.parts[i].sample_begin;
      part_end[i] = ap.parts[i].sample_end;
    }
    *total = ap.total;
    *n_centers = (int64_t)ap.frame_centers.size();
    if (*n_centers > centers_capacity) throw OracleError(kShapeError, "centers buffer too small");
    std::copy(ap.frame_centers.begin(), ap.frame_centers.end(), centers_out);
    *ctx_left = ap.context_left;
    *ctx_right = ap.context_right;
  });
}

struct oracle_enhance_cfg {
  int fft_size, shift, window, sample_rate;
  int enable_wpe, taps, delay, wpe_iterations, psd_context;
  double regularization;
  int bss_iterations;
};

// audio M x N; act T x K; parts as [begin,end) sample pairs; outputs concatenated
// into out_wave (capacity sum of part lengths); mono_out (N, nullable) full window;
// gamma_out (F,T,K nullable), h_out (F,M nullable); stage_seconds[5].
int oracle_enhance(const float* audio, int M, int64_t N, const uint8_t* act, int64_t act_frames, int K,
                   int target, int noise, int n_parts, const int64_t* part_begin, const int64_t* part_end,
                   const oracle_enhance_cfg* c, float* out_wave, int64_t* out_lengths, float* mono_out,
                   float* gamma_out, cd* h_out, double* ll_final, int64_t* zeroed, int* ref_channel,
                   int64_t* frames, double* stage_seconds) {
  return guarded([&] {
    Signal s;
    s.sample_rate = c->sample_rate;
    s.channels.resize(M);
    for (int m = 0; m < M; ++m) s.channels[m].assign(audio + m * N, audio + (m + 1) * N);
    Activity a = wrap_activity(act, act_frames, K, target, noise);
    std::vector<Part> parts(n_parts);
    for (int i = 0; i < n_parts; ++i) {
      parts[i].sample_begin = part_begin[i];
      parts[i].sample_end = part_end[i];
    }
    PipelineConfig cfg;
    cfg.stft.fft_size = c->fft_size;
    cfg.stft.shift = c->shift;
    cfg.stft.window = c->window;
    cfg.stft.sample_rate = c->sample_rate;
    cfg.enable_wpe = c->enable_wpe != 0;
    cfg.wpe.taps = c->taps;
    cfg.wpe.delay = c->delay;
    cfg.wpe.iterations = c->wpe_iterations;
    cfg.wpe.psd_context = c->psd_context;
    cfg.wpe.regularization = c->regularization;
    cfg.bss_iterations = c->bss_iterations;
    // same validation order as run_pipeline's cfg.validate() (scheduler.hpp:46-57)
    if (cfg.bss_iterations < 1) throw OracleError(kConfigError, "scheduler: bss_iterations must be >= 1");
    cfg.wpe.validate();
    cfg.stft.validate();
    const bool diag = mono_out || gamma_out || h_out;
    EnhanceOut r = enhance_batch(s, a, parts, cfg, diag);
    int64_t off = 0;
    for (int i = 0; i < n_parts; ++i) {
      std::copy(r.outputs[i].begin(), r.outputs[i].end(), out_wave + off);
      out_lengths[i] = (int64_t)r.outputs[i].size();
      off += out_lengths[i];
    }
    if (mono_out) std::copy(r.mono.begin(), r.mono.end(), mono_out);
    if (gamma_out) std::copy(r.gamma.begin(), r.gamma.end(), gamma_out);
    if (h_out) std::copy(r.h.begin(), r.h.end(), h_out);
    *ll_final = r.ll_final;
    *zeroed = r.zeroed_bins;
    *ref_channel = r.ref_channel;
    *frames = r.frames;
    if (stage_seconds) std::copy(r.stage_seconds, r.stage_seconds + 5, stage_seconds);
  });
}

}  // extern "C"
