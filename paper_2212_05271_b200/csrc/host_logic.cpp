// host_logic.cpp -- the integer / scalar half of the hot path that runs on the
// host in the reference too: frame geometry (stft.hpp:120-129), the activity
// guide (manifests.hpp:372-414), the index arithmetic of scheduler::assemble
// (scheduler.hpp:196-266) and the scalar known-answer forms of the cACGMM
// equations (cacgmm.hpp:66-112). Bit-exact with the reference by construction:
// same integer types, same llround / double comparisons, same ordering.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <set>
#include <string>
#include <vector>

#include "../../include/gss_b200.h"
#include "linalg.cuh"

namespace gssb {
void set_thread_error(int code, const std::string& msg, long long freq);
}

using gssb::cdbl;

extern "C" {

int64_t gss_b200_frame_count(int64_t num_samples, int32_t fft_size, int32_t shift) {
  // stft.hpp:120-124: padded = n + fft; (padded - fft) / shift + 1
  const int64_t padded = num_samples + fft_size;
  return (padded - fft_size) / shift + 1;
}

gss_status gss_b200_build_activity_at(int32_t n_segments, const char* const* speakers, const double* starts,
                                      const double* durations, const int64_t* centers, int64_t n_centers,
                                      int32_t sample_rate, const char* target, int32_t noise_class,
                                      uint8_t* grid, int64_t grid_capacity, int32_t* num_classes,
                                      int32_t* target_index, int32_t* noise_index, char* classes_out,
                                      int32_t classes_capacity) {
  std::set<std::string> uniq;
  for (int i = 0; i < n_segments; ++i) uniq.insert(speakers[i]);
  uniq.insert(target);
  std::vector<std::string> classes(uniq.begin(), uniq.end());
  const int tgt = (int)(std::find(classes.begin(), classes.end(), std::string(target)) - classes.begin());
  int noise = -1;
  if (noise_class) {
    noise = (int)classes.size();
    classes.push_back("noise");  // manifests.hpp:366
  }
  const int K = (int)classes.size();
  if ((int64_t)K * n_centers > grid_capacity) {
    gssb::set_thread_error(GSS_SHAPE_ERROR, "build_activity_at: grid buffer too small", -1);
    return GSS_SHAPE_ERROR;
  }
  std::memset(grid, 0, (size_t)K * n_centers);
  for (int i = 0; i < n_segments; ++i) {
    const int k = (int)(std::find(classes.begin(), classes.end(), std::string(speakers[i])) - classes.begin());
    const double lo = starts[i] * sample_rate;
    const double hi = (starts[i] + durations[i]) * sample_rate;  // Segment::end() = start + duration
    for (int64_t t = 0; t < n_centers; ++t) {
      const double c = (double)centers[t];
      if (c >= lo && c < hi) grid[t * K + k] = 1;
    }
  }
  if (noise >= 0)
    for (int64_t t = 0; t < n_centers; ++t) grid[t * K + noise] = 1;
  std::string joined;
  for (size_t i = 0; i < classes.size(); ++i) joined += (i ? "\n" : "") + classes[i];
  if ((int)joined.size() + 1 > classes_capacity) {
    gssb::set_thread_error(GSS_SHAPE_ERROR, "build_activity_at: label buffer too small", -1);
    return GSS_SHAPE_ERROR;
  }
  std::memcpy(classes_out, joined.c_str(), joined.size() + 1);
  *num_classes = K;
  *target_index = tgt;
  *noise_index = noise;
  bool active = false;
  for (int64_t t = 0; t < n_centers && !active; ++t) active = grid[t * K + tgt] != 0;
  if (!active) {
    gssb::set_thread_error(GSS_EMPTY_TARGET_ERROR,
                           std::string("speaker '") + target + "' has no active frame in the window", -1);
    return GSS_EMPTY_TARGET_ERROR;
  }
  return GSS_OK;
}

gss_status gss_b200_assemble_indices(int32_t n_parts, const double* starts, const double* durations,
                                     int32_t sr, int64_t rec_samples, double context_duration,
                                     int32_t fft_size, int32_t shift, int64_t* spans_out, int32_t* n_spans,
                                     int64_t* part_begin, int64_t* part_end, int64_t* total,
                                     int64_t* centers_out, int64_t centers_capacity, int64_t* n_centers,
                                     double* context_left, double* context_right) {
  if (n_parts < 1) {
    gssb::set_thread_error(GSS_SHAPE_ERROR, "assemble: no parts", -1);
    return GSS_SHAPE_ERROR;
  }
  std::vector<std::pair<int64_t, int64_t>> spans;
  const int64_t first_start = (int64_t)std::llround(starts[0] * sr);
  const int64_t ctx = (int64_t)std::llround(context_duration * sr);
  const int64_t left_begin = std::max<int64_t>(0, first_start - ctx);
  if (left_begin < first_start) spans.emplace_back(left_begin, first_start);
  *context_left = (double)(first_start - left_begin) / sr;
  std::vector<size_t> part_span;
  for (int p = 0; p < n_parts; ++p) {
    const int64_t s0 = (int64_t)std::llround(starts[p] * sr);
    const int64_t s1 = std::min<int64_t>(rec_samples, (int64_t)std::llround((starts[p] + durations[p]) * sr));
    if (s1 <= s0) {
      gssb::set_thread_error(GSS_SHAPE_ERROR, "segment maps to an empty sample range", -1);
      return GSS_SHAPE_ERROR;
    }
    part_span.push_back(spans.size());
    spans.emplace_back(s0, s1);
  }
  const int64_t last_end = spans.back().second;
  const int64_t right_end = std::min(rec_samples, last_end + ctx);
  if (right_end > last_end) spans.emplace_back(last_end, right_end);
  *context_right = (double)(right_end - last_end) / sr;
  std::vector<int64_t> offs;
  int64_t off = 0;
  for (const auto& s : spans) {
    offs.push_back(off);
    off += s.second - s.first;
  }
  *total = off;
  *n_spans = (int32_t)spans.size();
  for (size_t i = 0; i < spans.size(); ++i) {
    spans_out[2 * i] = spans[i].first;
    spans_out[2 * i + 1] = spans[i].second;
  }
  for (int p = 0; p < n_parts; ++p) {
    part_begin[p] = offs[part_span[p]];
    part_end[p] = part_begin[p] + (spans[part_span[p]].second - spans[part_span[p]].first);
  }
  const int64_t t_count = gss_b200_frame_count(off, fft_size, shift);
  *n_centers = t_count;
  if (t_count > centers_capacity) {
    gssb::set_thread_error(GSS_SHAPE_ERROR, "assemble: centers buffer too small", -1);
    return GSS_SHAPE_ERROR;
  }
  for (int64_t t = 0; t < t_count; ++t) {
    const int64_t c = std::min<int64_t>(t * shift, off - 1);  // stft::frame_center, clamped (scheduler.hpp:258)
    size_t s = 0;
    while (s + 1 < spans.size() && c >= offs[s] + (spans[s].second - spans[s].first)) ++s;
    centers_out[t] = spans[s].first + (c - offs[s]);
  }
  return GSS_OK;
}

gss_status gss_b200_cacg_log_pdf(int32_t m, const double* y, const double* b, double* out) {
  if (m < 1 || m > 64) {
    gssb::set_thread_error(GSS_SHAPE_ERROR, "cacg_log_pdf: B does not match y", -1);
    return GSS_SHAPE_ERROR;
  }
  std::vector<cdbl> a(m * m), inv(m * m), work(m * m);
  std::vector<double> wv(m);
  double log_det = 0.0;
  for (int i = 0; i < m * m; ++i) a[i] = gssb::cd_make(b[2 * i], b[2 * i + 1]);
  int st = gssb::hermitian_inverse_logdet<64>(a.data(), m, inv.data(), &log_det, work.data(), wv.data());
  if (st != gssb::kLinOk) {  // retry on regularize(B) (cacgmm.hpp:70-75)
    for (int i = 0; i < m * m; ++i) a[i] = gssb::cd_make(b[2 * i], b[2 * i + 1]);
    gssb::regularize_inplace(a.data(), m, m, gssb::kRegEps);
    st = gssb::hermitian_inverse_logdet<64>(a.data(), m, inv.data(), &log_det, work.data(), wv.data());
  }
  if (st != gssb::kLinOk) {
    gssb::set_thread_error(GSS_SINGULAR_MATRIX_ERROR, "matrix has no positive eigenvalue", -1);
    return GSS_SINGULAR_MATRIX_ERROR;
  }
  double qre = 0.0;
  for (int i = 0; i < m; ++i)
    for (int j = 0; j < m; ++j) {
      const cdbl yi = gssb::cd_make(y[2 * i], -y[2 * i + 1]);
      const cdbl yj = gssb::cd_make(y[2 * j], y[2 * j + 1]);
      qre += gssb::cd_mul(gssb::cd_mul(yi, inv[i * m + j]), yj).re;
    }
  const double quad = std::max(1e-10, qre);
  *out = -m * std::log(2.0 * M_PI) + std::lgamma((double)m) - log_det - m * std::log(quad);
  return GSS_OK;
}

gss_status gss_b200_time_varying_weights(int32_t k_count, const double* pi, const uint8_t* activity,
                                         int32_t noise_index, double* out) {
  double z = 0.0;
  for (int k = 0; k < k_count; ++k) {
    out[k] = 0.0;
    if (activity[k]) {
      out[k] = pi[k];
      z += pi[k];
    }
  }
  if (z <= 0.0) {
    if (noise_index >= 0 && noise_index < k_count) {
      for (int k = 0; k < k_count; ++k) out[k] = 0.0;
      out[noise_index] = 1.0;
    } else {
      for (int k = 0; k < k_count; ++k) out[k] = 1.0 / k_count;
    }
    return GSS_OK;
  }
  for (int k = 0; k < k_count; ++k) out[k] /= z;
  return GSS_OK;
}

}  // extern "C"
