// gss/cacgmm.hpp (B200 build) -- cacgmm.hpp:17-370 of the reference: CacgmmState, PosteriorTensor, EmResult,
// cacg_log_pdf, time_varying_weights, em_fit, log_likelihood. The EM runs in libgss_b200.so
// (cacgmm_kernels.cuh); the two scalar forms are host functions of the library (host_logic.cpp).
#pragma once

#include <algorithm>
#include <string>
#include <vector>

#include "manifests.hpp"
#include "numerics.hpp"
#include "stft.hpp"

namespace gss::cacgmm {

constexpr double kQuadraticFormFloor = 1e-10;  // cacgmm.hpp:17
constexpr double kWeightFloor = 1e-10;         // cacgmm.hpp:18

struct CacgmmState {  // cacgmm.hpp:22-49
  int num_bins = 0, num_classes = 0, num_channels = 0;
  std::vector<double> weights;             // (F,K)
  std::vector<numerics::CMatrix> shapes;   // (F,K) of MxM
  std::vector<std::string> class_list;
  double& weight(int f, int k) { return weights[f * num_classes + k]; }
  double weight(int f, int k) const { return weights[f * num_classes + k]; }
  numerics::CMatrix& shape(int f, int k) { return shapes[f * num_classes + k]; }
  const numerics::CMatrix& shape(int f, int k) const { return shapes[f * num_classes + k]; }
  static CacgmmState uniform(int bins, int classes, int channels, std::vector<std::string> labels) {
    CacgmmState s;
    s.num_bins = bins;
    s.num_classes = classes;
    s.num_channels = channels;
    s.class_list = std::move(labels);
    s.weights.assign(static_cast<size_t>(bins) * classes, 1.0 / classes);
    s.shapes.assign(static_cast<size_t>(bins) * classes, numerics::CMatrix::Identity(channels, channels));
    return s;
  }
};

struct PosteriorTensor {  // cacgmm.hpp:52-62
  int num_bins = 0;
  int64_t num_frames = 0;
  int num_classes = 0;
  std::vector<float> gamma;  // (F,T,K) row-major
  int64_t index(int f, int64_t t, int k) const { return (static_cast<int64_t>(f) * num_frames + t) * num_classes + k; }
  float at(int f, int64_t t, int k) const { return gamma[index(f, t, k)]; }
};

struct EmResult {  // cacgmm.hpp:178-182
  CacgmmState state;
  PosteriorTensor posteriors;
  std::vector<double> likelihood_trace;
};

inline double cacg_log_pdf(const numerics::CVector& y, const numerics::CMatrix& b) {  // cacgmm.hpp:66-82
  if (b.rows() != static_cast<int>(y.size()) || b.cols() != b.rows())
    throw ShapeError("cacg_log_pdf: B does not match y");
  double out = 0.0;
  b200::check_host(gss_b200_cacg_log_pdf(static_cast<int32_t>(y.size()), reinterpret_cast<const double*>(y.data()),
                                         reinterpret_cast<const double*>(b.data()), &out));
  return out;
}

inline std::vector<double> time_varying_weights(const std::vector<double>& pi, const std::vector<uint8_t>& activity,
                                                int noise_index = -1) {  // cacgmm.hpp:87-112
  if (activity.size() != pi.size()) throw ShapeError("time_varying_weights: activity row does not match pi");
  std::vector<double> out(pi.size());
  b200::check_host(gss_b200_time_varying_weights(static_cast<int32_t>(pi.size()), pi.data(), activity.data(),
                                                 noise_index, out.data()));
  return out;
}

namespace detail {
inline std::vector<cdouble> pack_shapes(const CacgmmState& st) {
  const int m = st.num_channels;
  std::vector<cdouble> flat(st.shapes.size() * static_cast<size_t>(m) * m);
  for (size_t i = 0; i < st.shapes.size(); ++i)
    std::copy(st.shapes[i].data(), st.shapes[i].data() + m * m, flat.begin() + i * m * m);
  return flat;
}
}  // namespace detail

inline EmResult em_fit(const stft::SpectrogramTensor& y, const manifests::ActivityMatrix& activity,
                       int iterations = 20, b200::Device& dev = b200::Device::current()) {  // cacgmm.hpp:264-340
  if (iterations < 1) throw ConfigError("cacgmm: iterations must be >= 1");
  if (activity.frames != y.num_frames) throw ShapeError("cacgmm: activity frames do not match tensor");
  const int F = y.num_bins, M = y.num_channels, K = activity.num_classes();
  EmResult res;
  res.state = CacgmmState::uniform(F, K, M, activity.classes);
  res.posteriors.num_bins = F;
  res.posteriors.num_frames = y.num_frames;
  res.posteriors.num_classes = K;
  res.posteriors.gamma.assign(static_cast<size_t>(F) * y.num_frames * K, 0.0f);
  res.likelihood_trace.assign(iterations + 1, 0.0);
  std::vector<cdouble> shapes(static_cast<size_t>(F) * K * M * M);
  dev.check(gss_b200_em_fit(dev.get(), reinterpret_cast<const float*>(y.data.data()), F, y.num_frames, M,
                            activity.grid.data(), activity.frames, K, activity.noise_index, iterations,
                            res.posteriors.gamma.data(), res.state.weights.data(),
                            reinterpret_cast<double*>(shapes.data()), res.likelihood_trace.data()));
  for (size_t i = 0; i < res.state.shapes.size(); ++i)
    std::copy(shapes.begin() + i * M * M, shapes.begin() + (i + 1) * M * M, res.state.shapes[i].data());
  return res;
}

inline double log_likelihood(const stft::SpectrogramTensor& y, const CacgmmState& state,
                             const manifests::ActivityMatrix& activity,
                             b200::Device& dev = b200::Device::current()) {  // cacgmm.hpp:343-370
  if (activity.frames != y.num_frames || activity.num_classes() != state.num_classes)
    throw ShapeError("log_likelihood: inconsistent shapes");
  const std::vector<cdouble> shapes = detail::pack_shapes(state);
  double out = 0.0;
  dev.check(gss_b200_log_likelihood(dev.get(), reinterpret_cast<const float*>(y.data.data()), y.num_bins,
                                    y.num_frames, y.num_channels, activity.grid.data(), state.num_classes,
                                    activity.noise_index, state.weights.data(),
                                    reinterpret_cast<const double*>(shapes.data()), &out));
  return out;
}

}  // namespace gss::cacgmm
