// gss/beamform.hpp (B200 build) -- beamform.hpp:18-165 of the reference: BeamformerStats, BeamformerFilter,
// accumulate_stats, select_reference, mvdr, apply.
#pragma once

#include <vector>

#include "cacgmm.hpp"
#include "numerics.hpp"
#include "stft.hpp"

namespace gss::beamform {

struct BeamformerStats {  // beamform.hpp:18-24
  int num_bins = 0;
  int num_channels = 0;
  int64_t frame_count = 0;
  std::vector<numerics::CMatrix> target;
  std::vector<numerics::CMatrix> background;
};

struct BeamformerFilter {  // beamform.hpp:26-31
  int num_channels = 0;
  int ref_channel = 0;
  std::vector<numerics::CVector> h;
  int64_t zeroed_bins = 0;
};

namespace detail {
inline std::vector<cdouble> pack(const std::vector<numerics::CMatrix>& v, int m) {
  std::vector<cdouble> flat(v.size() * static_cast<size_t>(m) * m);
  for (size_t f = 0; f < v.size(); ++f) std::copy(v[f].data(), v[f].data() + m * m, flat.begin() + f * m * m);
  return flat;
}
}  // namespace detail

inline BeamformerStats accumulate_stats(const stft::SpectrogramTensor& y, const cacgmm::PosteriorTensor& gamma,
                                        int target, b200::Device& dev = b200::Device::current()) {
  // beamform.hpp:35-85
  if (gamma.num_bins != y.num_bins || gamma.num_frames != y.num_frames)
    throw ShapeError("accumulate_stats: posterior does not match tensor");
  if (target < 0 || target >= gamma.num_classes) throw ShapeError("accumulate_stats: target class out of range");
  const int F = y.num_bins, M = y.num_channels;
  std::vector<cdouble> tgt(static_cast<size_t>(F) * M * M), bg(tgt.size());
  dev.check(gss_b200_mvdr_stats(dev.get(), reinterpret_cast<const float*>(y.data.data()), gamma.gamma.data(), F,
                                y.num_frames, M, gamma.num_classes, target, reinterpret_cast<double*>(tgt.data()),
                                reinterpret_cast<double*>(bg.data())));
  BeamformerStats st;
  st.num_bins = F;
  st.num_channels = M;
  st.frame_count = y.num_frames;
  st.target.assign(F, numerics::CMatrix(M, M));
  st.background.assign(F, numerics::CMatrix(M, M));
  for (int f = 0; f < F; ++f) {
    std::copy(tgt.begin() + static_cast<size_t>(f) * M * M, tgt.begin() + static_cast<size_t>(f + 1) * M * M,
              st.target[f].data());
    std::copy(bg.begin() + static_cast<size_t>(f) * M * M, bg.begin() + static_cast<size_t>(f + 1) * M * M,
              st.background[f].data());
  }
  return st;
}

inline int select_reference(const BeamformerStats& st, b200::Device& dev = b200::Device::current()) {
  // beamform.hpp:89-107
  const std::vector<cdouble> tgt = detail::pack(st.target, st.num_channels), bg = detail::pack(st.background, st.num_channels);
  int32_t ref = 0;
  dev.check(gss_b200_select_reference(dev.get(), reinterpret_cast<const double*>(tgt.data()),
                                      reinterpret_cast<const double*>(bg.data()), st.num_bins, st.num_channels, &ref));
  return ref;
}

inline BeamformerFilter mvdr(const BeamformerStats& st, int ref, b200::Device& dev = b200::Device::current()) {
  // beamform.hpp:111-135
  const int M = st.num_channels;
  if (ref < 0 || ref >= M) throw ShapeError("mvdr: reference channel out of range");
  const std::vector<cdouble> tgt = detail::pack(st.target, M), bg = detail::pack(st.background, M);
  std::vector<cdouble> h(static_cast<size_t>(st.num_bins) * M);
  int64_t zeroed = 0;
  dev.check(gss_b200_mvdr(dev.get(), reinterpret_cast<const double*>(tgt.data()),
                          reinterpret_cast<const double*>(bg.data()), st.num_bins, M, ref,
                          reinterpret_cast<double*>(h.data()), &zeroed));
  BeamformerFilter flt;
  flt.num_channels = M;
  flt.ref_channel = ref;
  flt.zeroed_bins = zeroed;
  flt.h.resize(st.num_bins);
  for (int f = 0; f < st.num_bins; ++f)
    flt.h[f].assign(h.begin() + static_cast<size_t>(f) * M, h.begin() + static_cast<size_t>(f + 1) * M);
  return flt;
}

inline stft::SpectrogramTensor apply(const BeamformerFilter& flt, const stft::SpectrogramTensor& y,
                                     b200::Device& dev = b200::Device::current()) {  // beamform.hpp:138-165
  if (flt.num_channels != y.num_channels || static_cast<int>(flt.h.size()) != y.num_bins)
    throw ShapeError("beamform.apply: filter does not match tensor");
  const int M = y.num_channels;
  std::vector<cdouble> h(static_cast<size_t>(y.num_bins) * M);
  for (int f = 0; f < y.num_bins; ++f) std::copy(flt.h[f].begin(), flt.h[f].end(), h.begin() + static_cast<size_t>(f) * M);
  stft::SpectrogramTensor out = stft::SpectrogramTensor::zeros(y.config, y.num_frames, 1);
  out.num_bins = y.num_bins;
  out.data.assign(static_cast<size_t>(y.num_bins) * y.num_frames, cfloat{});
  out.origin_samples = y.origin_samples;
  out.num_samples = y.num_samples;
  dev.check(gss_b200_apply(dev.get(), reinterpret_cast<const double*>(h.data()), y.num_bins, M,
                           reinterpret_cast<const float*>(y.data.data()), y.num_bins, y.num_frames, M,
                           reinterpret_cast<float*>(out.data.data())));
  return out;
}

}  // namespace gss::beamform
