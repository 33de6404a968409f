// gss/wpe.hpp (B200 build) -- wpe.hpp:15-140 of the reference: WpeConfig, dereverberate, unit_normalize.
#pragma once

#include "stft.hpp"

namespace gss::wpe {

struct WpeConfig {  // wpe.hpp:15-30
  int taps = 10;
  int delay = 2;
  int iterations = 3;
  int psd_context = 0;
  double regularization = 1e-10;
  void validate() const {
    if (taps < 1 || delay < 1 || iterations < 1) throw ConfigError("wpe: taps, delay and iterations must be >= 1");
    if (psd_context < 0 || regularization < 0.0) throw ConfigError("wpe: psd_context and regularization must be >= 0");
  }
  gss_wpe_config c() const { return gss_wpe_config{taps, delay, iterations, psd_context, regularization}; }
};

inline stft::SpectrogramTensor dereverberate(const stft::SpectrogramTensor& y, const WpeConfig& cfg,
                                             b200::Device& dev = b200::Device::current()) {  // wpe.hpp:105-120
  cfg.validate();
  stft::SpectrogramTensor out = y;
  const gss_wpe_config c = cfg.c();
  dev.check(gss_b200_wpe(dev.get(), reinterpret_cast<const float*>(y.data.data()), y.num_bins, y.num_frames,
                         y.num_channels, &c, reinterpret_cast<float*>(out.data.data())));
  return out;
}

inline stft::SpectrogramTensor unit_normalize(const stft::SpectrogramTensor& y,
                                              b200::Device& dev = b200::Device::current()) {  // wpe.hpp:124-140
  stft::SpectrogramTensor out = y;
  dev.check(gss_b200_unit_normalize(dev.get(), reinterpret_cast<const float*>(y.data.data()), y.num_bins,
                                    y.num_frames, y.num_channels, reinterpret_cast<float*>(out.data.data())));
  return out;
}

}  // namespace gss::wpe
