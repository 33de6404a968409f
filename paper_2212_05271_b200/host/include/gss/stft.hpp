// gss/stft.hpp (B200 build) -- stft.hpp:16-229 of the reference: StftConfig, RealSignal, SpectrogramTensor,
// frame_count, frame_center, analyze, synthesize. Transforms run in libgss_b200.so (stft_kernels.cu).
#pragma once

#include <algorithm>
#include <vector>

#include "common.hpp"

namespace gss::stft {

enum class Window { kHann = 0, kSqrtHann = 1 };

struct StftConfig {  // stft.hpp:16-36
  int fft_size = 1024;
  int shift = 256;
  Window window = Window::kHann;
  int sample_rate = 16000;
  int num_bins() const { return fft_size / 2 + 1; }
  void validate() const {
    if (fft_size <= 0 || shift <= 0) throw ConfigError("stft: fft_size and shift must be positive");
    if (fft_size % shift != 0) throw ConfigError("stft: shift must divide fft_size for overlap-add");
    if (sample_rate <= 0) throw ConfigError("stft: sample_rate must be positive");
  }
  gss_stft_config c() const { return gss_stft_config{fft_size, shift, static_cast<int>(window), sample_rate}; }
};

struct RealSignal {  // stft.hpp:39-47
  std::vector<std::vector<float>> channels;
  int sample_rate = 0;
  int num_channels() const { return static_cast<int>(channels.size()); }
  int64_t num_samples() const { return channels.empty() ? 0 : static_cast<int64_t>(channels[0].size()); }
};

struct SpectrogramTensor {  // stft.hpp:52-80, (F,T,M) row-major
  std::vector<cfloat> data;
  StftConfig config;
  int num_bins = 0;
  int64_t num_frames = 0;
  int num_channels = 0;
  int64_t origin_samples = 0;
  int64_t num_samples = 0;
  int64_t index(int f, int64_t t, int m) const { return (static_cast<int64_t>(f) * num_frames + t) * num_channels + m; }
  cfloat& at(int f, int64_t t, int m) { return data[index(f, t, m)]; }
  const cfloat& at(int f, int64_t t, int m) const { return data[index(f, t, m)]; }
  static SpectrogramTensor zeros(const StftConfig& cfg, int64_t frames, int channels) {
    SpectrogramTensor s;
    s.config = cfg;
    s.num_bins = cfg.num_bins();
    s.num_frames = frames;
    s.num_channels = channels;
    s.origin_samples = -cfg.fft_size / 2;
    s.data.assign(static_cast<size_t>(s.num_bins) * frames * channels, cfloat{});
    return s;
  }
};

inline int64_t frame_count(int64_t num_samples, const StftConfig& cfg) {  // stft.hpp:120-124
  return gss_b200_frame_count(num_samples, cfg.fft_size, cfg.shift);
}
inline int64_t frame_center(int64_t t, const StftConfig& cfg) { return t * cfg.shift; }  // stft.hpp:127-129

namespace detail {
/// channel-major contiguous copy of a RealSignal (what the C ABI takes)
inline std::vector<float> flatten(const RealSignal& s) {
  const int64_t n = s.num_samples();
  std::vector<float> flat(static_cast<size_t>(s.num_channels()) * n);
  for (int m = 0; m < s.num_channels(); ++m) {
    if (static_cast<int64_t>(s.channels[m].size()) != n) throw ShapeError("stft.analyze: channels differ in length");
    std::copy(s.channels[m].begin(), s.channels[m].end(), flat.begin() + static_cast<size_t>(m) * n);
  }
  return flat;
}
}  // namespace detail

inline SpectrogramTensor analyze(const RealSignal& signal, const StftConfig& cfg,
                                 b200::Device& dev = b200::Device::current()) {  // stft.hpp:131-175
  cfg.validate();
  if (signal.num_channels() < 1) throw ShapeError("stft.analyze: no channels");
  const std::vector<float> flat = detail::flatten(signal);
  const int64_t n = signal.num_samples();
  if (n < cfg.fft_size) throw InputTooShortError("stft.analyze: fewer samples than fft_size");
  SpectrogramTensor out = SpectrogramTensor::zeros(cfg, frame_count(n, cfg), signal.num_channels());
  out.num_samples = n;
  const gss_stft_config c = cfg.c();
  dev.check(gss_b200_stft(dev.get(), flat.data(), signal.num_channels(), n, signal.sample_rate, &c,
                          reinterpret_cast<float*>(out.data.data())));
  return out;
}

inline RealSignal synthesize(const SpectrogramTensor& spec, b200::Device& dev = b200::Device::current()) {
  // stft.hpp:179-229
  const StftConfig& cfg = spec.config;
  cfg.validate();
  if (spec.num_bins != cfg.num_bins()) throw ConfigError("stft.synthesize: tensor bins do not match config");
  const int64_t padded = (spec.num_frames - 1) * cfg.shift + cfg.fft_size;
  const int64_t out_len = spec.num_samples > 0 ? spec.num_samples : std::max<int64_t>(0, padded - cfg.fft_size);
  std::vector<float> flat(static_cast<size_t>(spec.num_channels) * out_len);
  const gss_stft_config c = cfg.c();
  dev.check(gss_b200_istft(dev.get(), reinterpret_cast<const float*>(spec.data.data()), spec.num_bins,
                           spec.num_frames, spec.num_channels, spec.num_samples, &c, flat.data()));
  RealSignal out;
  out.sample_rate = cfg.sample_rate;
  out.channels.resize(spec.num_channels);
  for (int m = 0; m < spec.num_channels; ++m)
    out.channels[m].assign(flat.begin() + static_cast<size_t>(m) * out_len,
                           flat.begin() + static_cast<size_t>(m + 1) * out_len);
  return out;
}

}  // namespace gss::stft
