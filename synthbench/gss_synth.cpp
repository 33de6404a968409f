// gss_synth.cpp -- synthetic multi-speaker reverberant mixture generator for the
// bench / test harness (NOT part of the enhancement product path and NOT the
// oracle). Restates the input specification of the reference's
// synthbench::generate (proj/include/gss/synthbench.hpp:27-66 RNG, :178-242
// sources, :247-266 impulse responses, :269-305 FFT convolution, :319-321
// steering delays, :323-438 mixing + sensor noise) so CPU and GPU arms consume
// identical bytes. Only `steering = delays` is provided (the BASELINE configs
// use it); `random_phase` steering is not restated.
#include <algorithm>
#include <cmath>
#include <complex>
#include <cstdint>
#include <cstring>
#include <string>
#include <vector>

namespace {

struct SplitMix64 {  // synthbench.hpp:27-61
  uint64_t state;
  double spare = 0.0;
  bool have_spare = false;
  explicit SplitMix64(uint64_t seed) : state(seed) {}
  uint64_t next() {
    state += 0x9E3779B97F4A7C15ULL;
    uint64_t z = state;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
  }
  double uniform() { return static_cast<double>(next() >> 11) * 0x1.0p-53; }
  double gaussian() {
    if (have_spare) {
      have_spare = false;
      return spare;
    }
    double u1 = uniform();
    while (u1 <= 0.0) u1 = uniform();
    const double u2 = uniform();
    const double r = std::sqrt(-2.0 * std::log(u1));
    spare = r * std::sin(2.0 * M_PI * u2);
    have_spare = true;
    return r * std::cos(2.0 * M_PI * u2);
  }
};

uint64_t derive_seed(uint64_t seed, uint64_t a, uint64_t b = 0) {  // synthbench.hpp:63-66
  SplitMix64 rng(seed ^ (a * 0x9E3779B97F4A7C15ULL) ^ (b * 0xC2B2AE3D27D4EB4FULL));
  return rng.next();
}

// chirp / resonated-noise bursts in a speaker-specific band (synthbench.hpp:178-242)
void render_source(std::vector<float>& track, int64_t start, int64_t len, int sr, int spk,
                   SplitMix64& rng) {
  const double band_lo = 140.0 * (1.0 + 0.4 * spk) + 30.0 * rng.uniform();
  const double band_hi = std::min(6500.0, band_lo * 24.0);
  const double log_span = std::log(band_hi / band_lo);
  const int64_t edge = sr / 100, outer = sr / 50;
  const double target_rms = 0.16;
  std::vector<double> burst;
  int64_t i = 0;
  while (i < len) {
    const int64_t nb = std::min<int64_t>(len - i, static_cast<int64_t>((0.10 + 0.22 * rng.uniform()) * sr));
    if (nb < 2 * edge) break;
    burst.assign(nb, 0.0);
    const double f1 = band_lo * std::exp(log_span * rng.uniform());
    const double f2 = band_lo * std::exp(log_span * rng.uniform());
    if (rng.uniform() < 0.6) {
      double ph1 = 2.0 * M_PI * rng.uniform();
      double ph2 = 2.0 * M_PI * rng.uniform();
      for (int64_t j = 0; j < nb; ++j) {
        const double f = f1 * std::pow(f2 / f1, static_cast<double>(j) / nb);
        ph1 += 2.0 * M_PI * f / sr;
        ph2 += 2.0 * M_PI * 2.0 * f / sr;
        burst[j] = std::sin(ph1) + 0.35 * std::sin(ph2);
      }
    } else {
      const double r = 0.97;
      double y1 = 0.0, y2 = 0.0;
      for (int64_t j = 0; j < nb; ++j) {
        const double f = f1 * std::pow(f2 / f1, static_cast<double>(j) / nb);
        const double theta = 2.0 * M_PI * f / sr;
        const double y = rng.gaussian() + 2.0 * r * std::cos(theta) * y1 - r * r * y2;
        y2 = y1;
        y1 = y;
        burst[j] = y;
      }
    }
    double energy = 0.0;
    for (double v : burst) energy += v * v;
    const double gain =
        (0.7 + 0.6 * rng.uniform()) * target_rms / std::max(1e-12, std::sqrt(energy / nb));
    for (int64_t j = 0; j < nb; ++j) {
      double w = gain;
      if (j < edge) w *= 0.5 * (1.0 - std::cos(M_PI * j / edge));
      if (nb - 1 - j < edge) w *= 0.5 * (1.0 - std::cos(M_PI * (nb - 1 - j) / edge));
      const int64_t at = i + j;
      double fade = 1.0;
      if (at < outer) fade = static_cast<double>(at) / outer;
      if (len - 1 - at < outer) fade = std::min(fade, static_cast<double>(len - 1 - at) / outer);
      track[start + at] += static_cast<float>(burst[j] * w * fade);
    }
    i += nb + static_cast<int64_t>((0.02 + 0.08 * rng.uniform()) * sr);
  }
}

// unit direct path at `delay`, gaussian tail decaying 60 dB over t60 (synthbench.hpp:247-266)
std::vector<float> exponential_ir(int delay, double t60, int sr, double tail_energy, SplitMix64& rng) {
  const int pre = sr / 64;
  const int tail_len = static_cast<int>(t60 * sr * 1.2);
  std::vector<float> ir(delay + pre + tail_len, 0.0f);
  ir[delay] = 1.0f;
  if (t60 <= 0.0 || tail_len <= 0) return ir;
  double energy = 0.0;
  std::vector<double> tail(tail_len);
  for (int n = 0; n < tail_len; ++n) {
    tail[n] = std::exp(-6.908 * n / (t60 * sr)) * rng.gaussian();
    energy += tail[n] * tail[n];
  }
  const double scale = std::sqrt(tail_energy / std::max(energy, 1e-30));
  for (int n = 0; n < tail_len; ++n) ir[delay + pre + n] = static_cast<float>(tail[n] * scale);
  return ir;
}

void fft_inplace(std::vector<std::complex<double>>& x, bool inverse) {
  const size_t n = x.size();
  for (size_t i = 1, j = 0; i < n; ++i) {
    size_t bit = n >> 1;
    for (; j & bit; bit >>= 1) j ^= bit;
    j ^= bit;
    if (i < j) std::swap(x[i], x[j]);
  }
  for (size_t len = 2; len <= n; len <<= 1) {
    const double ang = (inverse ? 2.0 : -2.0) * M_PI / static_cast<double>(len);
    std::vector<std::complex<double>> tw(len / 2);
    for (size_t k = 0; k < len / 2; ++k) tw[k] = {std::cos(ang * k), std::sin(ang * k)};
    for (size_t b = 0; b < n; b += len)
      for (size_t k = 0; k < len / 2; ++k) {
        const auto u = x[b + k], v = x[b + k + len / 2] * tw[k];
        x[b + k] = u + v;
        x[b + k + len / 2] = u - v;
      }
  }
}

// overlap-add FFT convolution, all-zero blocks skipped (synthbench.hpp:269-305)
std::vector<float> fft_convolve(const std::vector<float>& x, const std::vector<float>& ir) {
  const int64_t n = x.size(), l = ir.size(), block = 1 << 15;
  int64_t fft_size = 1;
  while (fft_size < block + l - 1) fft_size <<= 1;
  std::vector<std::complex<double>> ir_spec(fft_size, 0.0), buf(fft_size);
  for (int64_t i = 0; i < l; ++i) ir_spec[i] = ir[i];
  fft_inplace(ir_spec, false);
  std::vector<float> out(n, 0.0f);
  for (int64_t b0 = 0; b0 < n; b0 += block) {
    const int64_t len = std::min<int64_t>(block, n - b0);
    bool all_zero = true;
    for (int64_t i = 0; i < len && all_zero; ++i) all_zero = x[b0 + i] == 0.0f;
    if (all_zero) continue;
    std::fill(buf.begin(), buf.end(), 0.0);
    for (int64_t i = 0; i < len; ++i) buf[i] = x[b0 + i];
    fft_inplace(buf, false);
    for (int64_t i = 0; i < fft_size; ++i) buf[i] *= ir_spec[i];
    fft_inplace(buf, true);
    const int64_t out_len = std::min<int64_t>(len + l - 1, n - b0);
    const double inv = 1.0 / static_cast<double>(fft_size);
    for (int64_t i = 0; i < out_len; ++i) out[b0 + i] += static_cast<float>(buf[i].real() * inv);
  }
  return out;
}

int steering_delay(int speaker, int channel) {  // synthbench.hpp:319-321
  return channel == 0 ? 0 : 1 + (channel * (3 + 2 * speaker)) % 9;
}

thread_local std::string g_err;

}  // namespace

extern "C" {

const char* gss_synth_last_error() { return g_err.c_str(); }

int gss_synth_steering_delay(int speaker, int channel) { return steering_delay(speaker, channel); }

// Speaker k owns segments seg_offsets[k] .. seg_offsets[k+1]-1 of (seg_start, seg_dur) seconds.
// mixture: channels x n (row-major); dry / images0 (nullable): n_speakers x n.
// Returns 0, or 9 (SpecError) with a message in gss_synth_last_error().
int gss_synth_generate(double duration, int sample_rate, int channels, uint64_t seed, int n_speakers,
                       const int* seg_offsets, const double* seg_start, const double* seg_dur,
                       double reverb_t60, double noise_snr, float* mixture, float* dry, float* images0) {
  // MixtureSpec::validate (synthbench.hpp:89-109)
  if (duration <= 0 || sample_rate <= 0 || channels < 1) {
    g_err = "mixture spec: duration, sample_rate, channels must be positive";
    return 9;
  }
  if (n_speakers < 1) {
    g_err = "mixture spec: no speakers";
    return 9;
  }
  for (int k = 0; k < n_speakers; ++k) {
    if (seg_offsets[k + 1] <= seg_offsets[k]) {
      g_err = "mixture spec: speaker has no segments";
      return 9;
    }
    for (int s = seg_offsets[k]; s < seg_offsets[k + 1]; ++s)
      if (seg_start[s] < 0 || seg_dur[s] <= 0 || seg_start[s] + seg_dur[s] > duration) {
        g_err = "mixture spec: segment outside [0, duration)";
        return 9;
      }
  }
  if (reverb_t60 < 0 || reverb_t60 > 2.0) {
    g_err = "mixture spec: reverb_t60 must be in [0, 2]";
    return 9;
  }
  const int sr = sample_rate;
  const int64_t n = std::llround(duration * sr);
  const int m = channels;
  std::vector<std::vector<float>> mix(m, std::vector<float>(n, 0.0f));
  std::vector<std::vector<float>> dry_k(n_speakers, std::vector<float>(n, 0.0f));
  for (int k = 0; k < n_speakers; ++k) {
    int idx = 0;
    for (int s = seg_offsets[k]; s < seg_offsets[k + 1]; ++s, ++idx) {
      const int64_t s0 = std::llround(seg_start[s] * sr);
      const int64_t len = std::llround(seg_dur[s] * sr);
      SplitMix64 rng(derive_seed(seed, 1000 + k, idx));
      render_source(dry_k[k], s0, std::min(len, n - s0), sr, k, rng);
    }
  }
  for (int k = 0; k < n_speakers; ++k) {
    for (int c = 0; c < m; ++c) {
      const int d = steering_delay(k, c);
      std::vector<float> sig;
      if (reverb_t60 > 0.0) {
        SplitMix64 rng(derive_seed(seed, 2000 + k, c));
        sig = fft_convolve(dry_k[k], exponential_ir(d, reverb_t60, sr, 0.5, rng));
      } else {
        sig.assign(n, 0.0f);
        for (int64_t i = d; i < n; ++i) sig[i] = dry_k[k][i - d];
      }
      for (int64_t i = 0; i < n; ++i) mix[c][i] += sig[i];
      if (c == 0 && images0) std::memcpy(images0 + static_cast<size_t>(k) * n, sig.data(), n * sizeof(float));
    }
    if (dry) std::memcpy(dry + static_cast<size_t>(k) * n, dry_k[k].data(), n * sizeof(float));
  }
  double power = 0.0;
  for (int c = 0; c < m; ++c)
    for (int64_t i = 0; i < n; ++i) power += static_cast<double>(mix[c][i]) * mix[c][i];
  power /= static_cast<double>(m) * n;
  const double sigma = std::sqrt(power / std::pow(10.0, noise_snr / 10.0));
  for (int c = 0; c < m; ++c) {
    SplitMix64 rng(derive_seed(seed, 4000, c));
    for (int64_t i = 0; i < n; ++i) mix[c][i] += static_cast<float>(sigma * rng.gaussian());
    std::memcpy(mixture + static_cast<size_t>(c) * n, mix[c].data(), n * sizeof(float));
  }
  return 0;
}

}  // extern "C"
