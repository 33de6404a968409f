// gss/scheduler.hpp (B200 build, hot-path part) -- scheduler.hpp:30-82 PipelineConfig, :165-180 SuperSegment,
// :283-294 EnhancementResult, :303-308 output_name, :314-365 enhance_batch of the reference, plus
// enhance_batches: the same operator over many independent SuperSegments in ONE device batch (the
// north star's `enhance(segment batch, activity guide)`), of which enhance_batch is the size-1 case.
// plan_batches / assemble's audio I/O / run_pipeline are out of scope of this build.
#pragma once

#include <cmath>
#include <cstdio>
#include <exception>
#include <string>
#include <vector>

#include "beamform.hpp"
#include "cacgmm.hpp"
#include "manifests.hpp"
#include "stft.hpp"
#include "wpe.hpp"

namespace gss::scheduler {

struct PipelineConfig {  // scheduler.hpp:30-44
  double max_batch_duration = 50.0;
  double context_duration = 15.0;
  int bss_iterations = 20;
  bool enable_wpe = true;
  bool noise_class = true;
  wpe::WpeConfig wpe;
  stft::StftConfig stft;
  std::string out_dir = ".";
  void validate() const {  // scheduler.hpp:46-57
    if (bss_iterations < 1) throw ConfigError("scheduler: bss_iterations must be >= 1");
    wpe.validate();
    stft.validate();
  }
  gss_pipeline_config c() const { return gss_pipeline_config{stft.c(), wpe.c(), enable_wpe ? 1 : 0, bss_iterations}; }
};

struct SuperSegment {  // scheduler.hpp:165-180
  std::string recording_id;
  std::string speaker;
  struct Part {
    manifests::Segment segment;
    int64_t sample_begin = 0;
    int64_t sample_end = 0;
  };
  std::vector<Part> parts;
  double context_left = 0.0;
  double context_right = 0.0;
  stft::RealSignal audio;
  std::vector<int64_t> frame_centers;
  manifests::ActivityMatrix activity;
  int64_t batch_index = 0;
};

struct SegmentOutput {  // scheduler.hpp:277-281
  std::string segment_id;
  std::string path;
  stft::RealSignal audio;  // mono
};

struct EnhancementResult {  // scheduler.hpp:283-294
  std::vector<SegmentOutput> outputs;
  double ll_final = 0.0;
  int64_t zeroed_bins = 0;
  int ref_channel = 0;
  int64_t frames = 0;
  double stft_seconds = 0.0, wpe_seconds = 0.0, mask_seconds = 0.0, beamform_seconds = 0.0, istft_seconds = 0.0;
  std::exception_ptr error;  // enhance_batches only: what enhance_batch would have thrown for this segment
};

inline std::string output_name(const std::string& rec, const std::string& spk, double start, double end) {
  // scheduler.hpp:303-308
  char buf[64];
  std::snprintf(buf, sizeof buf, "%07lld_%07lld", static_cast<long long>(std::llround(start * 1000.0)),
                static_cast<long long>(std::llround(end * 1000.0)));
  return rec + "-" + spk + "-" + buf + ".wav";
}

/// scheduler::enhance_batch for a batch of independent SuperSegments. A failing segment carries its
/// exception in `.error`; the others are unaffected (the reference fails one batch at a time,
/// scheduler.hpp:565-575).
inline std::vector<EnhancementResult> enhance_batches(const std::vector<const SuperSegment*>& batch,
                                                      const PipelineConfig& cfg,
                                                      b200::Device& dev = b200::Device::current()) {
  cfg.validate();
  const size_t n = batch.size();
  std::vector<gss_segment_desc> desc(n);
  std::vector<gss_segment_diag> diag(n);
  std::vector<std::vector<float>> audio(n), wave(n);
  std::vector<std::vector<int64_t>> pb(n), pe(n), len(n);
  std::vector<EnhancementResult> res(n);
  for (size_t i = 0; i < n; ++i) {
    const SuperSegment& ss = *batch[i];
    gss_segment_desc& d = desc[i];
    d = gss_segment_desc{};
    try {
      audio[i] = stft::detail::flatten(ss.audio);
    } catch (...) {
      res[i].error = std::current_exception();
      audio[i].clear();
    }
    int64_t cap = 0;
    const int64_t ns = ss.audio.num_samples();
    for (const auto& p : ss.parts) {
      pb[i].push_back(p.sample_begin);
      pe[i].push_back(p.sample_end);
      cap += std::max<int64_t>(0, std::min<int64_t>(p.sample_end, ns) - p.sample_begin);
    }
    wave[i].assign(static_cast<size_t>(std::max<int64_t>(cap, 1)), 0.0f);
    len[i].assign(ss.parts.size() + 1, 0);
    d.audio = audio[i].data();
    d.channels = res[i].error ? 0 : ss.audio.num_channels();
    d.sample_rate = ss.audio.sample_rate;
    d.num_samples = ns;
    d.activity = ss.activity.grid.data();
    d.activity_frames = ss.activity.frames;
    d.num_classes = ss.activity.num_classes();
    d.target_index = ss.activity.target_index;
    d.noise_index = ss.activity.noise_index;
    d.num_parts = static_cast<int32_t>(ss.parts.size());
    d.part_begin = pb[i].data();
    d.part_end = pe[i].data();
    d.out_wave = wave[i].data();
    d.out_lengths = len[i].data();
  }
  const gss_pipeline_config c = cfg.c();
  dev.check(gss_b200_enhance_batch(dev.get(), static_cast<int32_t>(n), desc.data(), &c, diag.data()));
  double ms[GSS_B200_NUM_STAGES] = {0};
  gss_b200_stage_ms(dev.get(), ms);
  for (size_t i = 0; i < n; ++i) {
    const SuperSegment& ss = *batch[i];
    EnhancementResult& r = res[i];
    r.frames = diag[i].frames;
    if (r.error) continue;
    if (diag[i].status != GSS_OK) {
      try {
        b200::raise(diag[i].status, "enhance_batch: segment failed on the device path",
                    static_cast<long>(diag[i].error_frequency));
      } catch (...) {
        r.error = std::current_exception();
      }
      continue;
    }
    r.ll_final = diag[i].ll_final;
    r.zeroed_bins = diag[i].zeroed_bins;
    r.ref_channel = diag[i].ref_channel;
    r.stft_seconds = ms[0] * 1e-3 / n;
    r.wpe_seconds = ms[1] * 1e-3 / n;
    r.mask_seconds = ms[2] * 1e-3 / n;
    r.beamform_seconds = ms[3] * 1e-3 / n;
    r.istft_seconds = ms[4] * 1e-3 / n;
    int64_t off = 0;
    for (size_t p = 0; p < ss.parts.size(); ++p) {
      SegmentOutput o;
      const auto& seg = ss.parts[p].segment;
      o.segment_id = seg.id;
      o.path = cfg.out_dir + "/" + output_name(ss.recording_id, ss.speaker, seg.start, seg.end());
      o.audio.sample_rate = cfg.stft.sample_rate;
      o.audio.channels.emplace_back(wave[i].begin() + off, wave[i].begin() + off + len[i][p]);
      off += len[i][p];
      r.outputs.push_back(std::move(o));
    }
  }
  return res;
}

/// scheduler::enhance_batch (scheduler.hpp:314-365): the reference's signature and error behaviour.
inline EnhancementResult enhance_batch(const SuperSegment& ss, const PipelineConfig& cfg,
                                       b200::Device& dev = b200::Device::current()) {
  std::vector<EnhancementResult> r = enhance_batches({&ss}, cfg, dev);
  if (r[0].error) std::rethrow_exception(r[0].error);
  return std::move(r[0]);
}

}  // namespace gss::scheduler
