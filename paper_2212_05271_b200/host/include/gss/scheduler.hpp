// gss/scheduler.hpp (B200 build) -- the reference's scheduler.hpp: PipelineConfig (:30-82), plan_batches
// (:101-160), SuperSegment / assemble (:165-275), EnhancementResult (:283-294), output_name (:303-308),
// enhance_batch (:314-365), OrderedBatchQueue (:383-412) and run_pipeline (:423-638), plus enhance_batches:
// the hot path over many independent SuperSegments in ONE device batch (the north star's `enhance(segment
// batch, activity guide)`), of which enhance_batch is the size-1 case. run_pipeline's compute consumer is
// one slot per GPU taking several loaded batches per device call; everything else keeps the reference's
// contract (plan order, failure isolation, summary keys, worker-count-invariant output bytes).
#pragma once

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <condition_variable>
#include <cstdio>
#include <deque>
#include <exception>
#include <filesystem>
#include <functional>
#include <future>
#include <map>
#include <memory>
#include <mutex>
#include <optional>
#include <set>
#include <string>
#include <thread>
#include <utility>
#include <unordered_map>
#include <vector>

#include "beamform.hpp"
#include "cacgmm.hpp"
#include "manifests.hpp"
#include "stft.hpp"
#include "wav.hpp"
#include "wpe.hpp"

namespace gss::scheduler {

enum class BatchMode { kSuperSegment, kOnePerBatch };  // scheduler.hpp:28

struct PipelineConfig {  // scheduler.hpp:30-82
  double max_batch_duration = 50.0;
  double context_duration = 15.0;
  int bss_iterations = 20;
  bool enable_wpe = true;
  bool noise_class = true;
  std::vector<int> channels;  // stacked-channel subset; empty = all
  BatchMode mode = BatchMode::kSuperSegment;
  int workers = 0;         // data-loader threads; 0 = fully synchronous
  int queue_capacity = 2;  // prefetch depth of the loader -> compute queue
  uint64_t seed = 0;       // echoed into the summary; the pipeline is deterministic
  std::string out_dir = ".";
  wpe::WpeConfig wpe;
  stft::StftConfig stft;
  std::vector<std::pair<std::string, std::string>> extra_echo;
  void validate() const {  // scheduler.hpp:46-57
    if (max_batch_duration <= 0 || context_duration < 0) throw ConfigError("scheduler: durations must be positive");
    if (bss_iterations < 1) throw ConfigError("scheduler: bss_iterations must be >= 1");
    if (workers < 0 || queue_capacity < 1)
      throw ConfigError("scheduler: workers >= 0 and queue_capacity >= 1 required");
    wpe.validate();
    stft.validate();
  }
  /// Flag-style echo of every knob as a JSON object (scheduler.hpp:60-81), `indent` spaces deep.
  std::string echo(int indent = 2) const {
    using manifests::detail::json_escape;
    using manifests::detail::json_number;
    std::vector<std::pair<std::string, std::string>> kv = {
        {"max-batch-duration", json_number(max_batch_duration)},
        {"context-duration", json_number(context_duration)},
        {"bss-iterations", std::to_string(bss_iterations)},
        {"no-wpe", enable_wpe ? "false" : "true"},
        {"no-noise-class", noise_class ? "false" : "true"}};
    std::string ch = "[";
    for (size_t i = 0; i < channels.size(); ++i) ch += (i ? ", " : "") + std::to_string(channels[i]);
    kv.emplace_back("channels", ch + "]");
    kv.emplace_back("one-per-batch", mode == BatchMode::kOnePerBatch ? "true" : "false");
    kv.emplace_back("workers", std::to_string(workers));
    kv.emplace_back("queue-capacity", std::to_string(queue_capacity));
    kv.emplace_back("seed", std::to_string(seed));
    kv.emplace_back("out-dir", json_escape(out_dir));
    kv.emplace_back("wpe-taps", std::to_string(wpe.taps));
    kv.emplace_back("wpe-delay", std::to_string(wpe.delay));
    kv.emplace_back("wpe-iterations", std::to_string(wpe.iterations));
    kv.emplace_back("fft-size", std::to_string(stft.fft_size));
    kv.emplace_back("shift", std::to_string(stft.shift));
    for (const auto& e : extra_echo) kv.emplace_back(e.first, json_escape(e.second));
    const std::string pad(indent + 2, ' ');
    std::string out = "{\n";
    for (size_t i = 0; i < kv.size(); ++i)
      out += pad + json_escape(kv[i].first) + ": " + kv[i].second + (i + 1 < kv.size() ? ",\n" : "\n");
    return out + std::string(indent, ' ') + "}";
  }
  gss_pipeline_config c() const { return gss_pipeline_config{stft.c(), wpe.c(), enable_wpe ? 1 : 0, bss_iterations}; }
};

/// One planned batch: same-recording, same-speaker segments concatenated along time (scheduler.hpp:86-96).
struct BatchPlan {
  std::string recording_id;
  std::string speaker;
  std::vector<manifests::Segment> parts;  // temporal order
  double total_duration() const {
    double d = 0;
    for (const auto& p : parts) d += p.duration;
    return d;
  }
};

/// The batch plan (the reference's contract, scheduler.hpp:101-160): segments of one (recording, speaker) pair are
/// packed in temporal order into batches of at most `max_batch_duration` seconds of speech; a segment longer than
/// the cap is a batch of its own, and so is every segment in one-per-batch mode. Batches are emitted in rounds:
/// first batch of every pair (pairs in order of first appearance), then the second of every pair, and so on.
inline std::vector<BatchPlan> plan_batches(const std::vector<manifests::Segment>& segments, double max_batch_duration,
                                           BatchMode mode = BatchMode::kSuperSegment) {
  // pair number of every segment, in order of first appearance
  std::unordered_map<std::string, int> pair_of;
  std::vector<int> pair(segments.size());
  for (size_t i = 0; i < segments.size(); ++i)
    pair[i] = pair_of.emplace(segments[i].recording_id + '\n' + segments[i].speaker, static_cast<int>(pair_of.size()))
                  .first->second;
  // one pass over the segments sorted by (pair, start, id)
  std::vector<size_t> by_time(segments.size());
  for (size_t i = 0; i < by_time.size(); ++i) by_time[i] = i;
  std::sort(by_time.begin(), by_time.end(), [&](size_t x, size_t y) {
    if (pair[x] != pair[y]) return pair[x] < pair[y];
    if (segments[x].start != segments[y].start) return segments[x].start < segments[y].start;
    return segments[x].id < segments[y].id;
  });
  struct Ranked {
    int rank;  // position of the batch within its pair
    int pair;
    BatchPlan plan;
  };
  std::vector<Ranked> made;
  int current = -1;
  bool open = false;   // the last batch of `current` may still take segments
  double filled = 0;
  for (const size_t i : by_time) {
    const manifests::Segment& seg = segments[i];
    if (pair[i] != current) {
      current = pair[i];
      open = false;
    }
    const bool solitary = mode == BatchMode::kOnePerBatch || seg.duration > max_batch_duration;
    if (solitary || !open || filled + seg.duration > max_batch_duration) {
      const int rank = (!made.empty() && made.back().pair == current) ? made.back().rank + 1 : 0;
      made.push_back(Ranked{rank, current, BatchPlan{seg.recording_id, seg.speaker, {}}});
      filled = 0;
      open = !solitary;
    }
    made.back().plan.parts.push_back(seg);
    filled += seg.duration;
  }
  std::stable_sort(made.begin(), made.end(), [](const Ranked& x, const Ranked& y) {
    return x.rank != y.rank ? x.rank < y.rank : x.pair < y.pair;
  });
  std::vector<BatchPlan> plans;
  plans.reserve(made.size());
  for (Ranked& r : made) plans.push_back(std::move(r.plan));
  return plans;
}

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

/// Reads the audio spans of one plan ([left context][parts with the gaps removed][right context]) and builds
/// the activity guide over the assembled frames (scheduler.hpp:185-275). `all_segments` must hold every
/// segment of the plan's recording (any speaker) so that cross-speaker activity is right inside the context
/// windows. The span / offset / frame-centre arithmetic is the library's host code (bit-exact integer work).
inline SuperSegment assemble(const BatchPlan& plan, const manifests::Recording& rec,
                             const std::vector<manifests::Segment>& all_segments, const PipelineConfig& cfg) {
  SuperSegment ss;
  ss.recording_id = plan.recording_id;
  ss.speaker = plan.speaker;
  const int sr = rec.sample_rate;
  const int64_t rec_samples = rec.num_samples();
  const size_t n = plan.parts.size();
  std::vector<double> starts, durs;
  for (const auto& seg : plan.parts) {
    const int64_t s0 = std::llround(seg.start * sr);
    const int64_t s1 = std::min<int64_t>(rec_samples, std::llround(seg.end() * sr));
    if (s1 <= s0) throw ShapeError("segment '" + seg.id + "' maps to an empty sample range");
    starts.push_back(seg.start);
    durs.push_back(seg.duration);
  }
  std::vector<int64_t> spans(2 * (n + 2)), pb(n), pe(n);
  // spans are concatenated: overlapping parts make the assembled signal longer than the recording, so the
  // frame-centre buffer is sized from the span total (each span is within a sample of llround(duration * sr))
  int64_t total_cap = 2 * (std::llround(std::max(cfg.context_duration, 0.0) * sr) + 1);
  for (double d : durs) total_cap += std::llround(std::max(d, 0.0) * sr) + 1;
  const int64_t cap = total_cap / std::max(cfg.stft.shift, 1) + 2 + 2 * static_cast<int64_t>(n);
  std::vector<int64_t> centers(static_cast<size_t>(cap));
  int32_t n_spans = 0;
  int64_t total = 0, n_centers = 0;
  b200::check_host(gss_b200_assemble_indices(static_cast<int32_t>(n), starts.data(), durs.data(), sr, rec_samples,
                                             cfg.context_duration, cfg.stft.fft_size, cfg.stft.shift, spans.data(),
                                             &n_spans, pb.data(), pe.data(), &total, centers.data(), cap, &n_centers,
                                             &ss.context_left, &ss.context_right));
  ss.audio.sample_rate = sr;
  int64_t off = 0;
  for (int32_t i = 0; i < n_spans; ++i) {
    const int64_t b = spans[2 * i], e = spans[2 * i + 1];
    stft::RealSignal piece = manifests::load_audio(rec, b, e - b, cfg.channels);
    if (ss.audio.channels.empty())
      ss.audio.channels.assign(piece.num_channels(), std::vector<float>(static_cast<size_t>(total), 0.0f));
    for (int c = 0; c < piece.num_channels(); ++c)
      std::copy(piece.channels[c].begin(), piece.channels[c].end(), ss.audio.channels[c].begin() + off);
    off += e - b;
  }
  for (size_t p = 0; p < n; ++p) ss.parts.push_back(SuperSegment::Part{plan.parts[p], pb[p], pe[p]});
  ss.frame_centers.assign(centers.begin(), centers.begin() + n_centers);
  std::vector<manifests::Segment> rec_segments;
  for (const auto& s : all_segments)
    if (s.recording_id == plan.recording_id) rec_segments.push_back(s);
  ss.activity = manifests::build_activity_at(rec_segments, ss.frame_centers, sr, plan.speaker, cfg.noise_class);
  return ss;
}

// ---------------------------------------------------------------------------
// run_pipeline (scheduler.hpp:366-638)
// ---------------------------------------------------------------------------
namespace detail {

/// What a loader hands to the compute side: the assembled super-segment of plan entry `index`, or why it could
/// not be assembled (the role of the reference's LoadedBatch, scheduler.hpp:371-376).
struct LoadedBatch {
  int64_t index = 0;
  std::optional<SuperSegment> batch;  // empty on load failure
  std::string error;
  double load_seconds = 0.0;
};

/// Re-sequencer between the loader threads and the compute side. Loaders finish in any order; the consumer gets
/// plan entries 0, 1, 2, ... . At most `capacity` entries ahead of the consumer are admitted, so a loader that
/// runs far ahead waits instead of piling up audio in memory. This is what makes the worker count invisible in the
/// output (the contract of the reference's OrderedBatchQueue, scheduler.hpp:383-412). Here: a ring of `capacity`
/// slots addressed by index modulo capacity, one mutex, one condition variable.
class OrderedBatchQueue {
 public:
  explicit OrderedBatchQueue(int64_t capacity) : ring_(static_cast<size_t>(capacity < 1 ? 1 : capacity)) {}

  /// Blocks while item.index is `capacity` or more entries ahead of the consumer.
  void put(LoadedBatch&& item) {
    const int64_t n = static_cast<int64_t>(ring_.size());
    std::unique_lock<std::mutex> hold(lock_);
    changed_.wait(hold, [&] { return item.index - head_ < n; });
    ring_[static_cast<size_t>(item.index % n)] = std::move(item);
    changed_.notify_all();
  }

  /// Blocks until the next entry in plan order has arrived.
  LoadedBatch take() {
    std::unique_lock<std::mutex> hold(lock_);
    std::optional<LoadedBatch>& slot = ring_[static_cast<size_t>(head_ % static_cast<int64_t>(ring_.size()))];
    changed_.wait(hold, [&] { return slot.has_value(); });
    LoadedBatch out = std::move(*slot);
    slot.reset();
    ++head_;
    changed_.notify_all();
    return out;
  }

 private:
  std::vector<std::optional<LoadedBatch>> ring_;
  std::mutex lock_;
  std::condition_variable changed_;
  int64_t head_ = 0;  // plan index the consumer takes next
};

inline double seconds_since(std::chrono::steady_clock::time_point t0) {
  return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

/// One GPU: a thread that owns a b200::Device and runs the device batches handed to it in order.
class ComputeSlot {
 public:
  using Results = std::vector<EnhancementResult>;
  explicit ComputeSlot(int device) : thread_([this, device] { loop(device); }) {}
  ~ComputeSlot() {
    {
      std::lock_guard<std::mutex> lock(mu_);
      done_ = true;
    }
    cv_.notify_all();
    thread_.join();
  }
  std::future<Results> submit(std::function<Results(b200::Device&)> fn) {
    auto promise = std::make_shared<std::promise<Results>>();
    auto fut = promise->get_future();
    {
      std::lock_guard<std::mutex> lock(mu_);
      jobs_.push_back([promise, fn = std::move(fn)](b200::Device* dev, const std::string& why) {
        try {
          if (!dev) throw DeviceError(why);
          promise->set_value(fn(*dev));
        } catch (...) {
          promise->set_exception(std::current_exception());
        }
      });
    }
    cv_.notify_all();
    return fut;
  }

 private:
  void loop(int device) {
    std::unique_ptr<b200::Device> dev;
    std::string why;
    for (;;) {
      std::function<void(b200::Device*, const std::string&)> job;
      {
        std::unique_lock<std::mutex> lock(mu_);
        cv_.wait(lock, [&] { return done_ || !jobs_.empty(); });
        if (jobs_.empty()) return;
        job = std::move(jobs_.front());
        jobs_.pop_front();
      }
      if (!dev && why.empty()) {  // the context is created on the slot's own thread, once
        try {
          dev = std::make_unique<b200::Device>(device);
        } catch (const std::exception& e) {
          why = e.what();
        }
      }
      job(dev.get(), why);
    }
  }
  std::mutex mu_;
  std::condition_variable cv_;
  std::deque<std::function<void(b200::Device*, const std::string&)>> jobs_;
  bool done_ = false;
  std::thread thread_;
};

}  // namespace detail

struct RunSummary {  // scheduler.hpp:414-417; `json` is the text written to summary.json
  std::string json;
  int failed_segments = 0;
  int segments_written = 0;
  int64_t num_batches = 0;
  struct Failure {
    std::string segment_id;
    int64_t batch = -1;
    std::string error;
  };
  struct Batch {
    int64_t batch = 0, frames = 0, segments = 0, zeroed_bins = 0;
    std::string speaker;
    int ref_channel = 0;
    double log_likelihood = 0.0;
  };
  struct Output {
    std::string segment_id, path;
    int64_t samples = 0;
  };
  std::vector<Failure> failures;
  std::vector<Batch> batches;
  std::vector<Output> outputs;
  std::map<std::string, double> stage_seconds;
  double processed_audio_seconds = 0.0;
};

/// plan -> (loader threads) assemble -> enhance -> write, with a JSON summary (scheduler.hpp:423-638). The
/// compute slots are GPUs (`devices`): loaded batches are taken from the ordered queue in plan order, grouped
/// `gpu_batch` at a time into one device call and dealt to the slots round-robin; results are consumed strictly
/// in plan order, so outputs, summary and written bytes do not depend on the worker count, the number of GPUs
/// or the grouping (a segment's result is independent of its device batch).
inline RunSummary run_pipeline(const std::vector<manifests::Recording>& recordings,
                               const std::vector<manifests::Segment>& segments, const PipelineConfig& cfg,
                               std::vector<int> devices = {0}, int gpu_batch = 16) {
  using manifests::detail::json_escape;
  using manifests::detail::json_number;
  cfg.validate();
  const auto wall0 = std::chrono::steady_clock::now();
  if (const std::vector<std::string> findings = manifests::validate(recordings, segments); !findings.empty()) {
    std::string report = "manifest validation failed:";
    for (const std::string& line : findings) report.append("\n  ").append(line);
    throw ConfigError(report);
  }
  std::filesystem::create_directories(cfg.out_dir);
  std::unordered_map<std::string, const manifests::Recording*> rec_by_id;
  rec_by_id.reserve(recordings.size());
  for (const manifests::Recording& r : recordings) rec_by_id.emplace(r.id, &r);
  const std::vector<BatchPlan> plans = plan_batches(segments, cfg.max_batch_duration, cfg.mode);
  if (devices.empty()) devices.push_back(0);
  if (gpu_batch < 1) gpu_batch = 1;

  RunSummary run;
  run.num_batches = static_cast<int64_t>(plans.size());
  double load_s = 0, write_s = 0;
  std::map<std::string, double> stage;
  std::set<std::pair<int, int>> shapes;

  auto load_one = [&](int64_t i) {
    detail::LoadedBatch item;
    item.index = i;
    const auto t0 = std::chrono::steady_clock::now();
    try {
      item.batch = assemble(plans[i], *rec_by_id.at(plans[i].recording_id), segments, cfg);
      item.batch->batch_index = i;
    } catch (const std::exception& e) {  // a load failure fails every part of that batch, the run continues
      item.batch.reset();
      item.error = e.what();
    }
    item.load_seconds = detail::seconds_since(t0);
    return item;
  };

  // writer: a single thread keeps file output off the compute path, preserving enqueue order
  std::mutex write_mu;
  std::condition_variable write_cv;
  std::deque<SegmentOutput> write_queue;
  std::vector<std::pair<std::string, std::string>> write_failures;
  bool write_done = false;
  auto do_write = [&](const SegmentOutput& out) {
    try {
      wav::write(out.path, out.audio);
    } catch (const std::exception& e) {
      std::lock_guard<std::mutex> lock(write_mu);
      write_failures.emplace_back(out.segment_id, e.what());
    }
  };
  std::thread writer;
  if (cfg.workers > 0)
    writer = std::thread([&] {
      std::unique_lock<std::mutex> lock(write_mu);
      for (;;) {
        write_cv.wait(lock, [&] { return write_done || !write_queue.empty(); });
        if (write_queue.empty()) return;
        SegmentOutput out = std::move(write_queue.front());
        write_queue.pop_front();
        lock.unlock();
        const auto t0 = std::chrono::steady_clock::now();
        do_write(out);
        lock.lock();
        write_s += detail::seconds_since(t0);
      }
    });

  auto fail_batch = [&](int64_t index, const std::string& error) {
    for (const auto& part : plans[index].parts) {
      run.failures.push_back({part.id, index, error});
      ++run.failed_segments;
    }
  };
  auto consume = [&](detail::LoadedBatch& item, EnhancementResult* result) {  // strictly in plan order
    load_s += item.load_seconds;
    if (!item.batch) return fail_batch(item.index, item.error);
    if (result->error) {  // pooled statistics make the whole batch fail together
      try {
        std::rethrow_exception(result->error);
      } catch (const std::exception& e) {
        return fail_batch(item.index, e.what());
      }
    }
    const SuperSegment& ss = *item.batch;
    run.processed_audio_seconds += static_cast<double>(ss.audio.num_samples()) / ss.audio.sample_rate;
    shapes.insert({ss.audio.num_channels(), ss.activity.num_classes()});
    stage["stft"] += result->stft_seconds;
    stage["wpe"] += result->wpe_seconds;
    stage["mask"] += result->mask_seconds;
    stage["beamform"] += result->beamform_seconds;
    stage["istft"] += result->istft_seconds;
    run.batches.push_back({item.index, result->frames, static_cast<int64_t>(ss.parts.size()), result->zeroed_bins,
                           ss.speaker, result->ref_channel, result->ll_final});
    for (auto& out : result->outputs) {
      run.outputs.push_back({out.segment_id, out.path, out.audio.num_samples()});
      ++run.segments_written;
      if (cfg.workers > 0) {
        std::lock_guard<std::mutex> lock(write_mu);
        write_queue.push_back(std::move(out));
        write_cv.notify_one();
      } else {
        const auto t0 = std::chrono::steady_clock::now();
        do_write(out);
        write_s += detail::seconds_since(t0);
      }
    }
  };

  {
    std::vector<std::unique_ptr<detail::ComputeSlot>> slots;
    for (const int d : devices) slots.push_back(std::make_unique<detail::ComputeSlot>(d));
    struct InFlight {
      std::shared_ptr<std::vector<detail::LoadedBatch>> items;
      std::future<std::vector<EnhancementResult>> fut;
      bool has_job = false;
    };
    std::deque<InFlight> inflight;
    auto drain = [&](size_t limit) {
      while (inflight.size() > limit) {
        InFlight f = std::move(inflight.front());
        inflight.pop_front();
        std::vector<EnhancementResult> results;
        std::string device_error;
        if (f.has_job) {
          try {
            results = f.fut.get();
          } catch (const std::exception& e) {
            device_error = e.what();
          }
        }
        size_t r = 0;
        for (auto& it : *f.items) {
          if (!it.batch) {
            consume(it, nullptr);
          } else if (!device_error.empty()) {
            fail_batch(it.index, device_error);
          } else {
            consume(it, &results[r++]);
          }
        }
      }
    };
    size_t n_chunks = 0;
    auto submit = [&](std::shared_ptr<std::vector<detail::LoadedBatch>> items) {
      InFlight f;
      f.items = items;
      bool any = false;
      for (const auto& it : *items) any = any || it.batch.has_value();
      if (any) {
        f.has_job = true;
        f.fut = slots[n_chunks % slots.size()]->submit([items, &cfg](b200::Device& dev) {
          std::vector<const SuperSegment*> batch;
          for (const auto& it : *items)
            if (it.batch) batch.push_back(&*it.batch);
          return enhance_batches(batch, cfg, dev);
        });
      }
      ++n_chunks;
      inflight.push_back(std::move(f));
      drain(2 * slots.size());  // at most two device batches queued per GPU
    };

    std::vector<std::thread> loaders;
    std::unique_ptr<detail::OrderedBatchQueue> queue;
    std::atomic<int64_t> next_plan{0};
    if (cfg.workers > 0) {
      queue = std::make_unique<detail::OrderedBatchQueue>(cfg.queue_capacity);
      for (int w = 0; w < cfg.workers; ++w)
        loaders.emplace_back([&] {
          for (;;) {
            const int64_t i = next_plan.fetch_add(1);
            if (i >= static_cast<int64_t>(plans.size())) return;
            queue->put(load_one(i));
          }
        });
    }
    auto chunk = std::make_shared<std::vector<detail::LoadedBatch>>();
    for (int64_t i = 0; i < static_cast<int64_t>(plans.size()); ++i) {
      chunk->push_back(cfg.workers > 0 ? queue->take() : load_one(i));
      if (static_cast<int>(chunk->size()) == gpu_batch) {
        submit(chunk);
        chunk = std::make_shared<std::vector<detail::LoadedBatch>>();
      }
    }
    if (!chunk->empty()) submit(chunk);
    drain(0);
    for (auto& t : loaders) t.join();
  }
  if (writer.joinable()) {
    {
      std::lock_guard<std::mutex> lock(write_mu);
      write_done = true;
    }
    write_cv.notify_all();
    writer.join();
  }
  for (const auto& wf : write_failures) {
    run.failures.push_back({wf.first, -1, "write failed: " + wf.second});
    ++run.failed_segments;
    --run.segments_written;
  }
  run.stage_seconds = {{"load", load_s},        {"stft", stage["stft"]},         {"wpe", stage["wpe"]},
                       {"mask", stage["mask"]},  {"beamform", stage["beamform"]}, {"istft", stage["istft"]},
                       {"write", write_s},       {"total", detail::seconds_since(wall0)}};

  // summary.json with the reference's keys (scheduler.hpp:618-636)
  std::string j = "{\n  \"config\": " + cfg.echo(2) + ",\n";
  j += "  \"num_recordings\": " + std::to_string(recordings.size()) + ",\n";
  j += "  \"num_segments\": " + std::to_string(segments.size()) + ",\n";
  j += "  \"num_batches\": " + std::to_string(plans.size()) + ",\n";
  j += "  \"segments_written\": " + std::to_string(run.segments_written) + ",\n  \"failures\": [";
  for (size_t i = 0; i < run.failures.size(); ++i) {
    const auto& f = run.failures[i];
    j += std::string(i ? "," : "") + "\n    {\"segment_id\": " + json_escape(f.segment_id);
    if (f.batch >= 0) j += ", \"batch\": " + std::to_string(f.batch);
    j += ", \"error\": " + json_escape(f.error) + "}";
  }
  j += std::string(run.failures.empty() ? "" : "\n  ") + "],\n  \"batches\": [";
  for (size_t i = 0; i < run.batches.size(); ++i) {
    const auto& b = run.batches[i];
    j += std::string(i ? "," : "") + "\n    {\"batch\": " + std::to_string(b.batch) + ", \"speaker\": " +
         json_escape(b.speaker) + ", \"frames\": " + std::to_string(b.frames) + ", \"segments\": " +
         std::to_string(b.segments) + ", \"ref_channel\": " + std::to_string(b.ref_channel) +
         ", \"zeroed_bins\": " + std::to_string(b.zeroed_bins) + ", \"log_likelihood\": " +
         json_number(b.log_likelihood) + "}";
  }
  j += std::string(run.batches.empty() ? "" : "\n  ") + "],\n  \"outputs\": [";
  for (size_t i = 0; i < run.outputs.size(); ++i) {
    const auto& o = run.outputs[i];
    j += std::string(i ? "," : "") + "\n    {\"segment_id\": " + json_escape(o.segment_id) + ", \"path\": " +
         json_escape(o.path) + ", \"samples\": " + std::to_string(o.samples) + "}";
  }
  j += std::string(run.outputs.empty() ? "" : "\n  ") + "],\n";
  // the reference reports its einsum planner's cache here; on the device that contraction is hard-coded per
  // (channels, classes) kernel specialisation, which plays the planner's role: one entry per shape used
  const size_t hits = run.batches.size() > shapes.size() ? run.batches.size() - shapes.size() : 0;
  j += "  \"plan_cache\": {\"entries\": " + std::to_string(shapes.size()) + ", \"computed\": " +
       std::to_string(shapes.size()) + ", \"hits\": " + std::to_string(hits) + "},\n  \"stage_seconds\": {";
  const char* order[] = {"load", "stft", "wpe", "mask", "beamform", "istft", "write", "total"};
  for (int i = 0; i < 8; ++i)
    j += std::string(i ? ", " : "") + "\"" + order[i] + "\": " + json_number(run.stage_seconds[order[i]]);
  j += "},\n  \"processed_audio_seconds\": " + json_number(run.processed_audio_seconds) + ",\n  \"devices\": [";
  for (size_t i = 0; i < devices.size(); ++i) j += (i ? ", " : "") + std::to_string(devices[i]);
  j += "]\n}\n";
  run.json = j;
  manifests::write_text(cfg.out_dir + "/summary.json", run.json);
  return run;
}

}  // namespace gss::scheduler
