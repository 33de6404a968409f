// gss/manifests.hpp (B200 build, hot-path part) -- manifests.hpp:42-68 and :372-433 of the reference:
// Segment, ActivityMatrix, build_activity_at, build_activity. File formats (JSONL / RTTM / WAV) are out of
// scope of this build.
#pragma once

#include <string>
#include <vector>

#include "stft.hpp"

namespace gss::manifests {

struct Segment {  // manifests.hpp:42-51
  std::string id;
  std::string recording_id;
  std::string speaker;
  double start = 0.0;
  double duration = 0.0;
  double end() const { return start + duration; }
};

struct ActivityMatrix {  // manifests.hpp:58-68
  int64_t frames = 0;
  std::vector<std::string> classes;
  int target_index = 0;
  int noise_index = -1;
  std::vector<uint8_t> grid;  // (T,K) frame-major
  int num_classes() const { return static_cast<int>(classes.size()); }
  uint8_t at(int64_t t, int k) const { return grid[t * num_classes() + k]; }
  void set(int64_t t, int k, uint8_t v) { grid[t * num_classes() + k] = v; }
};

inline ActivityMatrix build_activity_at(const std::vector<Segment>& segments,
                                        const std::vector<int64_t>& frame_center_samples, int sample_rate,
                                        const std::string& target, bool noise_class) {  // manifests.hpp:372-414
  std::vector<const char*> spk;
  std::vector<double> starts, durs;
  size_t label_bytes = target.size() + 16;
  for (const auto& s : segments) {
    spk.push_back(s.speaker.c_str());
    starts.push_back(s.start);
    durs.push_back(s.duration);
    label_bytes += s.speaker.size() + 1;
  }
  const int64_t t_count = static_cast<int64_t>(frame_center_samples.size());
  const size_t kmax = segments.size() + 2;
  std::vector<uint8_t> grid(static_cast<size_t>(t_count) * kmax);
  std::vector<char> labels(label_bytes + 8);
  int32_t nk = 0, ti = 0, ni = -1;
  b200::check_host(gss_b200_build_activity_at(
      static_cast<int32_t>(segments.size()), spk.data(), starts.data(), durs.data(), frame_center_samples.data(),
      t_count, sample_rate, target.c_str(), noise_class ? 1 : 0, grid.data(), static_cast<int64_t>(grid.size()), &nk,
      &ti, &ni, labels.data(), static_cast<int32_t>(labels.size())));
  ActivityMatrix act;
  act.frames = t_count;
  act.target_index = ti;
  act.noise_index = ni;
  std::string cur;
  for (const char* p = labels.data();; ++p) {
    if (*p == '\n' || *p == '\0') {
      act.classes.push_back(cur);
      cur.clear();
      if (*p == '\0') break;
    } else {
      cur.push_back(*p);
    }
  }
  act.grid.assign(grid.begin(), grid.begin() + static_cast<size_t>(t_count) * nk);
  return act;
}

inline ActivityMatrix build_activity(const std::vector<Segment>& segments, int64_t frame_begin, int64_t frame_end,
                                     const std::string& target, const stft::StftConfig& cfg, bool noise_class) {
  // manifests.hpp:419-433
  if (frame_end < frame_begin) throw ShapeError("build_activity: frame window is inverted");
  std::vector<int64_t> centers(frame_end - frame_begin);
  for (int64_t t = 0; t < frame_end - frame_begin; ++t) centers[t] = stft::frame_center(frame_begin + t, cfg);
  return build_activity_at(segments, centers, cfg.sample_rate, target, noise_class);
}

}  // namespace gss::manifests
