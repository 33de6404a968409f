// gss/manifests.hpp (B200 build) -- the reference's manifests.hpp: Recording / Segment manifests (JSONL,
// gzip-transparent when built with GSS_WITH_ZLIB; RTTM), cross-manifest validation, the activity guide
// (build_activity_at / build_activity: bit-exact integer work in the library's host code) and multi-source
// audio loading. The reference parses JSON with nlohmann::json; this build carries a small reader for the
// flat objects the manifests use (gss::manifests::detail::Json).
#pragma once

#include <cctype>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <map>
#include <set>
#include <sstream>
#include <string>
#include <vector>

#ifdef GSS_WITH_ZLIB
#include <zlib.h>
#endif

#include "stft.hpp"
#include "wav.hpp"

namespace gss::manifests {

struct Source {  // manifests.hpp:22-25
  std::string path;
  std::vector<int> channels;
};

struct Recording {  // manifests.hpp:27-40
  std::string id;
  std::vector<Source> sources;
  int sample_rate = 0;
  double duration = 0.0;
  int channel_count() const {
    int m = 0;
    for (const auto& s : sources) m += static_cast<int>(s.channels.size());
    return m;
  }
  int64_t num_samples() const { return static_cast<int64_t>(std::llround(duration * sample_rate)); }
};

enum class SegmentFormat { kJsonl, kRttm };  // manifests.hpp:53

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

// ---------------------------------------------------------------------------
// file reading (gzip-transparent by extension), manifests.hpp:79-114
// ---------------------------------------------------------------------------
inline bool has_suffix(const std::string& s, const std::string& suffix) {
  return s.size() >= suffix.size() && s.compare(s.size() - suffix.size(), suffix.size(), suffix) == 0;
}

inline std::string read_text(const std::string& path) {
  if (has_suffix(path, ".gz")) {
#ifdef GSS_WITH_ZLIB
    gzFile gz = gzopen(path.c_str(), "rb");
    if (!gz) throw IoError("cannot open file: " + path);
    std::string out;
    char buf[1 << 16];
    int n;
    while ((n = gzread(gz, buf, sizeof buf)) > 0) out.append(buf, n);
    gzclose(gz);
    if (n < 0) throw IoError("gzip read failed: " + path);
    return out;
#else
    throw IoError("built without zlib (GSS_WITH_ZLIB): cannot read " + path);
#endif
  }
  std::ifstream in(path, std::ios::binary);
  if (!in) throw IoError("cannot open file: " + path);
  std::ostringstream ss;
  ss << in.rdbuf();
  return ss.str();
}

inline void write_text(const std::string& path, const std::string& content) {
  if (has_suffix(path, ".gz")) {
#ifdef GSS_WITH_ZLIB
    gzFile gz = gzopen(path.c_str(), "wb");
    if (!gz) throw IoError("cannot create file: " + path);
    const int n = gzwrite(gz, content.data(), static_cast<unsigned>(content.size()));
    gzclose(gz);
    if (n != static_cast<int>(content.size())) throw IoError("gzip write failed: " + path);
    return;
#else
    throw IoError("built without zlib (GSS_WITH_ZLIB): cannot write " + path);
#endif
  }
  std::ofstream os(path, std::ios::binary | std::ios::trunc);
  if (!os) throw IoError("cannot create file: " + path);
  os << content;
  if (!os) throw IoError("write failed: " + path);
}

namespace detail {

/// Minimal JSON value: what one manifest line needs (objects, arrays, strings, numbers, true/false/null).
struct Json {
  enum Kind { kNull, kBool, kNumber, kString, kArray, kObject } kind = kNull;
  double number = 0.0;
  bool boolean = false;
  std::string string;
  std::vector<Json> array;
  std::vector<std::pair<std::string, Json>> object;

  const Json& at(const std::string& key) const {
    if (kind != kObject) throw std::runtime_error("cannot use at() with a non-object value");
    for (const auto& kv : object)
      if (kv.first == key) return kv.second;
    throw std::runtime_error("key '" + key + "' not found");
  }
  double as_number() const {
    if (kind != kNumber) throw std::runtime_error("type must be number");
    return number;
  }
  const std::string& as_string() const {
    if (kind != kString) throw std::runtime_error("type must be string");
    return string;
  }
  const std::vector<Json>& as_array() const {
    if (kind != kArray) throw std::runtime_error("type must be array");
    return array;
  }
};

class JsonReader {
 public:
  explicit JsonReader(const std::string& text) : s_(text) {}
  Json parse() {
    Json v = value();
    ws();
    if (i_ != s_.size()) fail("unexpected trailing characters");
    return v;
  }

 private:
  [[noreturn]] void fail(const std::string& what) const {
    throw std::runtime_error("parse error at column " + std::to_string(i_ + 1) + ": " + what);
  }
  void ws() {
    while (i_ < s_.size() && (s_[i_] == ' ' || s_[i_] == '\t' || s_[i_] == '\r' || s_[i_] == '\n')) ++i_;
  }
  bool eat(char c) {
    ws();
    if (i_ < s_.size() && s_[i_] == c) {
      ++i_;
      return true;
    }
    return false;
  }
  Json value() {
    ws();
    if (i_ >= s_.size()) fail("unexpected end of input");
    const char c = s_[i_];
    Json v;
    if (c == '{') {
      ++i_;
      v.kind = Json::kObject;
      if (eat('}')) return v;
      do {
        ws();
        if (i_ >= s_.size() || s_[i_] != '"') fail("object key must be a string");
        std::string key = str();
        if (!eat(':')) fail("expected ':' after object key");
        v.object.emplace_back(std::move(key), value());
      } while (eat(','));
      if (!eat('}')) fail("expected ',' or '}' in object");
    } else if (c == '[') {
      ++i_;
      v.kind = Json::kArray;
      if (eat(']')) return v;
      do v.array.push_back(value());
      while (eat(','));
      if (!eat(']')) fail("expected ',' or ']' in array");
    } else if (c == '"') {
      v.kind = Json::kString;
      v.string = str();
    } else if (s_.compare(i_, 4, "true") == 0) {
      v.kind = Json::kBool;
      v.boolean = true;
      i_ += 4;
    } else if (s_.compare(i_, 5, "false") == 0) {
      v.kind = Json::kBool;
      i_ += 5;
    } else if (s_.compare(i_, 4, "null") == 0) {
      i_ += 4;
    } else {
      const char* b = s_.c_str() + i_;
      char* e = nullptr;
      v.number = std::strtod(b, &e);
      if (e == b || !(c == '-' || std::isdigit(static_cast<unsigned char>(c)))) fail("invalid literal");
      v.kind = Json::kNumber;
      i_ += static_cast<size_t>(e - b);
    }
    return v;
  }
  std::string str() {
    std::string out;
    for (++i_; i_ < s_.size() && s_[i_] != '"'; ++i_) {
      if (s_[i_] != '\\') {
        out.push_back(s_[i_]);
        continue;
      }
      if (++i_ >= s_.size()) break;
      switch (s_[i_]) {
        case 'n': out.push_back('\n'); break;
        case 't': out.push_back('\t'); break;
        case 'r': out.push_back('\r'); break;
        case 'b': out.push_back('\b'); break;
        case 'f': out.push_back('\f'); break;
        case 'u': {  // BMP code point -> UTF-8
          if (i_ + 4 >= s_.size()) fail("truncated \\u escape");
          const unsigned cp = static_cast<unsigned>(std::strtoul(s_.substr(i_ + 1, 4).c_str(), nullptr, 16));
          i_ += 4;
          if (cp < 0x80) {
            out.push_back(static_cast<char>(cp));
          } else if (cp < 0x800) {
            out.push_back(static_cast<char>(0xC0 | (cp >> 6)));
            out.push_back(static_cast<char>(0x80 | (cp & 0x3F)));
          } else {
            out.push_back(static_cast<char>(0xE0 | (cp >> 12)));
            out.push_back(static_cast<char>(0x80 | ((cp >> 6) & 0x3F)));
            out.push_back(static_cast<char>(0x80 | (cp & 0x3F)));
          }
          break;
        }
        default: out.push_back(s_[i_]);
      }
    }
    if (i_ >= s_.size()) fail("unterminated string");
    ++i_;
    return out;
  }
  const std::string s_;  // a copy: callers pass temporaries
  size_t i_ = 0;
};

inline std::string json_escape(const std::string& s) {
  std::string out = "\"";
  for (const char c : s) {
    if (c == '"' || c == '\\') {
      out.push_back('\\');
      out.push_back(c);
    } else if (c == '\n') {
      out += "\\n";
    } else if (c == '\t') {
      out += "\\t";
    } else if (c == '\r') {
      out += "\\r";
    } else {
      out.push_back(c);
    }
  }
  return out + "\"";
}

/// Shortest decimal that reads back as the same double, fixed notation with a ".0" on integral values for
/// decimal exponents in [-4, 16) and d.ddde[+-]xx outside (what nlohmann's dump() and Python's repr print).
inline std::string json_number(double v) {
  if (!std::isfinite(v)) return "null";
  if (v == 0) return std::signbit(v) ? "-0.0" : "0.0";
  char buf[40];
  int prec = 0;
  for (; prec <= 16; ++prec) {
    std::snprintf(buf, sizeof buf, "%.*e", prec, v);
    if (std::strtod(buf, nullptr) == v) break;
  }
  std::string digits;
  const char* p = buf;
  const bool neg = *p == '-';
  if (neg) ++p;
  for (; *p != 'e'; ++p)
    if (*p != '.') digits.push_back(*p);
  const int e10 = std::atoi(p + 1);
  while (digits.size() > 1 && digits.back() == '0') digits.pop_back();
  const int nd = static_cast<int>(digits.size());
  std::string out = neg ? "-" : "";
  if (e10 >= -4 && e10 < 16) {
    if (e10 < 0) {
      out += "0." + std::string(-e10 - 1, '0') + digits;
    } else if (nd <= e10 + 1) {
      out += digits + std::string(e10 + 1 - nd, '0') + ".0";
    } else {
      out += digits.substr(0, e10 + 1) + "." + digits.substr(e10 + 1);
    }
  } else {
    out += digits.substr(0, 1) + (nd > 1 ? "." + digits.substr(1) : "") + "e" + (e10 < 0 ? "-" : "+");
    const int ae = e10 < 0 ? -e10 : e10;
    out += (ae < 10 ? "0" : "") + std::to_string(ae);
  }
  return out;
}

inline std::string loc(const std::string& path, long line_no) { return path + ":" + std::to_string(line_no) + ": "; }

// Applies fn to every non-blank line; failures carry the 1-based line number (manifests.hpp:120-142).
template <typename Fn>
void for_each_jsonl(const std::string& path, Fn&& fn) {
  std::istringstream in(read_text(path));
  std::string line;
  long line_no = 0;
  while (std::getline(in, line)) {
    ++line_no;
    if (line.find_first_not_of(" \t\r") == std::string::npos) continue;
    Json j;
    try {
      j = JsonReader(line).parse();
    } catch (const std::runtime_error& e) {
      throw ParseError(loc(path, line_no) + "invalid JSON: " + e.what());
    }
    try {
      fn(j, line_no);
    } catch (const Error&) {
      throw;
    } catch (const std::runtime_error& e) {
      throw ParseError(loc(path, line_no) + e.what());
    }
  }
}

}  // namespace detail

// ---------------------------------------------------------------------------
// recording manifests (manifests.hpp:150-217)
// ---------------------------------------------------------------------------
inline std::vector<Recording> load_recordings(const std::string& path) {
  std::vector<Recording> out;
  std::set<std::string> seen;
  detail::for_each_jsonl(path, [&](const detail::Json& j, long line_no) {
    Recording r;
    r.id = j.at("id").as_string();
    r.sample_rate = static_cast<int>(j.at("sample_rate").as_number());
    r.duration = j.at("duration").as_number();
    for (const auto& s : j.at("sources").as_array()) {
      Source src;
      src.path = s.at("path").as_string();
      for (const auto& c : s.at("channels").as_array()) src.channels.push_back(static_cast<int>(c.as_number()));
      r.sources.push_back(std::move(src));
    }
    const std::string where = detail::loc(path, line_no);
    if (!seen.insert(r.id).second) throw ParseError(where + "duplicate recording id '" + r.id + "'");
    if (r.duration <= 0.0) throw ParseError(where + "recording '" + r.id + "' has a non-positive duration");
    if (r.sample_rate <= 0) throw ParseError(where + "recording '" + r.id + "' has a non-positive sample_rate");
    for (const auto& src : r.sources) {
      std::set<int> uniq(src.channels.begin(), src.channels.end());
      if (uniq.size() != src.channels.size())
        throw ParseError(where + "recording '" + r.id + "' repeats a channel index");
    }
    if (r.channel_count() < 1) throw ParseError(where + "recording '" + r.id + "' has no channels");
    out.push_back(std::move(r));
  });
  return out;
}

inline std::string serialize_recordings(const std::vector<Recording>& recs) {
  std::string out;
  for (const auto& r : recs) {
    out += "{\"id\":" + detail::json_escape(r.id) + ",\"sources\":[";
    for (size_t i = 0; i < r.sources.size(); ++i) {
      out += std::string(i ? "," : "") + "{\"path\":" + detail::json_escape(r.sources[i].path) + ",\"channels\":[";
      for (size_t c = 0; c < r.sources[i].channels.size(); ++c)
        out += (c ? "," : "") + std::to_string(r.sources[i].channels[c]);
      out += "]}";
    }
    out += "],\"sample_rate\":" + std::to_string(r.sample_rate) + ",\"duration\":" + detail::json_number(r.duration) +
           "}\n";
  }
  return out;
}

inline void save_recordings(const std::string& path, const std::vector<Recording>& recs) {
  write_text(path, serialize_recordings(recs));
}

// ---------------------------------------------------------------------------
// segment manifests: JSONL and RTTM (manifests.hpp:222-331)
// ---------------------------------------------------------------------------
inline std::string serialize_segments(const std::vector<Segment>& segs) {
  std::string out;
  for (const auto& s : segs)
    out += "{\"id\":" + detail::json_escape(s.id) + ",\"recording_id\":" + detail::json_escape(s.recording_id) +
           ",\"speaker\":" + detail::json_escape(s.speaker) + ",\"start\":" + detail::json_number(s.start) +
           ",\"duration\":" + detail::json_number(s.duration) + "}\n";
  return out;
}

inline void save_segments(const std::string& path, const std::vector<Segment>& segs) {
  write_text(path, serialize_segments(segs));
}

/// Segments of a JSONL or RTTM manifest; entries with duration <= 0 are dropped and counted in *skipped.
inline std::vector<Segment> load_segments(const std::string& path, SegmentFormat format = SegmentFormat::kJsonl,
                                          int* skipped = nullptr) {
  if (skipped) *skipped = 0;
  std::vector<Segment> out;
  if (format == SegmentFormat::kJsonl) {
    detail::for_each_jsonl(path, [&](const detail::Json& j, long) {
      Segment s;
      s.id = j.at("id").as_string();
      s.recording_id = j.at("recording_id").as_string();
      s.speaker = j.at("speaker").as_string();
      s.start = j.at("start").as_number();
      s.duration = j.at("duration").as_number();
      if (s.duration <= 0.0) {  // the reference warns and drops the entry
        if (skipped) ++*skipped;
        return;
      }
      out.push_back(std::move(s));
    });
    return out;
  }
  std::istringstream in(read_text(path));
  std::string line;
  long line_no = 0;
  std::map<std::pair<std::string, std::string>, int> counters;
  while (std::getline(in, line)) {
    ++line_no;
    std::istringstream ls(line);
    std::vector<std::string> fields;
    for (std::string tok; ls >> tok;) fields.push_back(tok);
    if (fields.empty() || fields[0] != "SPEAKER") continue;  // other record types are legal
    if (fields.size() < 9)
      throw ParseError(detail::loc(path, line_no) + "RTTM SPEAKER line has " + std::to_string(fields.size()) +
                       " fields, need 9+");
    Segment s;
    s.recording_id = fields[1];
    s.speaker = fields[7];
    try {
      size_t used = 0;
      s.start = std::stod(fields[3], &used);
      if (used != fields[3].size()) throw std::invalid_argument(fields[3]);
      s.duration = std::stod(fields[4], &used);
      if (used != fields[4].size()) throw std::invalid_argument(fields[4]);
    } catch (const std::exception&) {
      throw ParseError(detail::loc(path, line_no) + "RTTM line has non-numeric start/duration");
    }
    if (s.duration <= 0.0) {
      if (skipped) ++*skipped;
      continue;
    }
    const int n = counters[{s.recording_id, s.speaker}]++;
    char idx[16];
    std::snprintf(idx, sizeof idx, "%04d", n);
    s.id = s.recording_id + "-" + s.speaker + "-" + idx;
    out.push_back(std::move(s));
  }
  return out;
}

/// Cross-manifest validation; human-readable problems (empty = OK), manifests.hpp:334-361.
inline std::vector<std::string> validate(const std::vector<Recording>& recordings, const std::vector<Segment>& segments) {
  std::vector<std::string> problems;
  std::map<std::string, const Recording*> by_id;
  for (const auto& r : recordings) by_id[r.id] = &r;
  std::set<std::string> seg_ids;
  for (const auto& s : segments) {
    if (!seg_ids.insert(s.id).second) problems.push_back("duplicate segment id '" + s.id + "'");
    const auto it = by_id.find(s.recording_id);
    if (it == by_id.end()) {
      problems.push_back("segment '" + s.id + "' references unknown recording '" + s.recording_id + "'");
      continue;
    }
    if (s.start < 0.0) problems.push_back("segment '" + s.id + "' starts at " + detail::json_number(s.start));
    if (s.end() > it->second->duration + 1e-6)
      problems.push_back("segment '" + s.id + "' ends at " + detail::json_number(s.end()) + ", past recording end " +
                         detail::json_number(it->second->duration));
  }
  return problems;
}

/// [start_sample, start_sample + count) across all sources of a recording, channels stacked in source order;
/// channel_subset selects stacked indices (empty = all). manifests.hpp:442-479.
inline stft::RealSignal load_audio(const Recording& rec, int64_t start_sample, int64_t count,
                                   const std::vector<int>& channel_subset = {}) {
  stft::RealSignal all;
  all.sample_rate = rec.sample_rate;
  for (const auto& src : rec.sources) {
    stft::RealSignal part = wav::read(src.path, start_sample, count);
    if (part.sample_rate != rec.sample_rate)
      throw ConfigError("recording '" + rec.id + "': " + src.path + " is " + std::to_string(part.sample_rate) +
                        " Hz, manifest says " + std::to_string(rec.sample_rate));
    if (part.num_samples() < count)
      throw IoError("recording '" + rec.id + "': " + src.path + " has " + std::to_string(part.num_samples()) +
                    " samples at offset " + std::to_string(start_sample) + ", need " + std::to_string(count));
    for (const int c : src.channels) {
      if (c < 0 || c >= part.num_channels())
        throw ConfigError("recording '" + rec.id + "': " + src.path + " has no channel " + std::to_string(c));
      all.channels.push_back(std::move(part.channels[c]));
    }
  }
  if (channel_subset.empty()) return all;
  stft::RealSignal out;
  out.sample_rate = all.sample_rate;
  for (const int c : channel_subset) {
    if (c < 0 || c >= all.num_channels())
      throw ConfigError("channel subset index " + std::to_string(c) + " out of range [0, " +
                        std::to_string(all.num_channels()) + ")");
    out.channels.push_back(all.channels[c]);
  }
  return out;
}

}  // namespace gss::manifests
