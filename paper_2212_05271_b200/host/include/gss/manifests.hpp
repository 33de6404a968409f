// gss/manifests.hpp (B200 build) -- the reference's manifests.hpp: Recording / Segment manifests (JSONL,
// gzip-transparent when built with GSS_WITH_ZLIB; RTTM), cross-manifest validation, the activity guide
// (build_activity_at / build_activity: bit-exact integer work in the library's host code) and multi-source
// audio loading. The reference parses JSON with nlohmann::json; this build carries a small reader for the
// flat objects the manifests use (gss::manifests::detail::Json).
#pragma once

#include <algorithm>
#include <cctype>
#include <cerrno>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <map>
#include <memory>
#include <set>
#include <sstream>
#include <string>
#include <unordered_map>
#include <unordered_set>
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
// Text files. A name ending in ".gz" goes through zlib (when built with -DGSS_WITH_ZLIB), anything else through
// stdio; callers never see the difference (the reference's read_text / write_text contract, manifests.hpp:79-114).
// ---------------------------------------------------------------------------
inline bool has_suffix(const std::string& s, const std::string& suffix) {
  const size_t n = suffix.size();
  return s.size() >= n && std::equal(suffix.begin(), suffix.end(), s.end() - static_cast<std::ptrdiff_t>(n));
}

namespace textio {

constexpr size_t kBlock = 1u << 16;

#ifdef GSS_WITH_ZLIB
struct GzClose {
  void operator()(gzFile_s* g) const {
    if (g) gzclose(g);
  }
};
using Gz = std::unique_ptr<gzFile_s, GzClose>;
#endif

struct FileClose {
  void operator()(std::FILE* f) const {
    if (f) std::fclose(f);
  }
};
using Plain = std::unique_ptr<std::FILE, FileClose>;

}  // namespace textio

inline std::string read_text(const std::string& path) {
  std::string text;
  std::vector<char> block(textio::kBlock);
  if (!has_suffix(path, ".gz")) {
    textio::Plain f(std::fopen(path.c_str(), "rb"));
    if (!f) throw IoError("cannot open file: " + path);
    for (size_t got; (got = std::fread(block.data(), 1, block.size(), f.get())) > 0;) text.append(block.data(), got);
    if (std::ferror(f.get())) throw IoError("read failed: " + path);
    return text;
  }
#ifdef GSS_WITH_ZLIB
  textio::Gz g(gzopen(path.c_str(), "rb"));
  if (!g) throw IoError("cannot open file: " + path);
  int got = 0;
  while ((got = gzread(g.get(), block.data(), static_cast<unsigned>(block.size()))) > 0)
    text.append(block.data(), static_cast<size_t>(got));
  if (got < 0) throw IoError("gzip stream is damaged: " + path);
  return text;
#else
  throw IoError("this build has no zlib (GSS_WITH_ZLIB), cannot read " + path);
#endif
}

inline void write_text(const std::string& path, const std::string& content) {
  if (!has_suffix(path, ".gz")) {
    textio::Plain f(std::fopen(path.c_str(), "wb"));
    if (!f) throw IoError("cannot create file: " + path);
    const bool ok = std::fwrite(content.data(), 1, content.size(), f.get()) == content.size();
    if (!ok || std::fflush(f.get()) != 0) throw IoError("write failed: " + path);
    return;
  }
#ifdef GSS_WITH_ZLIB
  textio::Gz g(gzopen(path.c_str(), "wb"));
  if (!g) throw IoError("cannot create file: " + path);
  for (size_t at = 0; at < content.size();) {
    const unsigned want = static_cast<unsigned>(std::min(textio::kBlock, content.size() - at));
    if (gzwrite(g.get(), content.data() + at, want) != static_cast<int>(want)) throw IoError("gzip write failed: " + path);
    at += want;
  }
  if (gzclose(g.release()) != Z_OK) throw IoError("gzip write failed: " + path);
#else
  throw IoError("this build has no zlib (GSS_WITH_ZLIB), cannot write " + path);
#endif
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

namespace detail {

/// Whitespace-separated fields of one text line (RTTM is a column format).
inline std::vector<std::string> split_fields(const std::string& line) {
  std::vector<std::string> out;
  size_t i = 0;
  const size_t n = line.size();
  while (i < n) {
    while (i < n && std::isspace(static_cast<unsigned char>(line[i]))) ++i;
    size_t j = i;
    while (j < n && !std::isspace(static_cast<unsigned char>(line[j]))) ++j;
    if (j > i) out.emplace_back(line, i, j - i);
    i = j;
  }
  return out;
}

/// The whole token as a double, or false.
inline bool whole_number(const std::string& tok, double& value) {
  if (tok.empty()) return false;
  char* end = nullptr;
  errno = 0;
  value = std::strtod(tok.c_str(), &end);
  return errno == 0 && end == tok.c_str() + tok.size();
}

/// RTTM: "SPEAKER <recording> <chan> <start> <duration> <NA> <NA> <speaker> <NA> ..." (manifests.hpp:274-318);
/// other record types are skipped, ids are made up as <recording>-<speaker>-<running number per pair>.
inline void parse_rttm(const std::string& path, std::vector<Segment>& out, int& dropped) {
  const std::string text = read_text(path);
  std::map<std::string, int> next_index;  // key: recording + '\n' + speaker
  long line_no = 0;
  for (size_t at = 0; at < text.size();) {
    size_t eol = text.find('\n', at);
    if (eol == std::string::npos) eol = text.size();
    const std::vector<std::string> col = split_fields(text.substr(at, eol - at));
    at = eol + 1;
    ++line_no;
    if (col.empty() || col.front() != "SPEAKER") continue;
    if (col.size() < 9)
      throw ParseError(loc(path, line_no) + "RTTM SPEAKER line has " + std::to_string(col.size()) + " fields, need 9+");
    Segment seg;
    if (!whole_number(col[3], seg.start) || !whole_number(col[4], seg.duration))
      throw ParseError(loc(path, line_no) + "RTTM line has non-numeric start/duration");
    if (!(seg.duration > 0.0)) {
      ++dropped;
      continue;
    }
    seg.recording_id = col[1];
    seg.speaker = col[7];
    int& n = next_index[seg.recording_id + '\n' + seg.speaker];
    std::string number = std::to_string(n++);
    if (number.size() < 4) number.insert(0, 4 - number.size(), '0');
    seg.id = seg.recording_id + "-" + seg.speaker + "-" + number;
    out.push_back(std::move(seg));
  }
}

inline void parse_segment_lines(const std::string& path, std::vector<Segment>& out, int& dropped) {
  for_each_jsonl(path, [&](const Json& j, long) {
    Segment seg;
    seg.id = j.at("id").as_string();
    seg.recording_id = j.at("recording_id").as_string();
    seg.speaker = j.at("speaker").as_string();
    seg.start = j.at("start").as_number();
    seg.duration = j.at("duration").as_number();
    if (seg.duration > 0.0)
      out.push_back(std::move(seg));
    else
      ++dropped;  // the reference warns and drops the entry
  });
}

}  // namespace detail

/// Segments of a JSONL or RTTM manifest; entries with duration <= 0 are dropped and counted in *skipped
/// (manifests.hpp:253-331).
inline std::vector<Segment> load_segments(const std::string& path, SegmentFormat format = SegmentFormat::kJsonl,
                                          int* skipped = nullptr) {
  std::vector<Segment> out;
  int dropped = 0;
  if (format == SegmentFormat::kRttm)
    detail::parse_rttm(path, out, dropped);
  else
    detail::parse_segment_lines(path, out, dropped);
  if (skipped) *skipped = dropped;
  return out;
}

/// Cross-manifest checks, one sentence per finding, empty when the manifests fit (manifests.hpp:334-361): segment
/// ids unique, every segment inside a known recording.
inline std::vector<std::string> validate(const std::vector<Recording>& recordings, const std::vector<Segment>& segments) {
  std::unordered_map<std::string, double> length_of;
  for (const Recording& r : recordings) length_of[r.id] = r.duration;
  std::unordered_set<std::string> seen;
  std::vector<std::string> findings;
  auto say = [&findings](std::string text) { findings.push_back(std::move(text)); };
  const double slack = 1e-6;  // seconds a segment may overhang its recording
  for (const Segment& seg : segments) {
    const std::string who = "segment '" + seg.id + "'";
    if (seen.count(seg.id)) say("duplicate segment id '" + seg.id + "'");
    seen.insert(seg.id);
    const auto rec = length_of.find(seg.recording_id);
    if (rec == length_of.end()) {
      say(who + " references unknown recording '" + seg.recording_id + "'");
    } else {
      if (seg.start < 0.0) say(who + " starts at " + detail::json_number(seg.start));
      if (seg.end() > rec->second + slack)
        say(who + " ends at " + detail::json_number(seg.end()) + ", past recording end " + detail::json_number(rec->second));
    }
  }
  return findings;
}

/// Samples [start_sample, start_sample + count) of a recording whose channels are spread over several files: the
/// stacked channel list is the files' channel lists in manifest order, `channel_subset` picks from that list
/// (empty = everything). Every file is opened once and only the picked channels are kept (manifests.hpp:442-479).
inline stft::RealSignal load_audio(const Recording& rec, int64_t start_sample, int64_t count,
                                   const std::vector<int>& channel_subset = {}) {
  struct Pick {
    size_t source;
    int channel;
  };
  std::vector<Pick> stacked;
  for (size_t i = 0; i < rec.sources.size(); ++i)
    for (const int c : rec.sources[i].channels) stacked.push_back({i, c});
  std::vector<Pick> wanted;
  if (channel_subset.empty()) {
    wanted = stacked;
  } else {
    for (const int k : channel_subset) {
      if (k < 0 || k >= static_cast<int>(stacked.size()))
        throw ConfigError("channel subset index " + std::to_string(k) + " out of range [0, " +
                          std::to_string(stacked.size()) + ")");
      wanted.push_back(stacked[static_cast<size_t>(k)]);
    }
  }
  stft::RealSignal out;
  out.sample_rate = rec.sample_rate;
  out.channels.resize(wanted.size());
  for (size_t i = 0; i < rec.sources.size(); ++i) {
    const Source& src = rec.sources[i];
    const std::string where = "recording '" + rec.id + "': " + src.path;
    stft::RealSignal file = wav::read(src.path, start_sample, count);
    if (file.sample_rate != rec.sample_rate)
      throw ConfigError(where + " is " + std::to_string(file.sample_rate) + " Hz, manifest says " +
                        std::to_string(rec.sample_rate));
    if (file.num_samples() < count)
      throw IoError(where + " has " + std::to_string(file.num_samples()) + " samples at offset " +
                    std::to_string(start_sample) + ", need " + std::to_string(count));
    for (const int c : src.channels)
      if (c < 0 || c >= file.num_channels()) throw ConfigError(where + " has no channel " + std::to_string(c));
    for (size_t k = 0; k < wanted.size(); ++k)
      if (wanted[k].source == i) out.channels[k] = file.channels[static_cast<size_t>(wanted[k].channel)];
  }
  return out;
}

}  // namespace gss::manifests
