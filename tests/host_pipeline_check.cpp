// host_pipeline_check.cpp -- the pipeline rows of the C++ host mirror (gss/wav.hpp, gss/manifests.hpp loaders,
// gss/scheduler.hpp plan_batches / assemble / run_pipeline), written like the reference's own tests (cited
// inline). `cpu <golden dir> <tmp dir>` runs the file-format and planning checks without a device;
// `gpu <tmp dir>` writes a small recording, runs the pipeline on device 0 under several executors and leaves
// the inputs and outputs behind so that the Python mirror can be run on the same files.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <random>
#include <sstream>

#include "gss/scheduler.hpp"

using namespace gss;
namespace mf = gss::manifests;
namespace sc = gss::scheduler;

static int g_checks = 0;
#define CHECK(cond)                                                \
  do {                                                             \
    ++g_checks;                                                    \
    if (!(cond)) {                                                 \
      std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond); \
      return 1;                                                    \
    }                                                              \
  } while (0)
#define CHECK_THROWS(expr, Exc)                                                   \
  do {                                                                            \
    ++g_checks;                                                                   \
    bool caught = false;                                                          \
    try {                                                                         \
      (void)(expr);                                                               \
    } catch (const Exc&) {                                                        \
      caught = true;                                                              \
    } catch (const std::exception& e) {                                           \
      std::printf("FAIL %s:%d: %s threw %s\n", __FILE__, __LINE__, #expr, e.what()); \
      return 1;                                                                   \
    }                                                                             \
    if (!caught) {                                                                \
      std::printf("FAIL %s:%d: %s did not throw\n", __FILE__, __LINE__, #expr);  \
      return 1;                                                                   \
    }                                                                             \
  } while (0)

static std::string slurp(const std::string& path) {
  std::ifstream in(path, std::ios::binary);
  std::ostringstream os;
  os << in.rdbuf();
  return os.str();
}

static stft::RealSignal noise_signal(int channels, int64_t samples, unsigned seed) {
  std::mt19937 rng(seed);
  std::normal_distribution<float> gauss(0.f, 0.1f);
  stft::RealSignal sig;
  sig.sample_rate = 16000;
  sig.channels.assign(channels, std::vector<float>((size_t)samples));
  for (auto& ch : sig.channels)
    for (auto& v : ch) v = gauss(rng);
  return sig;
}

static mf::Segment seg(const std::string& rec, const std::string& spk, double start, double dur, const std::string& id) {
  mf::Segment s;
  s.recording_id = rec;
  s.speaker = spk;
  s.start = start;
  s.duration = dur;
  s.id = id;
  return s;
}

static int cpu_checks(const std::string& data, const std::string& tmp) {
  // --- wav (test_wav.cpp:33-116) ---
  {
    stft::RealSignal sig = noise_signal(3, 4000, 1);
    wav::write(tmp + "/a.wav", sig);
    const wav::WavInfo wi = wav::info(tmp + "/a.wav");
    CHECK(wi.channels == 3 && wi.sample_rate == 16000 && wi.bits_per_sample == 32 && wi.format == 3 &&
          wi.num_frames == 4000);
    stft::RealSignal back = wav::read(tmp + "/a.wav");
    CHECK(back.channels == sig.channels);  // float32 round trip is exact
    stft::RealSignal win = wav::read(tmp + "/a.wav", 1000, 500);
    CHECK(win.num_samples() == 500 && win.channels[2][0] == sig.channels[2][1000]);
    CHECK(wav::read(tmp + "/a.wav", 3900, 500).num_samples() == 100);  // clipped at the end of the file
    CHECK(wav::read(tmp + "/a.wav", 4000, 10).num_samples() == 0);
    CHECK_THROWS(wav::read(tmp + "/a.wav", 4001, 10), IoError);
    CHECK_THROWS(wav::info(tmp + "/missing.wav"), IoError);
    std::ofstream(tmp + "/junk.wav") << "this is not a wav file at all";
    CHECK_THROWS(wav::info(tmp + "/junk.wav"), ParseError);
    // PCM16 with an odd-sized unknown chunk before fmt
    std::string h("RIFF");
    wav::detail::put32(h, 0);
    h += "WAVEjunk";
    wav::detail::put32(h, 3);
    h += "abc";
    h.push_back('\0');
    h += "fmt ";
    wav::detail::put32(h, 16);
    wav::detail::put16(h, 1);
    wav::detail::put16(h, 2);
    wav::detail::put32(h, 8000);
    wav::detail::put32(h, 8000 * 4);
    wav::detail::put16(h, 4);
    wav::detail::put16(h, 16);
    h += "data";
    wav::detail::put32(h, 8);
    const int16_t pcm[4] = {16384, -16384, 32767, -32768};
    h.append(reinterpret_cast<const char*>(pcm), 8);
    std::ofstream(tmp + "/pcm16.wav", std::ios::binary) << h;
    stft::RealSignal p16 = wav::read(tmp + "/pcm16.wav");
    CHECK(p16.num_channels() == 2 && p16.num_samples() == 2 && p16.sample_rate == 8000);
    CHECK(p16.channels[0][0] == 0.5f && p16.channels[1][0] == -0.5f && p16.channels[1][1] == -1.0f);
  }
  // --- manifests (test_manifests.cpp:22-199) ---
  {
    auto recs = mf::load_recordings(data + "/recordings_golden.jsonl");
    CHECK(recs.size() == 2 && recs[0].id == "meet01" && recs[0].sources.size() == 2);
    CHECK(recs[0].sources[0].channels == std::vector<int>({0, 1}) && recs[0].channel_count() == 3);
    CHECK(recs[0].sample_rate == 16000 && recs[0].duration == 120.5 && recs[0].num_samples() == 1928000);
    CHECK(recs[1].channel_count() == 4);
    mf::save_recordings(tmp + "/recordings_echo.jsonl", recs);
    auto again = mf::load_recordings(tmp + "/recordings_echo.jsonl");
    CHECK(again.size() == 2 && again[0].sources[1].path == recs[0].sources[1].path &&
          again[1].duration == recs[1].duration);
    const std::string text = slurp(tmp + "/recordings_echo.jsonl");
    CHECK(text.substr(0, text.find('\n')) ==
          "{\"id\":\"meet01\",\"sources\":[{\"path\":\"audio/meet01_a.wav\",\"channels\":[0,1]},"
          "{\"path\":\"audio/meet01_b.wav\",\"channels\":[0]}],\"sample_rate\":16000,\"duration\":120.5}");
    CHECK_THROWS(mf::load_recordings(data + "/recordings_dup.jsonl"), ParseError);
    CHECK_THROWS(mf::load_recordings(data + "/missing.jsonl"), IoError);
    bool located = false;
    try {
      mf::load_recordings(data + "/segments_broken.jsonl");
    } catch (const ParseError& e) {
      located = std::string(e.what()).find("segments_broken.jsonl:1") != std::string::npos;
    }
    CHECK(located);

    int skipped = -1;
    auto segs = mf::load_segments(data + "/segments_golden.jsonl", mf::SegmentFormat::kJsonl, &skipped);
    CHECK(segs.size() == 4 && skipped == 0);
    CHECK(segs[0].id == "meet01-alice-0000" && segs[0].recording_id == "meet01" && segs[0].speaker == "alice" &&
          segs[0].start == 1.5 && segs[0].duration == 4.25 && segs[0].end() == 5.75 && segs[3].speaker == "carol");
    segs = mf::load_segments(data + "/segments_zero_duration.jsonl", mf::SegmentFormat::kJsonl, &skipped);
    CHECK(segs.size() == 2 && skipped == 2 && segs[1].id == "meet01-bob-0001");
    auto rttm = mf::load_segments(data + "/segments_golden.rttm", mf::SegmentFormat::kRttm, &skipped);
    CHECK(rttm.size() == 4 && skipped == 1);
    CHECK(rttm[0].id == "meet01-alice-0000" && rttm[1].id == "meet01-bob-0000" && rttm[2].id == "meet01-alice-0001" &&
          rttm[3].id == "meet02-carol-0000");
    auto golden = mf::load_segments(data + "/segments_golden.jsonl");
    for (size_t i = 0; i < 4; ++i)
      CHECK(rttm[i].start == golden[i].start && rttm[i].duration == golden[i].duration &&
            rttm[i].speaker == golden[i].speaker);
    CHECK_THROWS(mf::load_segments(data + "/segments_malformed.rttm", mf::SegmentFormat::kRttm), ParseError);
    CHECK_THROWS(mf::load_segments(data + "/segments_badnum.rttm", mf::SegmentFormat::kRttm), ParseError);
    mf::save_segments(tmp + "/segments_echo.jsonl", golden);
    auto echo = mf::load_segments(tmp + "/segments_echo.jsonl");
    CHECK(echo.size() == 4 && echo[2].id == golden[2].id && echo[2].start == golden[2].start);
#ifdef GSS_WITH_ZLIB
    mf::save_segments(tmp + "/segments_echo.jsonl.gz", golden);
    auto gz = mf::load_segments(tmp + "/segments_echo.jsonl.gz");
    CHECK(gz.size() == 4 && gz[3].duration == golden[3].duration);
    CHECK(mf::read_text(tmp + "/segments_echo.jsonl.gz") == mf::serialize_segments(golden));
#endif
    // validate (test_manifests.cpp:160-199)
    CHECK(mf::validate(recs, golden).empty());
    auto bad = golden;
    bad[0].recording_id = "nope";
    bad[1].start = 120.0;
    bad[1].duration = 5.0;
    bad[2].id = bad[3].id;
    CHECK(mf::validate(recs, bad).size() == 3);
  }
  // --- load_audio stacks sources in channel order (test_manifests.cpp:205-240) ---
  {
    stft::RealSignal a = noise_signal(2, 3000, 5), b = noise_signal(1, 3000, 6);
    wav::write(tmp + "/src_a.wav", a);
    wav::write(tmp + "/src_b.wav", b);
    mf::Recording rec;
    rec.id = "r";
    rec.sample_rate = 16000;
    rec.duration = 3000.0 / 16000;
    rec.sources = {mf::Source{tmp + "/src_a.wav", {0, 1}}, mf::Source{tmp + "/src_b.wav", {0}}};
    stft::RealSignal x = mf::load_audio(rec, 100, 400);
    CHECK(x.num_channels() == 3 && x.num_samples() == 400);
    CHECK(x.channels[0][0] == a.channels[0][100] && x.channels[1][399] == a.channels[1][499] &&
          x.channels[2][7] == b.channels[0][107]);
    stft::RealSignal sel = mf::load_audio(rec, 0, 10, {2, 0});
    CHECK(sel.num_channels() == 2 && sel.channels[0][3] == b.channels[0][3] && sel.channels[1][3] == a.channels[0][3]);
    CHECK_THROWS(mf::load_audio(rec, 0, 10, {3}), ConfigError);
  }
  // --- plan_batches (test_scheduler.cpp:61-127) ---
  {
    std::vector<mf::Segment> segs;
    for (int i = 0; i < 6; ++i) segs.push_back(seg("r0", "a", 10.0 * i, 4.0, "a" + std::to_string(i)));
    for (int i = 0; i < 3; ++i) segs.push_back(seg("r0", "b", 5.0 + 10.0 * i, 4.0, "b" + std::to_string(i)));
    segs.push_back(seg("r0", "a", 70.0, 30.0, "along"));
    auto plans = sc::plan_batches(segs, 10.0);
    // a: [a0 a1] [a2 a3] [a4 a5] [along]; b: [b0 b1] [b2]; emitted round-robin a, b, a, b, a, a
    CHECK(plans.size() == 6);
    CHECK(plans[0].speaker == "a" && plans[0].parts.size() == 2 && plans[1].speaker == "b" &&
          plans[1].parts.size() == 2);
    CHECK(plans[2].speaker == "a" && plans[3].speaker == "b" && plans[3].parts.size() == 1);
    CHECK(plans[5].parts.size() == 1 && plans[5].parts[0].id == "along" && plans[5].total_duration() == 30.0);
    size_t covered = 0;
    for (const auto& p : plans) {
      covered += p.parts.size();
      CHECK(p.parts.size() == 1 || p.total_duration() <= 10.0);
      for (size_t i = 1; i < p.parts.size(); ++i) CHECK(p.parts[i - 1].start <= p.parts[i].start);
    }
    CHECK(covered == segs.size());
    CHECK(sc::plan_batches(segs, 10.0, sc::BatchMode::kOnePerBatch).size() == segs.size());
    CHECK(sc::plan_batches({}, 10.0).empty());
  }
  // --- assemble (test_scheduler.cpp:133-212): spans, offsets, context clipping, activity ---
  {
    stft::RealSignal sig = noise_signal(2, 16000 * 12, 11);
    wav::write(tmp + "/asm.wav", sig);
    mf::Recording rec;
    rec.id = "r0";
    rec.sample_rate = 16000;
    rec.duration = 12.0;
    rec.sources = {mf::Source{tmp + "/asm.wav", {0, 1}}};
    std::vector<mf::Segment> all = {seg("r0", "a", 1.0, 2.0, "a0"), seg("r0", "a", 5.0, 1.5, "a1"),
                                    seg("r0", "b", 2.5, 3.0, "b0")};
    sc::PipelineConfig cfg;
    cfg.context_duration = 2.0;
    sc::BatchPlan plan{"r0", "a", {all[0], all[1]}};
    sc::SuperSegment ss = sc::assemble(plan, rec, all, cfg);
    CHECK(ss.context_left == 1.0 && ss.context_right == 2.0);  // the left context is clipped by the file start
    CHECK(ss.audio.num_channels() == 2 && ss.audio.num_samples() == 16000 * (1 + 2 + 1.5 + 2));
    CHECK(ss.parts.size() == 2 && ss.parts[0].sample_begin == 16000 && ss.parts[0].sample_end == 48000 &&
          ss.parts[1].sample_begin == 48000 && ss.parts[1].sample_end == 72000);
    CHECK(ss.audio.channels[1][0] == sig.channels[1][0] && ss.audio.channels[0][48000] == sig.channels[0][80000]);
    CHECK((int64_t)ss.frame_centers.size() == stft::frame_count(ss.audio.num_samples(), cfg.stft));
    CHECK(ss.activity.frames == (int64_t)ss.frame_centers.size() && ss.activity.num_classes() == 3);
    CHECK(ss.activity.classes[0] == "a" && ss.activity.classes[1] == "b" && ss.activity.classes[2] == "noise");
    for (int64_t t = 0; t < ss.activity.frames; ++t) {
      const double sec = (double)ss.frame_centers[t] / 16000;
      const bool in_a = (sec >= 1.0 && sec < 3.0) || (sec >= 5.0 && sec < 6.5);
      const bool in_b = sec >= 2.5 && sec < 5.5;
      if (ss.frame_centers[t] >= 0) CHECK(ss.activity.at(t, 0) == in_a && ss.activity.at(t, 1) == in_b);
      CHECK(ss.activity.at(t, 2) == 1);
    }
    cfg.noise_class = false;
    CHECK(sc::assemble(plan, rec, all, cfg).activity.num_classes() == 2);
    sc::BatchPlan off_end{"r0", "a", {seg("r0", "a", 12.5, 1.0, "late")}};
    CHECK_THROWS(sc::assemble(off_end, rec, all, cfg), ShapeError);
  }
  // --- config echo / validate (test_scheduler.cpp:42-55) ---
  {
    sc::PipelineConfig cfg;
    cfg.out_dir = "some \"dir\"";
    const std::string e = cfg.echo();
    CHECK(e.find("\"max-batch-duration\": 50") != std::string::npos && e.find("\"bss-iterations\": 20") != std::string::npos);
    CHECK(e.find("\"out-dir\": \"some \\\"dir\\\"\"") != std::string::npos);
    cfg.queue_capacity = 0;
    CHECK_THROWS(cfg.validate(), ConfigError);
  }
  // --- OrderedBatchQueue hands items over in plan order (test_scheduler.cpp:218-254) ---
  {
    sc::detail::OrderedBatchQueue q(3);
    std::vector<std::thread> producers;
    for (int w = 0; w < 3; ++w)
      producers.emplace_back([&q, w] {
        for (int64_t i = w; i < 30; i += 3) {
          sc::detail::LoadedBatch item;
          item.index = i;
          std::this_thread::sleep_for(std::chrono::microseconds(((i * 7919) % 13) * 50));
          q.put(std::move(item));
        }
      });
    bool ordered = true;
    for (int64_t i = 0; i < 30; ++i) ordered = ordered && q.take().index == i;
    for (auto& t : producers) t.join();
    CHECK(ordered);
  }
  std::printf("OK %d checks\n", g_checks);
  return 0;
}

// Two talkers with distinct inter-channel delays over diffuse noise: enough structure for the separation to
// be well posed; parity of the written waveforms is checked by the caller against the Python mirror.
static stft::RealSignal meeting(int channels, double seconds, const std::vector<std::array<double, 3>>& talk) {
  stft::RealSignal sig = noise_signal(channels, (int64_t)(seconds * 16000), 21);
  for (auto& ch : sig.channels)
    for (auto& v : ch) v *= 0.1f;
  std::mt19937 rng(22);
  std::normal_distribution<float> gauss(0.f, 0.3f);
  for (const auto& t : talk) {
    const int spk = (int)t[0];
    const int64_t b = (int64_t)(t[1] * 16000), e = (int64_t)((t[1] + t[2]) * 16000);
    std::vector<float> src((size_t)(e - b));
    float lp = 0;
    for (auto& v : src) v = lp = 0.7f * lp + gauss(rng);
    for (int c = 0; c < channels; ++c) {
      const int delay = (spk == 0 ? c : (channels - 1 - c)) * 2;
      for (int64_t i = 0; i + delay < e - b; ++i)
        sig.channels[c][(size_t)(b + i + delay)] += src[(size_t)i] * (1.0f - 0.1f * (float)c * (spk ? 1 : -1) / channels);
    }
  }
  return sig;
}

static int gpu_checks(const std::string& tmp) {
  const std::string in_dir = tmp + "/in";
  std::filesystem::create_directories(in_dir);
  stft::RealSignal sig = meeting(3, 14.0, {{0, 0.5, 2.5}, {1, 3.5, 2.0}, {0, 6.0, 2.0}, {1, 8.5, 3.0}, {0, 11.0, 2.0}});
  wav::write(in_dir + "/m0.wav", sig);
  mf::Recording rec;
  rec.id = "m0";
  rec.sample_rate = 16000;
  rec.duration = 14.0;
  rec.sources = {mf::Source{in_dir + "/m0.wav", {0, 1, 2}}};
  std::vector<mf::Segment> segs = {seg("m0", "s0", 0.5, 2.5, "m0-s0-0000"), seg("m0", "s1", 3.5, 2.0, "m0-s1-0000"),
                                   seg("m0", "s0", 6.0, 2.0, "m0-s0-0001"), seg("m0", "s1", 8.5, 3.0, "m0-s1-0001"),
                                   seg("m0", "s0", 11.0, 2.0, "m0-s0-0002")};
  mf::save_recordings(in_dir + "/recordings.jsonl", {rec});
  mf::save_segments(in_dir + "/segments.jsonl", segs);

  auto config = [&](const std::string& out, int workers) {
    sc::PipelineConfig cfg;
    cfg.max_batch_duration = 5.0;
    cfg.context_duration = 1.0;
    cfg.bss_iterations = 3;
    cfg.wpe.taps = 4;
    cfg.wpe.delay = 2;
    cfg.wpe.iterations = 1;
    cfg.out_dir = out;
    cfg.workers = workers;
    return cfg;
  };
  // test_scheduler.cpp:278-330: outputs, summary counts, naming
  sc::RunSummary base = sc::run_pipeline({rec}, segs, config(tmp + "/out_sync", 0));
  for (const auto& f : base.failures) std::printf("failure %s: %s\n", f.segment_id.c_str(), f.error.c_str());
  // s0: [2.5 + 2.0] [2.0]; s1: [2.0 + 3.0] -> 3 batches under the 5 s cap
  CHECK(base.failed_segments == 0 && base.segments_written == 5 && base.num_batches == 3);
  CHECK(base.outputs.size() == 5 && base.batches.size() == 3 && base.failures.empty());
  CHECK(std::filesystem::exists(tmp + "/out_sync/m0-s0-0000500_0003000.wav"));
  CHECK(std::filesystem::exists(tmp + "/out_sync/summary.json") && slurp(tmp + "/out_sync/summary.json") == base.json);
  for (const auto& o : base.outputs) CHECK(wav::info(o.path).num_frames == o.samples && wav::info(o.path).channels == 1);
  CHECK(base.outputs[0].samples == 40000);
  {
    mf::detail::JsonReader reader(base.json);  // the summary is well-formed JSON with the reference's keys
    const mf::detail::Json j = reader.parse();
    CHECK(j.at("num_segments").as_number() == 5 && j.at("segments_written").as_number() == 5);
    CHECK(j.at("config").at("bss-iterations").as_number() == 3 && j.at("stage_seconds").at("total").as_number() > 0);
    CHECK(j.at("batches").as_array().size() == 3 && j.at("outputs").as_array().size() == 5);
  }
  double energy = 0;
  const stft::RealSignal enhanced = wav::read(base.outputs[3].path);
  for (float v : enhanced.channels[0]) energy += (double)v * v;
  CHECK(energy > 1.0 && std::isfinite(energy));

  // test_scheduler.cpp:336-372: bytes do not depend on the worker count, the queue depth or the device batch
  struct Variant {
    const char* name;
    int workers, capacity, gpu_batch;
  };
  for (const Variant& v : {Variant{"out_w2", 2, 2, 16}, Variant{"out_w4_b1", 4, 1, 1}, Variant{"out_w1_b3", 1, 3, 3}}) {
    sc::PipelineConfig cfg = config(tmp + "/" + v.name, v.workers);
    cfg.queue_capacity = v.capacity;
    sc::RunSummary run = sc::run_pipeline({rec}, segs, cfg, {0}, v.gpu_batch);
    CHECK(run.failed_segments == 0 && run.outputs.size() == base.outputs.size());
    for (size_t i = 0; i < run.outputs.size(); ++i) {
      CHECK(run.outputs[i].segment_id == base.outputs[i].segment_id);
      CHECK(slurp(run.outputs[i].path) == slurp(base.outputs[i].path));
    }
    for (size_t i = 0; i < run.batches.size(); ++i)
      CHECK(run.batches[i].log_likelihood == base.batches[i].log_likelihood && run.batches[i].frames == base.batches[i].frames);
  }

  // test_scheduler.cpp:378-407: a recording whose audio is missing fails its own segments only
  {
    mf::Recording ghost = rec;
    ghost.id = "ghost";
    ghost.sources = {mf::Source{in_dir + "/ghost.wav", {0, 1, 2}}};
    std::vector<mf::Segment> mixed = segs;
    mixed.push_back(seg("ghost", "s0", 1.0, 2.0, "ghost-s0-0000"));
    sc::RunSummary run = sc::run_pipeline({rec, ghost}, mixed, config(tmp + "/out_ghost", 2));
    CHECK(run.failed_segments == 1 && run.segments_written == 5 && run.failures.size() == 1);
    CHECK(run.failures[0].segment_id == "ghost-s0-0000" && run.failures[0].error.find("ghost.wav") != std::string::npos);
    for (size_t i = 0; i < base.outputs.size(); ++i) {
      const std::string name = std::filesystem::path(base.outputs[i].path).filename().string();
      CHECK(slurp(tmp + "/out_ghost/" + name) == slurp(base.outputs[i].path));
    }
    // an invalid manifest is a configuration error before any work starts
    mixed.back().recording_id = "nowhere";
    CHECK_THROWS(sc::run_pipeline({rec, ghost}, mixed, config(tmp + "/out_bad", 0)), ConfigError);
  }
  std::printf("OK %d checks\n", g_checks);
  return 0;
}

int main(int argc, char** argv) {
  std::setvbuf(stdout, nullptr, _IONBF, 0);  // nothing is lost if a check crashes
  try {
    if (argc == 4 && std::string(argv[1]) == "cpu") return cpu_checks(argv[2], argv[3]);
    if (argc == 3 && std::string(argv[1]) == "gpu") return gpu_checks(argv[2]);
  } catch (const std::exception& e) {
    std::printf("FAIL uncaught: %s\n", e.what());
    return 1;
  }
  std::printf("usage: host_pipeline_check cpu <golden dir> <tmp dir> | gpu <tmp dir>\n");
  return 2;
}
