// host_api_check.cpp -- compiles against the C++ host mirror (paper_2212_05271_b200/host/include/gss/*.hpp)
// exactly as a caller of the reference's headers would, and runs the stage operators + enhance_batch on the
// device. Checks mirror reference tests (cited inline). Prints "OK <n checks>" or the first failure.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <random>

#include "gss/scheduler.hpp"

using namespace gss;

static int g_checks = 0;
#define CHECK(cond)                                                        \
  do {                                                                     \
    ++g_checks;                                                            \
    if (!(cond)) {                                                         \
      std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond);         \
      return 1;                                                            \
    }                                                                      \
  } while (0)

int main() {
  std::mt19937 rng(7);
  std::normal_distribution<float> gauss(0.f, 0.1f);
  // test_stft.cpp:90-99 geometry, :149-172 round trip
  stft::StftConfig cfg;
  stft::RealSignal sig;
  sig.sample_rate = 16000;
  sig.channels.assign(3, std::vector<float>(20000));
  for (auto& ch : sig.channels)
    for (auto& v : ch) v = gauss(rng);
  stft::SpectrogramTensor sp = stft::analyze(sig, cfg);
  CHECK(sp.num_bins == 513 && sp.origin_samples == -512 && sp.num_frames == stft::frame_count(20000, cfg));
  stft::RealSignal back = stft::synthesize(sp);
  double err = 0;
  for (int m = 0; m < 3; ++m)
    for (size_t i = 0; i < 20000; ++i) err = std::max(err, (double)std::fabs(back.channels[m][i] - sig.channels[m][i]));
  CHECK(err < 2e-6);
  // test_stft.cpp:101-118 error classes
  try {
    stft::RealSignal tiny;
    tiny.channels.assign(1, std::vector<float>(100));
    stft::analyze(tiny, cfg);
    CHECK(false);
  } catch (const InputTooShortError&) {
    ++g_checks;
  }
  // test_wpe.cpp:70-76 pass-through; :163-182 unit norm
  stft::SpectrogramTensor shortspec = stft::SpectrogramTensor::zeros(cfg, 8, 2);
  for (auto& v : shortspec.data) v = cfloat(gauss(rng), gauss(rng));
  stft::SpectrogramTensor same = wpe::dereverberate(shortspec, wpe::WpeConfig{});
  CHECK(std::memcmp(same.data.data(), shortspec.data.data(), same.data.size() * sizeof(cfloat)) == 0);
  stft::SpectrogramTensor un = wpe::unit_normalize(sp);
  double nrm = 0;
  for (int m = 0; m < 3; ++m) nrm += std::norm(un.at(10, 5, m));
  CHECK(std::fabs(std::sqrt(nrm) - 1.0) < 1e-5);
  // cACGMM: inactive posteriors exactly zero, rows sum to one, LL non-decreasing (test_cacgmm.cpp:224-301)
  manifests::ActivityMatrix act;
  act.frames = un.num_frames;
  act.classes = {"a", "b", "noise"};
  act.target_index = 0;
  act.noise_index = 2;
  act.grid.assign(act.frames * 3, 1);
  for (int64_t t = 0; t < act.frames / 2; ++t) act.set(t, 1, 0);
  cacgmm::EmResult em = cacgmm::em_fit(un, act, 5);
  CHECK(em.likelihood_trace.size() == 6);
  for (size_t i = 1; i < em.likelihood_trace.size(); ++i)
    CHECK(em.likelihood_trace[i] >= em.likelihood_trace[i - 1] - 1e-5 * std::fabs(em.likelihood_trace[i - 1]));
  CHECK(em.posteriors.at(3, 0, 1) == 0.0f);
  const float rs = em.posteriors.at(3, act.frames - 1, 0) + em.posteriors.at(3, act.frames - 1, 1) +
                   em.posteriors.at(3, act.frames - 1, 2);
  CHECK(std::fabs(rs - 1.0f) < 1e-5f);
  const double ll = cacgmm::log_likelihood(un, em.state, act);
  CHECK(std::fabs(ll - em.likelihood_trace.back()) <= 1e-6 * std::fabs(ll));
  // beamformer chain (test_beamform.cpp:211-237 apply = h^H y)
  beamform::BeamformerStats st = beamform::accumulate_stats(sp, em.posteriors, 0);
  const int ref = beamform::select_reference(st);
  beamform::BeamformerFilter flt = beamform::mvdr(st, ref);
  stft::SpectrogramTensor out = beamform::apply(flt, sp);
  cfloat want = 0;
  for (int m = 0; m < 3; ++m) want += sp.at(7, 9, m) * std::conj(static_cast<cfloat>(flt.h[7][m]));
  CHECK(std::abs(out.at(7, 9, 0) - want) < 1e-5f * (1.0f + std::abs(want)));
  // scalar forms: test_cacgmm.cpp:53-79, :116-124
  CHECK(std::fabs(cacgmm::cacg_log_pdf({cdouble(1, 0)}, numerics::CMatrix::Identity(1, 1)) + 1.8378770664093453) < 1e-12);
  const std::vector<double> w = cacgmm::time_varying_weights({0.2, 0.3, 0.5}, {1, 0, 1});
  CHECK(std::fabs(w[0] - 0.2857142857142857) < 1e-15 && w[1] == 0.0);
  // enhance_batch: output lengths and names (test_scheduler.cpp:238-272)
  scheduler::PipelineConfig pc;
  pc.bss_iterations = 3;
  pc.out_dir = "/tmp/out";
  scheduler::SuperSegment ss;
  ss.recording_id = "rec";
  ss.speaker = "a";
  ss.audio = sig;
  ss.activity = act;
  scheduler::SuperSegment::Part p1, p2;
  p1.segment.id = "s1";
  p1.segment.start = 0.25;
  p1.segment.duration = 0.5;
  p1.sample_begin = 4000;
  p1.sample_end = 12000;
  p2 = p1;
  p2.segment.id = "s2";
  p2.sample_begin = 15000;
  p2.sample_end = 25000;  // clipped to 20000
  ss.parts = {p1, p2};
  scheduler::EnhancementResult r = scheduler::enhance_batch(ss, pc);
  CHECK(r.outputs.size() == 2 && r.outputs[0].audio.num_samples() == 8000 && r.outputs[1].audio.num_samples() == 5000);
  CHECK(r.outputs[0].path == "/tmp/out/rec-a-0000250_0000750.wav");
  CHECK(r.frames == sp.num_frames && std::isfinite(r.ll_final) && r.ref_channel >= 0 && r.ref_channel < 3);
  // failure isolation in a batch + the exception enhance_batch throws
  scheduler::SuperSegment bad = ss;
  bad.activity.frames -= 1;
  bad.activity.grid.resize(bad.activity.frames * 3);
  auto both = scheduler::enhance_batches({&bad, &ss}, pc);
  CHECK(both[0].error && !both[1].error && both[1].outputs.size() == 2);
  CHECK(both[1].outputs[0].audio.channels[0] == r.outputs[0].audio.channels[0]);
  try {
    scheduler::enhance_batch(bad, pc);
    CHECK(false);
  } catch (const ShapeError&) {
    ++g_checks;
  }
  std::printf("OK %d checks\n", g_checks);
  return 0;
}
