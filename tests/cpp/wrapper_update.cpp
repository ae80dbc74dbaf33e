// C++ caller of the drop-in through include/ver_gpu.hpp, shaped like the
// reference's train_single (bench.cpp:95-205): RolloutBuffer -> begin_rollout
// -> append_step* -> set_bootstrap -> close_rollout -> Learner::update.
//
//   wrapper_update nodevice        expect DeviceError from Context (no GPU)
//   wrapper_update engine <dir>    drive ver::gpu::InferenceEngine over every
//                                  env for <steps> batches (obs from <dir>),
//                                  write the dispatched actions and the view's
//                                  log-probs
//   wrapper_update <dir>           read the records written by
//                                  tests/test_cpp_wrapper.py, run one update,
//                                  write <dir>/params_out.f32, print the stats
#include <algorithm>
#include <cstdio>
#include <fstream>
#include <iostream>
#include <string>
#include <vector>

#include "ver_gpu.hpp"

template <class T>
static std::vector<T> load(const std::string& path, size_t n) {
  std::vector<T> v(n);
  std::ifstream f(path, std::ios::binary);
  if (!f.read(reinterpret_cast<char*>(v.data()), (std::streamsize)(n * sizeof(T))))
    throw std::runtime_error("short read: " + path);
  return v;
}

int main(int argc, char** argv) {
  if (argc < 2) return 2;
  const std::string mode = argv[1];
  if (mode == "nodevice") {
    try {
      ver::gpu::Context ctx(0);
    } catch (const ver::gpu::DeviceError& e) {
      std::printf("DeviceError: %s\n", e.what());
      return 0;
    }
    std::printf("expected DeviceError\n");
    return 1;
  }
  if (mode == "engine") {
    const std::string d = std::string(argv[2]) + "/";
    int T, N, D, H, steps;
    {
      std::ifstream m(d + "meta.txt");
      m >> T >> N >> D >> H >> steps;
    }
    const ver_model_config mc{D, H, H, 0, 2, 0};
    int64_t P = 0;
    int nt = 0;
    ver::gpu::check(ver_param_count(&mc, &P, &nt));
    auto params = load<float>(d + "params.f32", (size_t)P);
    auto obs = load<float>(d + "obs.f32", (size_t)(steps + 1) * N * D);
    ver::gpu::Context ctx(0);
    ver_engine_config ec{{T, N, /*Variable*/ 1, 0, D, 0, H}, mc, 12345};
    ver::gpu::InferenceEngine eng(ctx, ec, params, 1);
    eng.begin_rollout();
    std::vector<int32_t> env(N), step(N);
    std::vector<int64_t> ep(N, 0);
    std::vector<uint8_t> first(N, 1), dn(N, 0);
    std::vector<float> rew(N, 0.5f);
    for (int e = 0; e < N; ++e) env[e] = e;
    std::ofstream out(d + "actions.i32", std::ios::binary);
    for (int s = 0; s <= steps && !eng.rollout_done(); ++s) {
      for (int e = 0; e < N; ++e) step[e] = s;
      ver_request_batch rb{N, env.data(), obs.data() + (size_t)s * N * D, rew.data(), dn.data(), first.data(),
                           nullptr, ep.data(), step.data()};
      auto r = eng.process_batch(rb);
      out.write(reinterpret_cast<const char*>(r.action.data()), (std::streamsize)(r.action.size() * 4));
      std::fill(first.begin(), first.end(), 0);
    }
    eng.force_close();  // preempted close (fewer steps than T x N)
    eng.finalize_bootstraps();
    ver::gpu::RolloutView v = eng.close();
    std::printf("engine ok\n");
    return 0;
  }
  const std::string d = mode + "/";
  int T, N, D, H, n;
  {
    std::ifstream m(d + "meta.txt");
    m >> T >> N >> D >> H >> n;
  }
  auto env = load<int32_t>(d + "env.i32", n);
  auto obs = load<float>(d + "obs.f32", (size_t)n * D);
  auto act = load<int32_t>(d + "act.i32", n);
  auto logp = load<float>(d + "logp.f32", n);
  auto val = load<float>(d + "value.f32", n);
  auto rew = load<float>(d + "reward.f32", n);
  auto done = load<uint8_t>(d + "done.u8", n);
  auto hb = load<float>(d + "hb.f32", (size_t)n * H);
  auto hbv = load<uint8_t>(d + "hbv.u8", n);
  auto boot = load<float>(d + "boot.f32", N);
  auto bootv = load<uint8_t>(d + "bootv.u8", N);

  ver::gpu::Context ctx(0);
  ver_rollout_config rc{T, N, /*Variable*/ 1, 0, D, 0, H};
  ver::gpu::RolloutBuffer buf(ctx, rc);
  buf.begin_rollout(1);
  ver_step_batch b{};
  b.n = n;
  b.env_index = env.data();
  b.obs = obs.data();
  b.act_disc = act.data();
  b.log_prob = logp.data();
  b.value = val.data();
  b.reward = rew.data();
  b.done = done.data();
  b.h_before = hb.data();
  b.h_before_valid = hbv.data();
  buf.append(b);
  for (int e = 0; e < N; ++e)
    if (bootv[e]) buf.set_bootstrap(e, boot[e]);
  ver::gpu::RolloutView view = buf.close_rollout();
  // the reference's contract (rollout.cpp:103-104, test_rollout.cpp:180):
  // closing an empty buffer, or one still open, is a ProtocolError
  {
    ver::gpu::RolloutBuffer empty(ctx, rc);
    bool threw = false;
    try {
      empty.close_rollout();
    } catch (const ver::gpu::ProtocolError&) {
      threw = true;
    }
    empty.begin_rollout(1);
    ver_step_batch one = b;
    one.n = 1;
    empty.append(one);
    bool threw_open = false;
    try {
      empty.close_rollout();
    } catch (const ver::gpu::ProtocolError&) {
      threw_open = true;
    }
    if (!threw || !threw_open) {
      std::printf("expected ProtocolError on empty (%d) / open (%d) close\n", (int)threw, (int)threw_open);
      return 1;
    }
  }
  ver_model_config mc{D, H, H, 0, 2, 0};
  int64_t P = 0;
  int nt = 0;
  ver::gpu::check(ver_param_count(&mc, &P, &nt));
  auto params = load<float>(d + "params.f32", (size_t)P);
  ver_ppo_config pc{0.99, 0.95, 0.2, 2, 2, 0.5, 1.0};
  ver_entropy_controller ec{1e-3, 0.0, 1e-4, 1.0, 2.5e-4};
  ver::gpu::Learner learner(ctx, mc, params, pc, ec, 2.5e-4, 1000000, 77);
  const ver_train_stats st = learner.update(view);
  auto out = learner.params();
  std::ofstream(d + "params_out.f32", std::ios::binary)
      .write(reinterpret_cast<const char*>(out.data()), (std::streamsize)(out.size() * sizeof(float)));
  std::printf("{\"steps\": %d, \"fresh_steps\": %d, \"loss\": %.9g, \"alpha\": %.9g}\n", st.steps,
              st.fresh_steps, st.loss, st.alpha);
  return 0;
}
