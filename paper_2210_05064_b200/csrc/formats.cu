// formats.cu — the reference's on-disk formats, host code:
//   * the JSONL rollout trace: dump_view / load_view (rollout.cpp:293-432):
//     one "meta" line, one "seq" line per sequence (with its h0 row), one
//     "step" line per slot; read by `ver replay` (bench.cpp:373-409);
//   * the "ver-checkpoint" v1 JSON: save_checkpoint / load_checkpoint
//     (bench.cpp:411-441) with params_to_json / adam_to_json
//     (nn.cpp:314-387): tensors by name as {rows, cols, data}, Adam m / v in
//     tensors() order, alpha, consumed_steps, update_index.
// The reference writes them with nlohmann::json (keys sorted); this writer
// emits the same keys in the same order and fp32 values with 9 significant
// digits (exact round trip of every fp32 value); the reader is a small
// recursive-descent JSON parser that accepts any valid JSON of that schema,
// including the reference's own files.
#include <algorithm>
#include <cerrno>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <map>
#include <sstream>
#include <string>
#include <vector>

#include "common.cuh"
#include "policy.cuh"

namespace verg {
namespace fmt {

// ------------------------------------------------------------------ parser
struct J {
  enum Kind { NUL, BOOL, NUM, STR, ARR, OBJ } k = NUL;
  bool b = false;
  double n = 0.0;
  std::string s;  // string value, or the number's text (exact 64-bit integers)
  std::vector<J> a;
  std::vector<std::pair<std::string, J>> o;

  const J* find(const char* key) const {
    for (const auto& kv : o)
      if (kv.first == key) return &kv.second;
    return nullptr;
  }
  const J& at(const char* key) const {
    const J* v = find(key);
    if (!v) config_error(std::string("json: missing key \"") + key + "\"");
    return *v;
  }
  double num() const {
    if (k == BOOL) return b ? 1.0 : 0.0;
    if (k != NUM) config_error("json: expected a number");
    return n;
  }
  int64_t i64() const {
    if (k != NUM) config_error("json: expected an integer");
    errno = 0;
    char* end = nullptr;
    const long long v = std::strtoll(s.c_str(), &end, 10);
    if (errno == 0 && end && *end == 0) return v;
    return (int64_t)n;
  }
  uint64_t u64() const {
    if (k != NUM) config_error("json: expected an integer");
    errno = 0;
    char* end = nullptr;
    const unsigned long long v = std::strtoull(s.c_str(), &end, 10);
    if (errno == 0 && end && *end == 0) return v;
    return (uint64_t)n;
  }
  bool boolean() const {
    if (k == BOOL) return b;
    if (k == NUM) return n != 0.0;
    config_error("json: expected a boolean");
    return false;
  }
};

struct Parser {
  const char* p;
  const char* e;
  void ws() {
    while (p < e && (*p == ' ' || *p == '\t' || *p == '\n' || *p == '\r')) ++p;
  }
  [[noreturn]] void fail(const char* what) { config_error(std::string("json: ") + what); }
  bool lit(const char* w) {
    const size_t n = std::strlen(w);
    if ((size_t)(e - p) >= n && std::memcmp(p, w, n) == 0) {
      p += n;
      return true;
    }
    return false;
  }
  std::string str() {
    if (p >= e || *p != '"') fail("expected a string");
    ++p;
    std::string out;
    while (p < e && *p != '"') {
      char c = *p++;
      if (c == '\\') {
        if (p >= e) fail("bad escape");
        c = *p++;
        switch (c) {
          case 'n': out += '\n'; break;
          case 't': out += '\t'; break;
          case 'r': out += '\r'; break;
          case 'b': out += '\b'; break;
          case 'f': out += '\f'; break;
          case 'u': {
            if (e - p < 4) fail("bad \\u escape");
            const unsigned cp = (unsigned)std::strtoul(std::string(p, p + 4).c_str(), nullptr, 16);
            p += 4;
            if (cp < 0x80) out += (char)cp;
            else if (cp < 0x800) {
              out += (char)(0xC0 | (cp >> 6));
              out += (char)(0x80 | (cp & 0x3F));
            } else {
              out += (char)(0xE0 | (cp >> 12));
              out += (char)(0x80 | ((cp >> 6) & 0x3F));
              out += (char)(0x80 | (cp & 0x3F));
            }
            break;
          }
          default: out += c;
        }
      } else {
        out += c;
      }
    }
    if (p >= e) fail("unterminated string");
    ++p;
    return out;
  }
  J value() {
    ws();
    if (p >= e) fail("unexpected end");
    J v;
    const char c = *p;
    if (c == '{') {
      v.k = J::OBJ;
      ++p;
      ws();
      if (p < e && *p == '}') {
        ++p;
        return v;
      }
      while (true) {
        ws();
        std::string key = str();
        ws();
        if (p >= e || *p != ':') fail("expected ':'");
        ++p;
        v.o.emplace_back(std::move(key), value());
        ws();
        if (p < e && *p == ',') {
          ++p;
          continue;
        }
        if (p < e && *p == '}') {
          ++p;
          return v;
        }
        fail("expected ',' or '}'");
      }
    }
    if (c == '[') {
      v.k = J::ARR;
      ++p;
      ws();
      if (p < e && *p == ']') {
        ++p;
        return v;
      }
      while (true) {
        v.a.push_back(value());
        ws();
        if (p < e && *p == ',') {
          ++p;
          continue;
        }
        if (p < e && *p == ']') {
          ++p;
          return v;
        }
        fail("expected ',' or ']'");
      }
    }
    if (c == '"') {
      v.k = J::STR;
      v.s = str();
      return v;
    }
    if (lit("true")) {
      v.k = J::BOOL;
      v.b = true;
      return v;
    }
    if (lit("false")) {
      v.k = J::BOOL;
      return v;
    }
    if (lit("null")) return v;
    const char* s0 = p;
    while (p < e && (std::strchr("+-0123456789.eE", *p) != nullptr)) ++p;
    if (p == s0) fail("unexpected character");
    v.k = J::NUM;
    v.s.assign(s0, p);
    v.n = std::strtod(v.s.c_str(), nullptr);
    return v;
  }
};

J parse(const std::string& text) {
  Parser ps{text.data(), text.data() + text.size()};
  J v = ps.value();
  ps.ws();
  if (ps.p != ps.e) config_error("json: trailing characters");
  return v;
}

// ------------------------------------------------------------------ writer
struct W {
  std::string s;
  std::vector<bool> first;  // per open object: no member written yet
  void open() {
    s += '{';
    first.push_back(true);
  }
  void close() {
    s += '}';
    first.pop_back();
  }
  void key(const char* k) {
    if (!first.back()) s += ',';
    first.back() = false;
    s += '"';
    s += k;
    s += "\":";
  }
  void f32(float v) {
    if (!std::isfinite(v)) {
      s += "null";  // nlohmann::json writes non-finite numbers as null
      return;
    }
    char b[32];
    std::snprintf(b, sizeof b, "%.9g", (double)v);
    s += b;
  }
  void f64(double v) {
    if (!std::isfinite(v)) {
      s += "null";
      return;
    }
    char b[40];
    std::snprintf(b, sizeof b, "%.17g", v);
    s += b;
  }
  void i64(long long v) { s += std::to_string(v); }
  void u64(unsigned long long v) { s += std::to_string(v); }
  void boolean(bool v) { s += v ? "true" : "false"; }
  void str(const char* v) {
    s += '"';
    s += v;
    s += '"';
  }
  template <class T, class F>
  void arr(const T* v, size_t n, F f) {
    s += '[';
    for (size_t i = 0; i < n; ++i) {
      if (i) s += ',';
      f(v[i]);
    }
    s += ']';
  }
};

static float jf(const J& v) { return v.k == J::NUL ? NAN : (float)v.num(); }

}  // namespace fmt

// the learner's model config (learner.cu)
const ver_model_config* learner_model_config(ver_learner_s* l);

}  // namespace verg

using namespace verg;
using namespace verg::fmt;

extern "C" {

// dump_view (rollout.cpp:293-344)
ver_status ver_view_dump_jsonl(ver_view v, const char* path) {
  VER_API_BEGIN
  ver_view_host h{};
  if (ver_view_info(v, &h) != VER_OK) config_error("dump_view: bad view");
  const int S = h.size, D = h.obs_dim, A = h.act_dim, H = h.hidden_dim, K = h.num_seqs, N = h.N;
  std::vector<float> obs((size_t)S * D), actc((size_t)S * std::max(A, 1)), lp(S), val(S), rw(S), lat(S),
      h0((size_t)std::max(h.h0_rows, 1) * H), boot(N);
  std::vector<int32_t> actd(S), env(S), seq(S), step(S), counts(N);
  std::vector<uint8_t> done(S), stale(S), repl(S), bootv(N);
  std::vector<int64_t> ep(S);
  std::vector<uint64_t> ver(S);
  std::vector<ver_seq_desc> seqs(std::max(K, 1));
  h.obs = obs.data();
  h.act_cont = h.action_kind ? actc.data() : nullptr;
  h.act_disc = h.action_kind ? nullptr : actd.data();
  h.log_prob = lp.data();
  h.value = val.data();
  h.reward = rw.data();
  h.latency = lat.data();
  h.advantage = h.returns = nullptr;
  h.done = done.data();
  h.stale = stale.data();
  h.replayed = repl.data();
  h.env_index = env.data();
  h.seq_of_slot = seq.data();
  h.step_in_episode = step.data();
  h.episode_index = ep.data();
  h.version = ver.data();
  h.seqs = seqs.data();
  h.h0 = h0.data();
  h.per_env_counts = counts.data();
  h.env_bootstrap = boot.data();
  h.env_bootstrap_valid = bootv.data();
  const ver_status st = ver_view_download(v, &h);
  if (st != VER_OK) return st;
  std::ofstream out(path);
  if (!out) config_error(std::string("dump_view: cannot write ") + path);
  {
    W w;
    w.open();
    w.key("N"); w.i64(h.N);
    w.key("T"); w.i64(h.T);
    w.key("act_dim"); w.i64(A);
    w.key("action_kind"); w.str(h.action_kind ? "continuous" : "discrete");
    w.key("collect_wall_time"); w.f64(h.collect_wall_time);
    w.key("deficit"); w.i64(h.deficit);
    w.key("env_bootstrap"); w.arr(boot.data(), N, [&](float x) { w.f32(x); });
    w.key("env_bootstrap_valid"); w.arr(bootv.data(), N, [&](uint8_t x) { w.i64(x); });
    w.key("hidden_dim"); w.i64(H);
    w.key("obs_dim"); w.i64(D);
    w.key("per_env_counts"); w.arr(counts.data(), N, [&](int32_t x) { w.i64(x); });
    w.key("replayed_steps"); w.i64(h.replayed_steps);
    w.key("snapshot_version"); w.u64(h.snapshot_version);
    w.key("stale_steps"); w.i64(h.stale_steps);
    w.key("type"); w.str("meta");
    w.close();
    out << w.s << "\n";
  }
  for (int k = 0; k < K; ++k) {
    const ver_seq_desc& d = seqs[k];
    W w;
    w.open();
    w.key("env"); w.i64(d.env_index);
    w.key("h0"); w.arr(h0.data() + (size_t)d.h0_index * H, H, [&](float x) { w.f32(x); });
    w.key("length"); w.i64(d.length);
    w.key("seq_id"); w.i64(d.seq_id);
    w.key("stale"); w.boolean(d.stale != 0);
    w.key("start_offset"); w.i64(d.start_offset);
    w.key("type"); w.str("seq");
    w.close();
    out << w.s << "\n";
  }
  for (int i = 0; i < S; ++i) {
    W w;
    w.open();
    w.key("action");
    if (h.action_kind) w.arr(actc.data() + (size_t)i * A, A, [&](float x) { w.f32(x); });
    else w.i64(actd[i]);
    w.key("done"); w.boolean(done[i] != 0);
    w.key("env"); w.i64(env[i]);
    w.key("episode"); w.i64(ep[i]);
    w.key("latency"); w.f32(lat[i]);
    w.key("log_prob"); w.f32(lp[i]);
    w.key("obs"); w.arr(obs.data() + (size_t)i * D, D, [&](float x) { w.f32(x); });
    w.key("replayed"); w.boolean(repl[i] != 0);
    w.key("reward"); w.f32(rw[i]);
    w.key("seq"); w.i64(seq[i]);
    w.key("stale"); w.boolean(stale[i] != 0);
    w.key("t"); w.i64(step[i]);
    w.key("type"); w.str("step");
    w.key("value"); w.f32(val[i]);
    w.key("version"); w.u64(ver[i]);
    w.close();
    out << w.s << "\n";
  }
  if (!out) config_error(std::string("dump_view: write failed: ") + path);
  VER_API_END
}

// load_view (rollout.cpp:346-432): advantages / returns zero, seqs with
// parent_start_offset = start_offset, skip 0, h0_index = line order
ver_status ver_view_load_jsonl(ver_ctx ctx, const char* path, ver_view* out) {
  VER_API_BEGIN
  std::ifstream in(path);
  if (!in) config_error(std::string("load_view: cannot open ") + path);
  ver_view_host h{};
  bool have_meta = false;
  std::vector<float> boot, obs, actc, lp, val, rw, lat, h0;
  std::vector<uint8_t> bootv, done, stale, repl;
  std::vector<int32_t> counts, actd, env, seq, step;
  std::vector<int64_t> ep;
  std::vector<uint64_t> ver;
  std::vector<ver_seq_desc> seqs;
  std::string line;
  while (std::getline(in, line)) {
    if (line.empty()) continue;
    const J j = parse(line);
    const std::string type = j.at("type").s;
    if (type == "meta") {
      have_meta = true;
      h.T = (int)j.at("T").i64();
      h.N = (int)j.at("N").i64();
      h.action_kind = j.at("action_kind").s == "discrete" ? 0 : 1;
      h.obs_dim = (int)j.at("obs_dim").i64();
      h.act_dim = (int)j.at("act_dim").i64();
      h.hidden_dim = (int)j.at("hidden_dim").i64();
      h.deficit = (int)j.at("deficit").i64();
      h.stale_steps = (int)j.at("stale_steps").i64();
      const J* rs = j.find("replayed_steps");
      h.replayed_steps = rs ? (int)rs->i64() : 0;
      h.snapshot_version = j.at("snapshot_version").u64();
      h.collect_wall_time = j.at("collect_wall_time").num();
      for (const J& x : j.at("per_env_counts").a) counts.push_back((int32_t)x.i64());
      for (const J& x : j.at("env_bootstrap").a) boot.push_back(jf(x));
      for (const J& x : j.at("env_bootstrap_valid").a) bootv.push_back(x.boolean() ? 1 : 0);
    } else if (type == "seq") {
      if (!have_meta) config_error("load_view: seq line before meta");
      ver_seq_desc d{};
      d.seq_id = (int32_t)j.at("seq_id").i64();
      d.env_index = (int32_t)j.at("env").i64();
      d.length = (int32_t)j.at("length").i64();
      d.start_offset = (int32_t)j.at("start_offset").i64();
      d.parent_start_offset = d.start_offset;
      d.h0_index = (int32_t)seqs.size();
      d.stale = j.at("stale").boolean() ? 1 : 0;
      d.skip = 0;
      const auto& hv = j.at("h0").a;
      if ((int)hv.size() != h.hidden_dim) config_error("load_view: h0 row length != hidden_dim");
      for (const J& x : hv) h0.push_back(jf(x));
      seqs.push_back(d);
    } else if (type == "step") {
      if (!have_meta) config_error("load_view: step line before meta");
      const auto& ov = j.at("obs").a;
      if ((int)ov.size() != h.obs_dim) config_error("load_view: obs length != obs_dim");
      for (const J& x : ov) obs.push_back(jf(x));
      if (h.action_kind == 0) {
        actd.push_back((int32_t)j.at("action").i64());
      } else {
        const auto& av = j.at("action").a;
        if ((int)av.size() != h.act_dim) config_error("load_view: action length != act_dim");
        for (const J& x : av) actc.push_back(jf(x));
      }
      lp.push_back(jf(j.at("log_prob")));
      val.push_back(jf(j.at("value")));
      rw.push_back(jf(j.at("reward")));
      done.push_back(j.at("done").boolean() ? 1 : 0);
      stale.push_back(j.at("stale").boolean() ? 1 : 0);
      const J* rp = j.find("replayed");
      repl.push_back(rp && rp->boolean() ? 1 : 0);
      lat.push_back(jf(j.at("latency")));
      env.push_back((int32_t)j.at("env").i64());
      seq.push_back((int32_t)j.at("seq").i64());
      ep.push_back(j.at("episode").i64());
      step.push_back((int32_t)j.at("t").i64());
      ver.push_back(j.at("version").u64());
    }
  }
  if (!have_meta) config_error(std::string("load_view: no meta line in ") + path);
  const int S = (int)env.size();
  std::vector<float> zeros(std::max(S, 1), 0.f);
  h.size = S;
  h.num_seqs = (int)seqs.size();
  h.h0_rows = (int)seqs.size();
  h.obs = obs.data();
  h.act_cont = h.action_kind ? actc.data() : nullptr;
  h.act_disc = h.action_kind ? nullptr : actd.data();
  h.log_prob = lp.data();
  h.value = val.data();
  h.reward = rw.data();
  h.latency = lat.data();
  h.advantage = zeros.data();
  h.returns = zeros.data();
  h.done = done.data();
  h.stale = stale.data();
  h.replayed = repl.data();
  h.env_index = env.data();
  h.seq_of_slot = seq.data();
  h.step_in_episode = step.data();
  h.episode_index = ep.data();
  h.version = ver.data();
  h.seqs = seqs.data();
  h.h0 = h0.data();
  h.per_env_counts = counts.data();
  h.env_bootstrap = boot.data();
  h.env_bootstrap_valid = bootv.data();
  return ver_view_upload(ctx, &h, out);
  VER_API_END
}

// save_checkpoint (bench.cpp:411-424) with params_to_json / adam_to_json (nn.cpp:314-371)
ver_status ver_learner_save_checkpoint(ver_learner l, const char* path) {
  VER_API_BEGIN
  const ver_model_config mc = *learner_model_config(l);
  int64_t P = 0;
  int nt = 0;
  ver_param_count(&mc, &P, &nt);
  std::vector<float> params(P), m(P), v(P);
  int64_t step = 0, consumed = 0, upd = 0;
  double alpha = 0.0;
  ver_status st;
  if ((st = ver_learner_get_params(l, params.data())) != VER_OK) return st;
  if ((st = ver_learner_get_adam(l, m.data(), v.data(), &step)) != VER_OK) return st;
  if ((st = ver_learner_get_state(l, &alpha, &consumed, &upd)) != VER_OK) return st;
  struct T {
    std::string name;
    int rows, cols;
    int64_t off;
  };
  std::vector<T> ts;
  for (int i = 0; i < nt; ++i) {
    char name[16] = {0};
    int r = 0, c = 0;
    int64_t off = 0;
    ver_param_tensor(&mc, i, name, &r, &c, &off);
    ts.push_back({name, r, c, off});
  }
  auto matrix = [&](W& w, const std::vector<float>& src, const T& t) {
    w.open();
    w.key("cols"); w.i64(t.cols);
    w.key("data"); w.arr(src.data() + t.off, (size_t)t.rows * t.cols, [&](float x) { w.f32(x); });
    w.key("rows"); w.i64(t.rows);
    w.close();
  };
  W w;
  w.open();
  w.key("adam");
  {
    w.open();
    w.key("m");
    w.s += '[';
    for (size_t i = 0; i < ts.size(); ++i) {
      if (i) w.s += ',';
      matrix(w, m, ts[i]);
    }
    w.s += ']';
    w.key("step"); w.i64(step);
    w.key("v");
    w.s += '[';
    for (size_t i = 0; i < ts.size(); ++i) {
      if (i) w.s += ',';
      matrix(w, v, ts[i]);
    }
    w.s += ']';
    w.close();
  }
  w.key("alpha"); w.f64(alpha);
  w.key("consumed_steps"); w.i64(consumed);
  w.key("format"); w.str("ver-checkpoint");
  w.key("params");
  {
    w.open();
    w.key("act_dim"); w.i64(mc.act_dim);
    w.key("action_kind"); w.str(mc.action_kind ? "continuous" : "discrete");
    w.key("encoder_dim"); w.i64(mc.encoder_dim);
    w.key("hidden_dim"); w.i64(mc.hidden_dim);
    w.key("num_actions"); w.i64(mc.num_actions);
    w.key("obs_dim"); w.i64(mc.obs_dim);
    w.key("tensors");
    // nlohmann sorts object keys: tensors by name
    std::vector<size_t> order(ts.size());
    for (size_t i = 0; i < order.size(); ++i) order[i] = i;
    std::sort(order.begin(), order.end(), [&](size_t a, size_t b) { return ts[a].name < ts[b].name; });
    w.open();
    for (size_t i : order) {
      w.key(ts[i].name.c_str());
      matrix(w, params, ts[i]);
    }
    w.close();
    w.close();
  }
  w.key("update_index"); w.i64(upd);
  w.key("version"); w.i64(1);
  w.close();
  std::ofstream out(path);
  if (!out) config_error(std::string("cannot write checkpoint: ") + path);
  out << w.s << "\n";
  VER_API_END
}

static J read_checkpoint(const char* path) {
  std::ifstream in(path);
  if (!in) config_error(std::string("cannot open checkpoint: ") + path);
  std::stringstream ss;
  ss << in.rdbuf();
  J j = parse(ss.str());
  const J* f = j.find("format");
  const J* v = j.find("version");
  if (!f || f->k != J::STR || f->s != "ver-checkpoint" || !v || v->k != J::NUM || v->i64() != 1)
    config_error(std::string("unrecognized checkpoint format: ") + path);
  return j;
}

static ver_model_config checkpoint_config(const J& p) {
  ver_model_config mc{};
  mc.obs_dim = (int)p.at("obs_dim").i64();
  mc.encoder_dim = (int)p.at("encoder_dim").i64();
  mc.hidden_dim = (int)p.at("hidden_dim").i64();
  mc.action_kind = p.at("action_kind").s == "discrete" ? 0 : 1;
  mc.num_actions = (int)p.at("num_actions").i64();
  mc.act_dim = (int)p.at("act_dim").i64();
  return mc;
}

// the model config stored in a checkpoint (to construct a matching learner)
ver_status ver_checkpoint_model_config(const char* path, ver_model_config* out) {
  VER_API_BEGIN
  *out = checkpoint_config(read_checkpoint(path).at("params"));
  VER_API_END
}

// load_checkpoint (bench.cpp:426-441) into an existing learner of the same model
ver_status ver_learner_load_checkpoint(ver_learner l, const char* path) {
  VER_API_BEGIN
  const J j = read_checkpoint(path);
  const J& pj = j.at("params");
  const ver_model_config mc = checkpoint_config(pj);
  const ver_model_config& lm = *learner_model_config(l);
  // only the fields that fix tensor shapes for this action kind (an unused
  // num_actions / act_dim may differ); the per-tensor rows / cols checks follow
  const bool discrete = mc.action_kind == 0;
  if (mc.obs_dim != lm.obs_dim || mc.encoder_dim != lm.encoder_dim || mc.hidden_dim != lm.hidden_dim ||
      mc.action_kind != lm.action_kind || (discrete && mc.num_actions != lm.num_actions) ||
      (!discrete && mc.act_dim != lm.act_dim))
    config_error("load_checkpoint: model differs from the learner's");
  int64_t P = 0;
  int nt = 0;
  ver_param_count(&mc, &P, &nt);
  std::vector<float> params(P), m(P), v(P);
  const J& tj = pj.at("tensors");
  const J& aj = j.at("adam");
  const auto& ma = aj.at("m").a;
  const auto& va = aj.at("v").a;
  if ((int)ma.size() != nt || (int)va.size() != nt) config_error("load_checkpoint: adam tensor count");
  for (int i = 0; i < nt; ++i) {
    char name[16] = {0};
    int r = 0, c = 0;
    int64_t off = 0;
    ver_param_tensor(&mc, i, name, &r, &c, &off);
    auto fill = [&](const J& mj, std::vector<float>& dst) {
      if (mj.at("rows").i64() != r || mj.at("cols").i64() != c)
        config_error(std::string("load_checkpoint: shape of ") + name);
      const auto& d = mj.at("data").a;
      if ((int64_t)d.size() != (int64_t)r * c) config_error(std::string("load_checkpoint: size of ") + name);
      for (int64_t k = 0; k < (int64_t)r * c; ++k) dst[off + k] = jf(d[k]);
    };
    fill(tj.at(name), params);
    fill(ma[i], m);
    fill(va[i], v);
  }
  ver_status st;
  if ((st = ver_learner_set_params(l, params.data())) != VER_OK) return st;
  if ((st = ver_learner_set_adam(l, m.data(), v.data(), aj.at("step").i64())) != VER_OK) return st;
  if ((st = ver_learner_set_state(l, j.at("alpha").num(), j.at("consumed_steps").i64(),
                                  j.at("update_index").i64())) != VER_OK)
    return st;
  VER_API_END
}

}  // extern "C"
