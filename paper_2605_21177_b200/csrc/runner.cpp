// runner.cpp -- experiment configs, the built-in presets and the artifact bundle, driving the
// GPU engine ("config/presets for CLI parity").
//
// Reference surface this serves (same behaviour, files and error text):
//   * ExperimentConfig + parse_config / load_config_file / config_to_json
//     (include/chunkft/config.hpp:20-67, src/config.cpp:138-352);
//   * make_preset / preset_names / run_experiment / summary_text / run_preset_checks
//     (include/chunkft/runner.hpp:14-42, src/runner.cpp:40-260);
//   * the synthetic data generators (src/model.cpp:162-264) and the random / formula
//     parameter inits (model.cpp:99-128) -- std::mt19937_64 and the libstdc++ distributions,
//     so the batches and the initial parameters are the reference's bit for bit;
//   * the memory trace, jitter and measured back-prop cost (src/accounting.cpp:14-166,
//     src/trainer.cpp:31-99).
// The training itself is the engine's (engine.cpp): the model is built once on the device,
// every step runs there, and the host only does this bookkeeping around it.
#include <cinttypes>
#include <cmath>
#include <cstring>
#include <cstdio>
#include <filesystem>
#include <fstream>
#include <functional>
#include <memory>
#include <random>
#include <sstream>
#include <string>
#include <vector>

#include <json.hpp>

#include "cft_common.h"
#include "engine.h"

namespace cft::run {

using nlohmann::json;

enum LayerType { kLinear = 0, kEmbedding = 1, kLayerNorm = 2, kTanh = 3 };
enum Loss { kSum = 0, kSquared = 1, kHalfSq = 2, kSoftmaxCe = 3 };

struct LayerCfg {
  int type = kLinear;
  int in = 0, out = 0;
  bool bias = true;
  int vocab = 0, dim = 0, seq = 1;
};

struct DatasetCfg {  // DatasetSpec (model.hpp:104-114)
  std::string generator = "regression";
  int size = 256, batch = 32, input_dim = 8, target_dim = 1, classes = 2, vocab = 16, seq = 1;
  uint64_t seed = 7;
};

struct Experiment {  // ExperimentConfig (config.hpp:36-49)
  std::vector<LayerCfg> layers;
  int loss = kHalfSq;
  DatasetCfg data;
  int K = 1, T = 1;
  int64_t steps = 0;
  bool prefetch = false;
  int64_t bandwidth = 0;
  cft_adamw_hyper hyper{1e-3, 0.9, 0.999, 1e-8, 0.0};
  bool plain = false;  // OptimKind::plain
  host::CostPolicy policy;
  bool per_tensor = false;
  bool formula_init = false;
  int micro_batches = 1;
  int64_t activation_bytes = 0;
  std::string out_dir;
  uint64_t seed = 7;
};

const char* const kLossNames[] = {"sum", "squared", "half_sq", "softmax_ce"};

// ---- parse_config (config.cpp:138-298) ------------------------------------------------------
// Each JSON object is read through a Section: it knows its dotted path for error messages,
// checks keys against the allowed set up front and types every field it hands out.
class Section {
 public:
  Section(const json& j, std::string where, std::initializer_list<const char*> allowed)
      : j_(j), where_(std::move(where)) {
    if (!j_.is_object()) fail(where_, "expected an object");
    for (const auto& item : j_.items()) {
      bool known = false;
      for (const char* k : allowed) known = known || item.key() == k;
      if (!known) fail(where_, "unknown key '" + item.key() + "'");
    }
  }
  [[noreturn]] static void fail(const std::string& where, const std::string& what) {
    throw Error(where + ": " + what);
  }
  std::string at(const char* key) const { return where_ + "." + key; }
  bool has(const char* key) const { return j_.contains(key); }
  int64_t i64(const char* key, int64_t dflt) const {
    if (!has(key)) return dflt;
    if (!j_.at(key).is_number_integer()) fail(at(key), "expected an integer");
    return j_.at(key).get<int64_t>();
  }
  int i32(const char* key, int dflt) const { return static_cast<int>(i64(key, dflt)); }
  double num(const char* key, double dflt) const {
    if (!has(key)) return dflt;
    if (!j_.at(key).is_number()) fail(at(key), "expected a number");
    return j_.at(key).get<double>();
  }
  bool flag(const char* key, bool dflt) const {
    if (!has(key)) return dflt;
    if (!j_.at(key).is_boolean()) fail(at(key), "expected a boolean");
    return j_.at(key).get<bool>();
  }
  std::string str(const char* key, const std::string& dflt) const {
    if (!has(key)) return dflt;
    if (!j_.at(key).is_string()) fail(at(key), "expected a string");
    return j_.at(key).get<std::string>();
  }
  // choose one of `names` (returns its index) or fail with the reference's listing
  int pick(const char* key, const std::string& dflt, const std::vector<std::string>& names,
           const char* what) const {
    const std::string v = str(key, dflt);
    std::string list;
    for (size_t i = 0; i < names.size(); ++i) {
      if (v == names[i]) return static_cast<int>(i);
      list += (i ? ", " : "") + names[i];
    }
    fail(at(key), std::string("unknown ") + what + " '" + v + "' (" + list + ")");
  }
  const json& raw(const char* key) const { return j_.at(key); }
  void at_least(const char* key, int64_t v, int64_t lo) const {
    if (v < lo) fail(at(key), "must be >= " + std::to_string(lo));
  }

 private:
  const json& j_;
  std::string where_;
};

LayerCfg parse_layer(const json& j, const std::string& where) {
  if (!j.is_object()) Section::fail(where, "expected an object");
  std::string type;
  if (j.contains("type")) {
    if (!j.at("type").is_string()) Section::fail(where + ".type", "expected a string");
    type = j.at("type").get<std::string>();
  }
  LayerCfg L;
  if (type == "linear") {
    Section s(j, where, {"type", "in", "out", "bias"});
    L.type = kLinear;
    L.in = s.i32("in", 0);
    L.out = s.i32("out", 0);
    L.bias = s.flag("bias", true);
    s.at_least("in", L.in, 1);
    s.at_least("out", L.out, 1);
  } else if (type == "embedding") {
    Section s(j, where, {"type", "vocab", "dim", "seq"});
    L.type = kEmbedding;
    L.vocab = s.i32("vocab", 0);
    L.dim = s.i32("dim", 0);
    L.seq = s.i32("seq", 1);
    s.at_least("vocab", L.vocab, 1);
    s.at_least("dim", L.dim, 1);
    s.at_least("seq", L.seq, 1);
  } else if (type == "layernorm") {
    Section s(j, where, {"type", "dim"});
    L.type = kLayerNorm;
    L.dim = s.i32("dim", 0);
    s.at_least("dim", L.dim, 1);
  } else if (type == "tanh") {
    Section s(j, where, {"type"});
    L.type = kTanh;
  } else {
    Section::fail(where + ".type",
                  "unknown layer type '" + type + "' (linear, embedding, layernorm, tanh)");
  }
  return L;
}

// trainable rows the model will register (bias / norm vectors are out x 1: one row per scalar)
int64_t trainable_rows(const std::vector<LayerCfg>& layers) {
  int64_t rows = 0;
  for (const LayerCfg& L : layers) {
    if (L.type == kLinear) rows += L.bias ? 2 * L.out : L.out;
    if (L.type == kEmbedding) rows += L.vocab;
    if (L.type == kLayerNorm) rows += 2 * L.dim;
  }
  return rows;
}

void validate_hyper(const cft_adamw_hyper& h) {  // AdamWHyper::validate (optimizer.cpp:12-18)
  if (h.eta <= 0.0) throw Error("optimizer: eta must be positive");
  if (h.beta1 < 0.0 || h.beta1 >= 1.0) throw Error("optimizer: beta1 must be in [0,1)");
  if (h.beta2 < 0.0 || h.beta2 >= 1.0) throw Error("optimizer: beta2 must be in [0,1)");
  if (h.epsilon <= 0.0) throw Error("optimizer: epsilon must be positive");
  if (h.weight_decay < 0.0) throw Error("optimizer: weight_decay must be non-negative");
}

Experiment parse_config(const json& doc) {
  Section top(doc, "config", {"model", "dataset", "schedule", "optimizer", "policy", "plan",
                              "init", "micro_batches", "activation_bytes", "out_dir", "seed"});
  Experiment e;

  if (!top.has("model")) Section::fail("config.model", "required");
  {
    Section m(top.raw("model"), "config.model", {"layers", "loss"});
    if (!m.has("layers")) Section::fail("config.model.layers", "required");
    const json& layers = m.raw("layers");
    if (!layers.is_array() || layers.empty())
      Section::fail("config.model.layers", "expected a non-empty array");
    for (size_t i = 0; i < layers.size(); ++i)
      e.layers.push_back(parse_layer(layers[i], "config.model.layers[" + std::to_string(i) + "]"));
    e.loss = m.pick("loss", "half_sq", {"sum", "squared", "half_sq", "softmax_ce"}, "loss");
  }

  if (top.has("dataset")) {
    Section d(top.raw("dataset"), "config.dataset",
              {"generator", "size", "batch", "input_dim", "target_dim", "classes", "vocab", "seq",
               "seed"});
    DatasetCfg& D = e.data;
    const std::vector<std::string> generators = {"regression", "classification", "tokens",
                                                 "identity"};
    D.generator = generators[d.pick("generator", "regression", generators, "generator")];
    D.size = d.i32("size", D.size);
    D.batch = d.i32("batch", D.batch);
    D.input_dim = d.i32("input_dim", D.input_dim);
    D.target_dim = d.i32("target_dim", D.target_dim);
    D.classes = d.i32("classes", D.classes);
    D.vocab = d.i32("vocab", D.vocab);
    D.seq = d.i32("seq", D.seq);
    D.seed = static_cast<uint64_t>(d.i64("seed", static_cast<int64_t>(D.seed)));
    d.at_least("size", D.size, 1);
    d.at_least("batch", D.batch, 1);
    if (D.batch > D.size) Section::fail("config.dataset.batch", "must not exceed dataset size");
  }

  if (!top.has("schedule")) Section::fail("config.schedule", "required");
  {
    Section s(top.raw("schedule"), "config.schedule",
              {"K", "T", "steps", "prefetch", "bandwidth_bytes_per_step"});
    e.K = s.i32("K", 8);
    s.at_least("K", e.K, 1);
    e.T = s.i32("T", e.K);  // T defaults to K (config.cpp:192-194)
    s.at_least("T", e.T, 1);
    if (!s.has("steps")) Section::fail("config.schedule.steps", "required");
    e.steps = s.i64("steps", 0);
    s.at_least("steps", e.steps, 1);
    e.prefetch = s.flag("prefetch", false);
    e.bandwidth = s.i64("bandwidth_bytes_per_step", 0);
    s.at_least("bandwidth_bytes_per_step", e.bandwidth, 0);
  }

  if (top.has("optimizer")) {
    Section o(top.raw("optimizer"), "config.optimizer",
              {"kind", "eta", "beta1", "beta2", "epsilon", "weight_decay"});
    e.plain = o.pick("kind", "adamw", {"adamw", "plain"}, "kind") == 1;
    e.hyper.eta = o.num("eta", e.hyper.eta);
    e.hyper.beta1 = o.num("beta1", e.hyper.beta1);
    e.hyper.beta2 = o.num("beta2", e.hyper.beta2);
    e.hyper.epsilon = o.num("epsilon", e.hyper.epsilon);
    e.hyper.weight_decay = o.num("weight_decay", e.hyper.weight_decay);
    try {
      validate_hyper(e.hyper);
    } catch (const Error& err) {
      Section::fail("config.optimizer", err.what());
    }
  }

  if (top.has("policy")) {
    Section p(top.raw("policy"), "config.policy",
              {"param_bytes", "grad_bytes", "master_bytes", "moment1_bytes", "moment2_bytes"});
    host::CostPolicy& P = e.policy;
    P.param_bytes = p.i32("param_bytes", P.param_bytes);
    P.grad_bytes = p.i32("grad_bytes", P.grad_bytes);
    P.master_bytes = p.i32("master_bytes", P.master_bytes);
    P.moment1_bytes = p.i32("moment1_bytes", P.moment1_bytes);
    P.moment2_bytes = p.i32("moment2_bytes", P.moment2_bytes);
    try {
      P.validate();
    } catch (const std::exception& err) {
      Section::fail("config.policy", err.what());
    }
  }

  e.per_tensor = top.pick("plan", "byte_balanced", {"byte_balanced", "per_tensor"}, "plan") == 1;
  e.formula_init = top.pick("init", "random", {"random", "formula"}, "init") == 1;
  e.micro_batches = top.i32("micro_batches", 1);
  top.at_least("micro_batches", e.micro_batches, 1);
  e.activation_bytes = top.i64("activation_bytes", 0);
  top.at_least("activation_bytes", e.activation_bytes, 0);
  e.out_dir = top.str("out_dir", "");
  e.seed = static_cast<uint64_t>(top.i64("seed", 7));

  // a plan cannot have more chunks than the model has trainable rows (config.cpp:287-295)
  const int64_t rows = trainable_rows(e.layers);
  if (e.K > rows)
    Section::fail("config.schedule.K", "chunk count exceeds row granularity (K=" +
                                           std::to_string(e.K) +
                                           ", trainable rows=" + std::to_string(rows) + ")");
  return e;
}

// ---- config_to_json (config.cpp:312-352): nlohmann's default (sorted) object, dump(2) -------
json to_json(const Experiment& e) {
  json layers = json::array();
  for (const LayerCfg& L : e.layers) {
    switch (L.type) {
      case kLinear:
        layers.push_back({{"type", "linear"}, {"in", L.in}, {"out", L.out}, {"bias", L.bias}});
        break;
      case kEmbedding:
        layers.push_back({{"type", "embedding"}, {"vocab", L.vocab}, {"dim", L.dim}, {"seq", L.seq}});
        break;
      case kLayerNorm:
        layers.push_back({{"type", "layernorm"}, {"dim", L.dim}});
        break;
      default:
        layers.push_back({{"type", "tanh"}});
    }
  }
  const DatasetCfg& D = e.data;
  json j;
  j["model"] = {{"layers", layers}, {"loss", kLossNames[e.loss]}};
  j["dataset"] = {{"generator", D.generator}, {"size", D.size},          {"batch", D.batch},
                  {"input_dim", D.input_dim}, {"target_dim", D.target_dim},
                  {"classes", D.classes},     {"vocab", D.vocab},        {"seq", D.seq},
                  {"seed", D.seed}};
  j["schedule"] = {{"K", e.K}, {"T", e.T}, {"steps", e.steps}, {"prefetch", e.prefetch},
                   {"bandwidth_bytes_per_step", e.bandwidth}};
  j["optimizer"] = {{"kind", e.plain ? "plain" : "adamw"}, {"eta", e.hyper.eta},
                    {"beta1", e.hyper.beta1},               {"beta2", e.hyper.beta2},
                    {"epsilon", e.hyper.epsilon},           {"weight_decay", e.hyper.weight_decay}};
  j["policy"] = {{"param_bytes", e.policy.param_bytes},     {"grad_bytes", e.policy.grad_bytes},
                 {"master_bytes", e.policy.master_bytes},   {"moment1_bytes", e.policy.moment1_bytes},
                 {"moment2_bytes", e.policy.moment2_bytes}};
  j["plan"] = e.per_tensor ? "per_tensor" : "byte_balanced";
  j["init"] = e.formula_init ? "formula" : "random";
  j["micro_batches"] = e.micro_batches;
  j["activation_bytes"] = e.activation_bytes;
  j["out_dir"] = e.out_dir;
  j["seed"] = e.seed;
  return j;
}

// ---- presets (runner.cpp:40-129) ------------------------------------------------------------
LayerCfg linear(int in, int out, bool bias = true) {
  LayerCfg L;
  L.type = kLinear;
  L.in = in;
  L.out = out;
  L.bias = bias;
  return L;
}
LayerCfg embedding(int vocab, int dim, int seq) {
  LayerCfg L;
  L.type = kEmbedding;
  L.vocab = vocab;
  L.dim = dim;
  L.seq = seq;
  return L;
}
LayerCfg tanh_layer() {
  LayerCfg L;
  L.type = kTanh;
  return L;
}

const std::vector<std::string>& preset_names() {
  static const std::vector<std::string> names = {"quadratic-k2", "mlp-imbalanced-layers",
                                                 "mlp-imbalanced-layers-identity",
                                                 "dense-reduction", "classification-sanity"};
  return names;
}

Experiment make_preset(const std::string& name) {
  Experiment e;
  if (name == "quadratic-k2") {
    // one square linear on the identity batch: loss = 0.5 ||W||^2 exactly
    e.layers = {linear(8, 8, false)};
    e.loss = kHalfSq;
    e.data.generator = "identity";
    e.data.input_dim = e.data.target_dim = e.data.size = e.data.batch = 8;
    e.K = 2;
    e.T = 1;
    e.steps = 8;
    e.plain = true;
    e.hyper.eta = 0.5;
    e.formula_init = true;
  } else if (name == "mlp-imbalanced-layers" || name == "mlp-imbalanced-layers-identity") {
    // a dominant embedding table next to a small head; the per-tensor plan makes the step
    // totals swing with the table
    e.layers = {embedding(512, 16, 4), linear(64, 4)};
    e.loss = kSoftmaxCe;
    e.data.generator = "tokens";
    e.data.vocab = 512;
    e.data.seq = 4;
    e.data.batch = 8;
    e.data.size = 64;
    e.T = 1;
    e.hyper.eta = 1e-3;
    e.per_tensor = name == "mlp-imbalanced-layers-identity";
    e.K = e.per_tensor ? 3 : 4;
    e.steps = e.per_tensor ? 15 : 16;
  } else if (name == "dense-reduction") {
    e.layers = {linear(8, 16), tanh_layer(), linear(16, 1)};
    e.loss = kHalfSq;
    e.data.generator = "regression";
    e.data.input_dim = 8;
    e.data.target_dim = 1;
    e.data.batch = 16;
    e.data.size = 128;
    e.K = e.T = 1;
    e.steps = 32;
    e.hyper.eta = 1e-3;
  } else if (name == "classification-sanity") {
    e.layers = {linear(8, 32), tanh_layer(), linear(32, 2)};
    e.loss = kSoftmaxCe;
    e.data.generator = "classification";
    e.data.input_dim = 8;
    e.data.classes = 2;
    e.data.size = 1024;
    e.data.batch = 32;
    e.K = e.T = 8;
    e.steps = 640;  // ten rotations
    e.hyper.eta = 5e-3;
  } else {
    std::string known;
    for (const auto& n : preset_names()) known += " " + n;
    throw Error("unknown preset '" + name + "' (known:" + known + ")");
  }
  return e;
}

// ---- the model's tensors, initial parameters and batches ------------------------------------
struct TensorDesc {
  std::string name;
  int64_t rows, cols;
  int layer;
  char role;  // 'w' weight/table, 'b' bias, 'g' gamma, 'e' beta
};

std::vector<TensorDesc> tensors_of(const std::vector<LayerCfg>& layers) {
  std::vector<TensorDesc> t;
  for (size_t i = 0; i < layers.size(); ++i) {
    const LayerCfg& L = layers[i];
    const std::string idx = std::to_string(i);
    const int li = static_cast<int>(i);
    if (L.type == kLinear) {
      t.push_back({"linear" + idx + ".weight", L.out, L.in, li, 'w'});
      if (L.bias) t.push_back({"linear" + idx + ".bias", L.out, 1, li, 'b'});
    } else if (L.type == kEmbedding) {
      t.push_back({"embedding" + idx + ".table", L.vocab, L.dim, li, 'w'});
    } else if (L.type == kLayerNorm) {
      t.push_back({"layernorm" + idx + ".gamma", L.dim, 1, li, 'g'});
      t.push_back({"layernorm" + idx + ".beta", L.dim, 1, li, 'e'});
    }
  }
  return t;
}

// Model::init_params (model.cpp:99-117) / init_params_formula (model.cpp:119-128)
std::vector<double> initial_params(const std::vector<TensorDesc>& ts, bool formula,
                                   uint64_t seed) {
  std::vector<double> p;
  std::mt19937_64 rng(seed);
  std::uniform_real_distribution<double> uni(-0.5, 0.5);
  for (size_t i = 0; i < ts.size(); ++i) {
    const TensorDesc& t = ts[i];
    const int64_t n = t.rows * t.cols;
    for (int64_t k = 0; k < n; ++k) {
      if (formula) {
        const double v = 0.1 * std::sin(0.7 * static_cast<double>(i) + 0.3 * static_cast<double>(k));
        p.push_back(t.role == 'g' ? 1.0 + v : v);
      } else if (t.role == 'g') {
        p.push_back(1.0);
      } else if (t.role != 'w') {
        p.push_back(0.0);  // biases and betas start at zero and draw nothing from the stream
      } else {
        p.push_back(uni(rng) * (1.0 / std::sqrt(static_cast<double>(t.cols))));
      }
    }
  }
  return p;
}

struct HostBatch {
  int rows = 0;
  std::vector<double> x, target;
  std::vector<int32_t> tokens, labels;
};

int output_dim(const std::vector<LayerCfg>& layers) {  // Model::output_dim (model.cpp:54-64)
  int dim = -1;
  for (const LayerCfg& L : layers) {
    if (L.type == kLinear) dim = L.out;
    if (L.type == kEmbedding) dim = L.dim * L.seq;
  }
  if (dim < 0) throw Error("model output width undetermined");
  return dim;
}

// make_stream (model.cpp:162-264): one generator stream per dataset, batch after batch
std::vector<HostBatch> make_batches(const DatasetCfg& D, const std::vector<LayerCfg>& layers,
                                    int loss) {
  std::vector<HostBatch> out;
  const int nb = std::max(1, D.size / D.batch);
  std::mt19937_64 rng(D.seed);
  std::normal_distribution<double> gauss(0.0, 1.0);
  if (D.generator == "identity") {
    HostBatch b;
    b.rows = D.input_dim;
    b.x.assign(static_cast<size_t>(D.input_dim) * D.input_dim, 0.0);
    for (int i = 0; i < D.input_dim; ++i) b.x[static_cast<size_t>(i) * D.input_dim + i] = 1.0;
    b.target.assign(static_cast<size_t>(D.input_dim) * D.target_dim, 0.0);
    out.push_back(std::move(b));
  } else if (D.generator == "regression") {
    // a fixed random teacher (target_dim x input_dim), then x ~ N(0,1), y = tanh(teacher x)
    std::vector<double> teacher(static_cast<size_t>(D.target_dim) * D.input_dim);
    for (double& v : teacher) v = gauss(rng) / std::sqrt(static_cast<double>(D.input_dim));
    for (int n = 0; n < nb; ++n) {
      HostBatch b;
      b.rows = D.batch;
      b.x.resize(static_cast<size_t>(D.batch) * D.input_dim);
      for (double& v : b.x) v = gauss(rng);
      b.target.resize(static_cast<size_t>(D.batch) * D.target_dim);
      for (int r = 0; r < D.batch; ++r)
        for (int c = 0; c < D.target_dim; ++c) {
          double acc = 0.0;
          for (int i = 0; i < D.input_dim; ++i)
            acc += teacher[static_cast<size_t>(c) * D.input_dim + i] *
                   b.x[static_cast<size_t>(r) * D.input_dim + i];
          b.target[static_cast<size_t>(r) * D.target_dim + c] = std::tanh(acc);
        }
      out.push_back(std::move(b));
    }
  } else if (D.generator == "classification") {
    // class centres on a circle in the first two features; x = centre + 0.4 N(0,1)
    std::uniform_int_distribution<int> pick_class(0, D.classes - 1);
    std::vector<double> centre(static_cast<size_t>(D.classes) * D.input_dim, 0.0);
    for (int c = 0; c < D.classes; ++c) {
      const double ang = 2.0 * 3.14159265358979323846 * c / D.classes;
      centre[static_cast<size_t>(c) * D.input_dim] = 2.0 * std::cos(ang);
      if (D.input_dim > 1) centre[static_cast<size_t>(c) * D.input_dim + 1] = 2.0 * std::sin(ang);
    }
    for (int n = 0; n < nb; ++n) {
      HostBatch b;
      b.rows = D.batch;
      b.x.resize(static_cast<size_t>(D.batch) * D.input_dim);
      b.labels.resize(D.batch);
      for (int r = 0; r < D.batch; ++r) {
        const int cls = pick_class(rng);
        b.labels[r] = cls;
        for (int i = 0; i < D.input_dim; ++i)
          b.x[static_cast<size_t>(r) * D.input_dim + i] =
              centre[static_cast<size_t>(cls) * D.input_dim + i] + 0.4 * gauss(rng);
      }
      out.push_back(std::move(b));
    }
  } else if (D.generator == "tokens") {
    const int width = output_dim(layers);
    std::uniform_int_distribution<int> pick_token(0, D.vocab - 1);
    for (int n = 0; n < nb; ++n) {
      HostBatch b;
      b.rows = D.batch;
      b.tokens.resize(static_cast<size_t>(D.batch) * D.seq);
      for (int32_t& t : b.tokens) t = pick_token(rng);
      if (loss == kSoftmaxCe) {
        std::uniform_int_distribution<int> pick_label(0, width - 1);
        b.labels.resize(D.batch);
        for (int32_t& l : b.labels) l = pick_label(rng);
      } else if (loss != kSum) {
        b.target.resize(static_cast<size_t>(D.batch) * width);
        for (double& v : b.target) v = gauss(rng);
      }
      out.push_back(std::move(b));
    }
  } else {
    throw Error("unknown data generator '" + D.generator + "'");
  }
  return out;
}

// ---- accounting (accounting.cpp) ------------------------------------------------------------
struct MemorySample {
  int64_t step, params, state, activations, transfers;
  int64_t total() const { return params + state + activations + transfers; }
};

std::string fmt(double v) {  // format_double (csvio.cpp:13-17)
  char b[64];
  std::snprintf(b, sizeof b, "%.17g", v);
  return b;
}

struct Result {
  Experiment cfg;  // effective: K snapped to the plan
  host::ChunkPlan plan;
  std::vector<MemorySample> memory;
  int64_t transfer_events = 0, noop_loads = 0;
  int64_t chunked_macs = 0, rotations = 0, dense_macs = 0;
  double initial_loss = 0.0, final_loss = 0.0;
  double peak = 0.0, mean = 0.0, jitter = 0.0, jitter_bound = 0.0, bp_ratio = 0.0;
};

// parameter-gradient multiply-accumulates for one micro-batch, restricted to the active
// chunk's slices (ops.cpp:38-119) or dense over every tensor (autodiff.cpp:108-167)
int64_t grad_macs(const std::vector<LayerCfg>& layers, const std::vector<TensorDesc>& ts,
                  const HostBatch& b, const std::vector<host::SliceRef>* mask) {
  auto layer_rows = [&](const TensorDesc& t) -> int64_t {
    const LayerCfg& L = layers[t.layer];
    return L.type == kEmbedding ? static_cast<int64_t>(b.rows) * L.seq : b.rows;
  };
  int64_t macs = 0;
  if (!mask) {
    for (const TensorDesc& t : ts) {
      const LayerCfg& L = layers[t.layer];
      if (L.type == kEmbedding) macs += layer_rows(t) * L.dim;
      else macs += t.rows * t.cols * layer_rows(t);  // weight, bias, gamma, beta alike
    }
    return macs;
  }
  for (const host::SliceRef& s : *mask) {
    const TensorDesc& t = ts[s.tensor_id];
    const LayerCfg& L = layers[t.layer];
    if (L.type == kEmbedding) {
      int64_t matched = 0;
      for (int32_t tok : b.tokens) matched += tok >= s.row_begin && tok < s.row_end;
      macs += matched * L.dim;
    } else {
      macs += s.row_count() * t.cols * layer_rows(t);
    }
  }
  return macs;
}

std::string summary_text(const struct Result& R);

Result run_experiment(const Experiment& cfg, int dtype, cudaStream_t stream) {
  Result R;
  R.cfg = cfg;
  validate_hyper(cfg.hyper);
  const std::vector<TensorDesc> ts = tensors_of(cfg.layers);
  const std::vector<double> init = initial_params(ts, cfg.formula_init, cfg.seed);
  const std::vector<HostBatch> batches = make_batches(cfg.data, cfg.layers, cfg.loss);

  std::vector<LayerSpec> specs;
  for (const LayerCfg& L : cfg.layers) {
    LayerSpec s;
    s.type = L.type;
    if (L.type == kLinear) {
      s.a = L.in;
      s.b = L.out;
      s.bias = L.bias ? 1 : 0;
    } else if (L.type == kEmbedding) {
      s.a = L.vocab;
      s.b = L.dim;
      s.c = L.seq;
    } else if (L.type == kLayerNorm) {
      s.a = L.dim;
    }
    specs.push_back(s);
  }
  EngineConfig ec;
  ec.dtype = dtype;
  ec.loss = cfg.loss;
  ec.optim = cfg.plain ? 1 : 0;
  ec.micro_batches = cfg.micro_batches;
  ec.batch_rows = batches.front().rows;
  ec.plan_mode = cfg.per_tensor ? 2 : 0;
  ec.K = cfg.K;
  ec.T = cfg.T;
  ec.total_steps = cfg.steps;
  ec.prefetch = cfg.prefetch ? 1 : 0;
  ec.bandwidth_bytes_per_step = cfg.bandwidth;
  ec.hyper = cfg.hyper;
  ec.policy = cfg.policy;
  Engine eng(specs, ec, init.data(), stream);
  R.plan = eng.plan();
  R.cfg.K = R.plan.K();  // the per-tensor plan decides its own chunk count
  const int K = R.cfg.K, T = cfg.T;

  int64_t resident_param_bytes = 0;
  for (const TensorDesc& t : ts) resident_param_bytes += t.rows * t.cols * cfg.policy.param_bytes;

  // the engine reads host batches in its compute dtype: fp64 as generated, fp32 / bf16 rounded
  // to nearest (the bf16 through fp32, like the Python binding's torch conversion)
  auto narrow = [dtype](const std::vector<double>& v) {
    const size_t w = dtype == CFT_F64 ? 8 : dtype == CFT_F32 ? 4 : 2;
    std::vector<char> out(v.size() * w);
    for (size_t i = 0; i < v.size(); ++i) {
      if (w == 8) {
        std::memcpy(out.data() + 8 * i, &v[i], 8);
        continue;
      }
      const float f = static_cast<float>(v[i]);
      if (w == 4) {
        std::memcpy(out.data() + 4 * i, &f, 4);
        continue;
      }
      uint32_t u;
      std::memcpy(&u, &f, 4);
      const uint16_t h = std::isnan(f) ? uint16_t(0x7fc0)
                                       : uint16_t((u + 0x7fffu + ((u >> 16) & 1u)) >> 16);
      std::memcpy(out.data() + 2 * i, &h, 2);
    }
    return out;
  };
  std::vector<std::vector<char>> xs, ys;
  for (const HostBatch& hb : batches) {
    xs.push_back(narrow(hb.x));
    ys.push_back(narrow(hb.target));
  }

  host::RotationScheduler& sched = eng.scheduler();
  size_t cursor = 0;
  int64_t rotation_macs = 0;
  for (int64_t t = 0; t < cfg.steps; ++t) {
    const int active = eng.step_begin();
    for (int mb = 0; mb < cfg.micro_batches; ++mb) {
      const HostBatch& hb = batches[cursor];
      Batch b;
      b.x = hb.x.empty() ? nullptr : xs[cursor].data();
      b.tokens = hb.tokens.empty() ? nullptr : hb.tokens.data();
      b.target = hb.target.empty() ? nullptr : ys[cursor].data();
      cursor = (cursor + 1) % batches.size();
      b.labels = hb.labels.empty() ? nullptr : hb.labels.data();
      b.on_device = 0;
      eng.forward_backward(b, mb);
      rotation_macs += grad_macs(cfg.layers, ts, hb, &R.plan.chunks[active].slices);
      if (R.dense_macs == 0) R.dense_macs = grad_macs(cfg.layers, ts, hb, nullptr);
    }
    // sample_memory (accounting.cpp:141-153): the scheduler's view of this step
    MemorySample m{t, resident_param_bytes, sched.device_state_bytes(), cfg.activation_bytes,
                   sched.transfer_inflight_bytes(t)};
    if (active >= 0 && sched.is_resident(active))
      m.state += R.plan.chunk_elements(active) * cfg.policy.grad_bytes;
    R.memory.push_back(m);
    eng.step_end();
    // a rotation completes when the index counter wraps back to chunk 0 (trainer.cpp:77-86)
    if (t % T == T - 1 && sched.active_index_counter() % K == 0) {
      R.chunked_macs += rotation_macs;
      R.rotations += 1;
      rotation_macs = 0;
    }
  }
  eng.finish();

  int64_t n = 0;
  eng.trajectory(nullptr, nullptr, nullptr, nullptr, &n);
  std::vector<int64_t> steps(n);
  std::vector<int32_t> chunks(n);
  std::vector<double> loss(n), gsq(n);
  eng.trajectory(steps.data(), chunks.data(), loss.data(), gsq.data(), &n);
  R.initial_loss = n ? loss.front() : 0.0;
  R.final_loss = n ? loss.back() : 0.0;
  R.transfer_events = static_cast<int64_t>(sched.events().size());
  R.noop_loads = sched.noop_loads();

  // peak / mean / jitter / jitter bound / measured back-prop cost (accounting.cpp:22-131)
  if (R.memory.empty()) throw Error("empty memory trace");
  int64_t lo = R.memory.front().total(), hi = lo;
  double acc = 0.0;
  for (const MemorySample& m : R.memory) {
    lo = std::min(lo, m.total());
    hi = std::max(hi, m.total());
    acc += static_cast<double>(m.total());
  }
  R.peak = static_cast<double>(hi);
  R.mean = acc / static_cast<double>(R.memory.size());
  if (R.mean <= 0.0) throw Error("jitter: non-positive mean");
  R.jitter = (static_cast<double>(hi) - static_cast<double>(lo)) / R.mean;
  if (R.mean > 0.0) {
    const double avg = static_cast<double>(R.plan.total_mutable_bytes) / R.plan.K();
    double worst = 0.0;
    for (const auto& ch : R.plan.chunks)
      worst = std::max(worst, std::fabs(static_cast<double>(ch.byte_cost) - avg));
    R.jitter_bound = 2.0 * static_cast<double>(static_cast<int64_t>(std::ceil(worst))) / R.mean;
  }
  if (R.rotations < 1) throw Error("measured_bp_cost: no completed rotations");
  if (R.dense_macs < 1) throw Error("measured_bp_cost: dense reference count missing");
  R.bp_ratio = static_cast<double>(R.chunked_macs) /
               (static_cast<double>(R.rotations) * T * static_cast<double>(R.dense_macs));

  // the artifact bundle (runner.cpp:168-190)
  if (!cfg.out_dir.empty()) {
    namespace fs = std::filesystem;
    const fs::path out(cfg.out_dir);
    std::error_code ec2;
    fs::create_directories(out / "checkpoints", ec2);
    if (ec2) throw Error("run: cannot create output directory " + out.string());
    auto write = [](const fs::path& p, const std::string& text) {
      std::ofstream f(p, std::ios::binary);
      if (!f) throw Error("cannot open '" + p.string() + "' for writing");
      f << text;
      if (!f) throw Error("write failed for '" + p.string() + "'");
    };
    std::ostringstream mt;
    mt << "step,resident_param_bytes,active_state_bytes,activation_bytes,"
          "transfer_buffer_bytes,total\n";
    for (const MemorySample& m : R.memory)
      mt << m.step << ',' << m.params << ',' << m.state << ',' << m.activations << ','
         << m.transfers << ',' << m.total() << '\n';
    write(out / "memory_trace.csv", mt.str());
    eng.write_transfer_log_csv((out / "transfer_log.csv").string());
    eng.write_trajectory_csv((out / "trajectory.csv").string());
    write(out / "plan.json", eng.plan_json() + "\n");
    write(out / "effective_config.json", to_json(R.cfg).dump(2) + "\n");
    eng.write_checkpoints((out / "checkpoints").string());
    write(out / "summary.txt", summary_text(R));
  }
  return R;
}

// summary_text (runner.cpp:194-212)
std::string summary_text(const Result& R) {
  char hash[32];
  std::snprintf(hash, sizeof hash, "%016" PRIx64, host::plan_hash(R.plan));
  std::ostringstream os;
  os << "steps " << R.cfg.steps << '\n'
     << "chunks " << R.plan.K() << '\n'
     << "rotation_interval " << R.cfg.T << '\n'
     << "plan_hash " << hash << '\n'
     << "peak_bytes " << fmt(R.peak) << '\n'
     << "mean_total_bytes " << fmt(R.mean) << '\n'
     << "jitter " << fmt(R.jitter) << '\n'
     << "jitter_bound " << fmt(R.jitter_bound) << '\n'
     << "measured_bp_ratio " << fmt(R.bp_ratio) << '\n'
     << "noop_loads " << R.noop_loads << '\n'
     << "transfer_events " << R.transfer_events << '\n'
     << "initial_loss " << fmt(R.initial_loss) << '\n'
     << "final_loss " << fmt(R.final_loss) << '\n';
  return os.str();
}

// run_preset_checks (runner.cpp:214-260): the built-in expectation of every preset
int preset_checks(int dtype, cudaStream_t stream, std::ostream& os) {
  int failures = 0;
  auto check = [&](const std::string& name, const std::string& what, bool ok) {
    os << "check " << name << ": " << what << (ok ? " ... ok" : " ... FAIL") << '\n';
    failures += ok ? 0 : 1;
  };
  auto run = [&](const char* name) { return run_experiment(make_preset(name), dtype, stream); };
  {
    const Result r = run("quadratic-k2");
    check("quadratic-k2", "jitter " + fmt(r.jitter) + " == 0", r.jitter == 0.0);
    check("quadratic-k2", "measured_bp_ratio " + fmt(r.bp_ratio) + " == 1", r.bp_ratio == 1.0);
  }
  {
    const Result r = run("mlp-imbalanced-layers");
    check("mlp-imbalanced-layers", "jitter " + fmt(r.jitter) + " <= 0.02", r.jitter <= 0.02);
  }
  {
    const Result r = run("mlp-imbalanced-layers-identity");
    check("mlp-imbalanced-layers-identity", "jitter " + fmt(r.jitter) + " >= 0.2",
          r.jitter >= 0.2);
  }
  {
    const Result r = run("dense-reduction");
    check("dense-reduction", "measured_bp_ratio " + fmt(r.bp_ratio) + " == 1", r.bp_ratio == 1.0);
    check("dense-reduction", "jitter " + fmt(r.jitter) + " == 0", r.jitter == 0.0);
  }
  {
    const Result r = run("classification-sanity");
    check("classification-sanity",
          "final_loss " + fmt(r.final_loss) + " < initial " + fmt(r.initial_loss),
          std::isfinite(r.final_loss) && r.final_loss < r.initial_loss);
  }
  return failures;
}

}  // namespace cft::run

// ---- C ABI (include/chunkft_b200.h, "experiments") ------------------------------------------
struct cft_experiment {
  cft::run::Experiment cfg;
};

namespace {
// the library's text-out convention (cft_engine_plan_json): *needed = length + 1, the copy is
// truncated to cap - 1 characters and always terminated
void put_text(const std::string& s, char* buf, int64_t cap, int64_t* needed) {
  if (needed) *needed = static_cast<int64_t>(s.size()) + 1;
  if (buf && cap > 0) {
    const size_t n = std::min(s.size(), static_cast<size_t>(cap - 1));
    std::memcpy(buf, s.data(), n);
    buf[n] = '\0';
  }
}
}  // namespace

extern "C" {

int cft_preset_names(char* buf, int64_t cap, int64_t* needed) {
  return cft::guarded([&] {
    std::string s;
    for (const auto& n : cft::run::preset_names()) s += n + "\n";
    put_text(s, buf, cap, needed);
  });
}

int cft_experiment_preset(const char* name, cft_experiment** out) {
  return cft::guarded([&] {
    CFT_CHECK(name && out, "experiment: null argument");
    *out = new cft_experiment{cft::run::make_preset(name)};
  });
}

int cft_experiment_parse(const char* json_text, cft_experiment** out) {
  return cft::guarded([&] {
    CFT_CHECK(json_text && out, "experiment: null argument");
    nlohmann::json doc;
    try {
      doc = nlohmann::json::parse(json_text);
    } catch (const nlohmann::json::parse_error& e) {
      throw cft::Error(std::string("config: ") + e.what());
    }
    *out = new cft_experiment{cft::run::parse_config(doc)};
  });
}

int cft_experiment_load(const char* path, cft_experiment** out) {
  return cft::guarded([&] {
    CFT_CHECK(path && out, "experiment: null argument");
    std::ifstream in(path);
    if (!in) throw cft::Error(std::string("config: cannot open ") + path);
    nlohmann::json doc;
    try {
      doc = nlohmann::json::parse(in);
    } catch (const nlohmann::json::parse_error& e) {
      throw cft::Error(std::string("config: ") + path + ": " + e.what());
    }
    *out = new cft_experiment{cft::run::parse_config(doc)};
  });
}

void cft_experiment_destroy(cft_experiment* e) { delete e; }

int cft_experiment_set_out_dir(cft_experiment* e, const char* dir) {
  return cft::guarded([&] { e->cfg.out_dir = dir ? dir : ""; });
}

int cft_experiment_set_seed(cft_experiment* e, uint64_t seed) {
  return cft::guarded([&] { e->cfg.seed = seed; });
}

int cft_experiment_to_json(const cft_experiment* e, char* buf, int64_t cap, int64_t* needed) {
  return cft::guarded([&] { put_text(cft::run::to_json(e->cfg).dump(2), buf, cap, needed); });
}

int cft_experiment_run(const cft_experiment* e, cft_dtype dtype, cft_stream_t stream,
                       char* summary, int64_t cap, int64_t* needed) {
  return cft::guarded([&] {
    const cft::run::Result r =
        cft::run::run_experiment(e->cfg, dtype, static_cast<cudaStream_t>(stream));
    put_text(cft::run::summary_text(r), summary, cap, needed);
  });
}

int cft_run_preset_checks(cft_dtype dtype, cft_stream_t stream, char* report, int64_t cap,
                          int64_t* needed, int32_t* failures) {
  return cft::guarded([&] {
    std::ostringstream os;
    const int f = cft::run::preset_checks(dtype, static_cast<cudaStream_t>(stream), os);
    if (failures) *failures = f;
    put_text(os.str(), report, cap, needed);
  });
}

}  // extern "C"
