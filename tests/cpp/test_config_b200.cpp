// CPU test of include/helixsim/config_b200.hpp (the reference's L0/L1 surface
// in C++): validate_config against the reference's own verdicts
// (tests/golden/validate_config.json, generated from /root/reference by
// oracle/gen_config_golden.cpp), the JSON schema and its diagnostics, presets,
// and the lowering onto the C ABI. Environment: HX_GOLDEN_DIR (tests/golden),
// HX_REF_PRESETS (optional: the reference's presets/ directory).
#define DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
#include <doctest.h>

#include <cstdlib>
#include <fstream>
#include <string>

#include "helixsim/config_b200.hpp"

using namespace helixsim;
using nlohmann::json;

namespace {
const std::string golden_dir = std::getenv("HX_GOLDEN_DIR") ? std::getenv("HX_GOLDEN_DIR") : "tests/golden";
const std::string presets_dir = std::getenv("HX_REF_PRESETS") ? std::getenv("HX_REF_PRESETS") : "";

ModelSpec golden_model(const std::string& name) {  // the four models gen_config_golden.cpp enumerates
  ModelSpec m = llama405b_like();
  m.name = name;
  m.layers = 2;
  if (name == "mla") {
    m.kv_heads = 1;
    m.attention_kind = AttentionKind::MLA;
    m.kv_latent_dim = 288;
  } else if (name == "moe") {
    m.moe = MoESpec{256, 8, 2048, 2048};
  } else if (name == "moe_odd") {
    m.moe = MoESpec{6, 2, 24, 0};
  }
  return m;
}

template <class F>
std::string config_error(F&& f) {
  try {
    f();
  } catch (const ConfigError& e) {
    return e.what();
  }
  return "";
}
}  // namespace

TEST_CASE("validate_config matches the reference's verdicts and rules") {
  std::ifstream in(golden_dir + "/validate_config.json");
  REQUIRE(in.good());
  const json g = json::parse(in);
  i64 n = 0;
  for (const json& row : g.at("rows")) {
    HardwareSpec hw;
    hw.max_gpus = row[1].get<i64>();
    ParallelismConfig c;
    c.strategy = *strategy_from_name(row[2].get<std::string>());
    c.tpa = row[3].get<i64>();
    c.kvp = row[4].get<i64>();
    c.tpf = row[5].get<i64>();
    c.ep = row[6].get<i64>();
    c.pp = row[7].get<i64>();
    const Validity v = validate_config(c, golden_model(row[0].get<std::string>()), hw);
    CHECK(static_cast<bool>(v) == (row[9].get<int>() != 0));
    CHECK(v.rule == row[10].get<std::string>());
    CHECK(c.total_gpus() == row[8].get<i64>());
    ++n;
  }
  CHECK(n == 3600);  // every row of the golden file
}

TEST_CASE("JSON round trips and schema diagnostics") {
  for (const std::string& name : model_preset_names()) {
    const ModelSpec m = load_model(name);
    const ModelSpec r = model_from_json(to_json(m));
    CHECK(to_json(r) == to_json(m));
  }
  for (const std::string& name : hardware_preset_names()) CHECK(to_json(hardware_from_json(to_json(load_hardware(name)))) == to_json(load_hardware(name)));
  json m = to_json(llama405b_like());
  m["extra"] = 1;
  CHECK(config_error([&] { model_from_json(m); }) == "model config: unknown key 'extra'");
  m = to_json(llama405b_like());
  m.erase("layers");
  CHECK(config_error([&] { model_from_json(m); }) == "model config: missing field 'layers'");
  m = to_json(llama405b_like());
  m["attention"] = "dense";
  CHECK(config_error([&] { model_from_json(m); }) == "model config: field 'attention' must be \"gqa\" or \"mla\"");
  json h = to_json(gb200_like());
  h["max_gpus"] = 1.5;
  CHECK(config_error([&] { hardware_from_json(h); }) == "hardware config: field 'max_gpus' must be an integer");
  ParallelismConfig c{Strategy::Helix, 1, 8, 8, 1, 1};
  CHECK(c.to_string() == "helix(tpa=1,kvp=8,tpf=8,ep=1,pp=1)");
  json pj = to_json(c);
  pj["strategy"] = "bogus";
  CHECK(config_error([&] { parallelism_from_json(pj); }) ==
        "parallelism config: field 'strategy' has unknown value 'bogus'");
  CHECK(config_error([&] { load_model("/nonexistent.json"); }) == "cannot open config file: /nonexistent.json");
  CHECK_THROWS_AS(load_model("no-such-preset"), ConfigError);
}

TEST_CASE("the reference's own preset files load to the same specs") {
  if (presets_dir.empty()) return;  // /root/reference is absent on the GPU box
  CHECK(to_json(load_model(presets_dir + "/llama405b-like.json")) == to_json(llama405b_like()));
  CHECK(to_json(load_model(presets_dir + "/deepseek-r1-like.json")) == to_json(deepseek_r1_like()));
  CHECK(to_json(load_hardware(presets_dir + "/gb200-like.json")) == to_json(gb200_like()));
}

TEST_CASE("helix layouts lower onto the C ABI; invalid ones are rejected first") {
  const HardwareSpec hw = b200_measured();
  const HxConfig x = to_hx_config(deepseek_r1_like(), {Strategy::Helix, 1, 8, 1, 8, 1}, hw, 4096, HX_POOL_NCCL, 3);
  CHECK(x.model.kv_latent == 288);
  CHECK(x.model.n_experts == 256);
  CHECK(x.model.ffn == 2048);  // the shared expert
  CHECK(x.par.kvp == 8);
  CHECK(x.par.ep == 8);
  CHECK(x.par.rank == 3);
  std::string msg;
  try {
    to_hx_config(llama405b_like(), {Strategy::Helix, 1, 8, 4, 1, 1}, hw);
  } catch (const std::invalid_argument& e) {
    msg = e.what();
  }
  CHECK(msg == "invalid config helix(tpa=1,kvp=8,tpf=4,ep=1,pp=1): helix re-provisions one pool: kvp*tpa must "
               "equal tpf*ep");
  CHECK_THROWS_AS(to_hx_config(llama405b_like(), {Strategy::TP, 8, 1, 8, 1, 1}, hw), std::invalid_argument);
}
