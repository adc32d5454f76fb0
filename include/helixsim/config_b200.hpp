// helixsim/config_b200.hpp -- the reference's L0/L1 configuration surface for
// the B200 decode path: model / hardware / workload / parallelism specs, their
// validation rules and diagnostics, the JSON schema and presets, and the
// Helix-pool validity check (reference: proj/include/helixsim/types.hpp:1-110,
// proj/src/types.cpp:1-141, proj/include/helixsim/presets.hpp,
// proj/src/presets.cpp:11-252). Header-only; JSON via nlohmann/json (the
// reference's own dependency: `#include <json.hpp>` on the same include path).
//
// The names, fields, JSON keys, error types (std::invalid_argument for spec
// validation, ConfigError for configuration files) and message texts are the
// reference's, so a caller of types.hpp / presets.hpp can switch headers.
// to_hx_config() lowers a validated Helix layout onto the C-ABI structs of
// include/helix_b200.h (one engine = one rank of the tpa x kvp pool).
#pragma once

#include <json.hpp>

#include <cstdint>
#include <fstream>
#include <optional>
#include <set>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "../helix_b200.h"

namespace helixsim {

using i64 = std::int64_t;

constexpr i64 ceil_div(i64 a, i64 b) { return (a + b - 1) / b; }

struct ConfigError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

namespace cfg_detail {
inline void require(bool ok, const char* msg) {
  if (!ok) throw std::invalid_argument(msg);
}
}  // namespace cfg_detail

// ---------------------------------------------------------------- specs (types.hpp:13-80)
enum class AttentionKind { GQA, MLA };

struct MoESpec {
  i64 total_experts = 0;
  i64 active_experts_per_token = 0;
  i64 expert_ffn_dim = 0;
  i64 shared_expert_ffn_dim = 0;  // 0: no shared expert
};

struct ModelSpec {
  std::string name;
  i64 layers = 0, hidden_dim = 0, query_heads = 0, kv_heads = 0, head_size = 0, ffn_dim = 0;
  i64 ffn_gate_factor = 3;
  AttentionKind attention_kind = AttentionKind::GQA;
  i64 kv_latent_dim = 0;  // MLA: latent width per token half (the cache is one KV head of this width)
  std::optional<MoESpec> moe;

  i64 effective_kv_heads() const { return attention_kind == AttentionKind::MLA ? 1 : kv_heads; }
  i64 kv_head_size() const {
    return (attention_kind == AttentionKind::MLA && kv_latent_dim > 0) ? kv_latent_dim : head_size;
  }
  void validate() const {
    using cfg_detail::require;
    require(layers >= 1, "layers must be >= 1");
    require(hidden_dim >= 1, "hidden_dim must be >= 1");
    require(query_heads >= 1, "query_heads must be >= 1");
    require(kv_heads >= 1, "kv_heads must be >= 1");
    require(head_size >= 1, "head_size must be >= 1");
    require(ffn_dim >= 1, "ffn_dim must be >= 1");
    require(ffn_gate_factor >= 1, "ffn_gate_factor must be >= 1");
    require(hidden_dim == query_heads * head_size, "hidden_dim must equal query_heads * head_size");
    if (attention_kind == AttentionKind::GQA) {
      require(query_heads % kv_heads == 0, "query_heads must be a multiple of kv_heads");
      require(kv_latent_dim == 0, "kv_latent_dim is only meaningful for MLA");
    } else {
      require(kv_heads == 1, "MLA keeps a single latent KV head");
      require(kv_latent_dim >= 0, "kv_latent_dim must be >= 0");
    }
    if (!moe) return;
    require(moe->total_experts >= 1, "moe.total_experts must be >= 1");
    require(moe->active_experts_per_token >= 1, "moe.active_experts_per_token must be >= 1");
    require(moe->active_experts_per_token <= moe->total_experts,
            "moe.active_experts_per_token must not exceed moe.total_experts");
    require(moe->expert_ffn_dim >= 1, "moe.expert_ffn_dim must be >= 1");
    require(moe->shared_expert_ffn_dim >= 0, "moe.shared_expert_ffn_dim must be >= 0");
  }
};

struct HardwareSpec {
  std::string name;
  double mem_bw = 8.0e12;              // bytes/s
  double compute_throughput = 5.0e15;  // FLOP/s at the serving precision
  double link_bw = 9.0e11;             // bytes/s per direction
  double link_latency = 1.0e-7;        // s per hop
  i64 max_gpus = 64;
  double bytes_per_param = 0.5;
  double dram_capacity = 192.0e9;
  void validate() const {
    using cfg_detail::require;
    require(mem_bw > 0, "mem_bw must be > 0");
    require(compute_throughput > 0, "compute_throughput must be > 0");
    require(link_bw > 0, "link_bw must be > 0");
    require(link_latency >= 0, "link_latency must be >= 0");
    require(max_gpus >= 1, "max_gpus must be >= 1");
    require(bytes_per_param > 0, "bytes_per_param must be > 0");
    require(dram_capacity > 0, "dram_capacity must be > 0");
  }
};

struct WorkloadSpec {
  i64 batch = 1;
  i64 kv_seq_len = 1;
  i64 decode_steps = 1;
  void validate() const {
    using cfg_detail::require;
    require(batch >= 1, "batch must be >= 1");
    require(kv_seq_len >= 1, "kv_seq_len must be >= 1");
    require(decode_steps >= 1, "decode_steps must be >= 1");
  }
};

// ---------------------------------------------------------------- parallelism (types.hpp:82-110)
enum class Strategy { Helix, TP, TP_PP, EP_DPAttention, MedhaKVP };

inline const char* strategy_name(Strategy s) {
  constexpr const char* names[] = {"helix", "tp", "tp_pp", "ep_dp", "medha_kvp"};
  const int i = static_cast<int>(s);
  return (i >= 0 && i < 5) ? names[i] : "?";
}
inline std::optional<Strategy> strategy_from_name(const std::string& s) {
  for (int i = 0; i < 5; ++i)
    if (s == strategy_name(static_cast<Strategy>(i))) return static_cast<Strategy>(i);
  return std::nullopt;
}

struct ParallelismConfig {
  Strategy strategy = Strategy::TP;
  i64 tpa = 1, kvp = 1, tpf = 1, ep = 1, pp = 1;
  // GPUs of one pipeline stage: the attention grid, except data-parallel
  // attention, whose stage is the FFN grid it feeds.
  i64 stage_pool() const { return strategy == Strategy::EP_DPAttention ? tpf * ep : kvp * tpa; }
  i64 total_gpus() const { return stage_pool() * pp; }
  std::string to_string() const {
    std::ostringstream o;
    o << strategy_name(strategy) << "(tpa=" << tpa << ",kvp=" << kvp << ",tpf=" << tpf << ",ep=" << ep
      << ",pp=" << pp << ")";
    return o.str();
  }
};

struct Validity {
  bool ok = true;
  std::string rule;  // the first broken rule
  explicit operator bool() const { return ok; }
};

// The reference's layout rules (types.cpp:86-141), first broken rule wins.
inline Validity validate_config(const ParallelismConfig& c, const ModelSpec& m, const HardwareSpec& hw) {
  auto bad = [](const char* rule) { return Validity{false, rule}; };
  if (c.tpa < 1 || c.kvp < 1 || c.tpf < 1 || c.ep < 1 || c.pp < 1) return bad("all parallelism widths must be >= 1");
  if (c.total_gpus() > hw.max_gpus) return bad("total GPUs exceed max_gpus");
  switch (c.strategy) {
    case Strategy::Helix:
      if (c.pp != 1) return bad("helix runs as a single pipeline stage");
      if (c.tpa > m.effective_kv_heads()) return bad("helix requires tpa <= effective KV heads");
      if (c.kvp * c.tpa != c.tpf * c.ep) return bad("helix re-provisions one pool: kvp*tpa must equal tpf*ep");
      break;
    case Strategy::TP:
    case Strategy::TP_PP:
      if (c.strategy == Strategy::TP && c.pp != 1) return bad("tp has no pipeline stages");
      if (c.kvp != 1) return bad("tp keeps the whole sequence per GPU (kvp=1)");
      if (c.ep != 1) return bad("tp shards experts with tensor parallelism (ep=1)");
      if (c.tpf != c.tpa) return bad("tp ties attention and FFN widths");
      break;
    case Strategy::EP_DPAttention:
      if (c.tpa != 1 || c.kvp != 1) return bad("ep_dp replicates attention (tpa=1, kvp=1)");
      break;
    case Strategy::MedhaKVP:
      if (c.tpf != c.tpa) return bad("medha_kvp keeps the FFN on the tpa group");
      if (c.ep != 1) return bad("medha_kvp does not shard experts (ep=1)");
      break;
  }
  if (m.query_heads % c.tpa != 0) return bad("tpa must divide query_heads");
  const bool kv_sharded = c.strategy == Strategy::Helix || c.strategy == Strategy::MedhaKVP;
  if (kv_sharded && m.hidden_dim % (c.kvp * c.tpa) != 0) return bad("kvp*tpa must divide hidden_dim");
  if (m.moe) {
    if (m.moe->total_experts % c.ep != 0) return bad("ep must divide total_experts");
    if (m.moe->expert_ffn_dim % c.tpf != 0) return bad("tpf must divide expert_ffn_dim");
    if (m.moe->shared_expert_ffn_dim > 0 && m.moe->shared_expert_ffn_dim % c.tpf != 0)
      return bad("tpf must divide shared_expert_ffn_dim");
  } else {
    if (c.ep != 1) return bad("expert parallelism needs an MoE model");
    if (m.ffn_dim % c.tpf != 0) return bad("tpf must divide ffn_dim");
  }
  return {};
}

// ---------------------------------------------------------------- presets (presets.cpp:11-56)
inline ModelSpec llama405b_like() {
  ModelSpec m;
  m.name = "llama405b-like";
  m.layers = 126;
  m.hidden_dim = 16384;
  m.query_heads = 128;
  m.kv_heads = 8;
  m.head_size = 128;
  m.ffn_dim = 65536;
  return m;
}
inline ModelSpec deepseek_r1_like() {
  ModelSpec m;
  m.name = "deepseek-r1-like";
  m.layers = 61;
  m.hidden_dim = 16384;
  m.query_heads = 128;
  m.kv_heads = 1;
  m.head_size = 128;
  m.ffn_dim = 18432;
  m.attention_kind = AttentionKind::MLA;
  m.kv_latent_dim = 288;
  m.moe = MoESpec{256, 8, 2048, 2048};
  return m;
}
// Builder presets (the reference ships no small model)
inline ModelSpec llama3_8b_like() {
  ModelSpec m;
  m.name = "llama3-8b-like";
  m.layers = 32;
  m.hidden_dim = 4096;
  m.query_heads = 32;
  m.kv_heads = 8;
  m.head_size = 128;
  m.ffn_dim = 14336;
  return m;
}
inline ModelSpec tiny_gqa() {
  ModelSpec m;
  m.name = "tiny-gqa";
  m.layers = 2;
  m.hidden_dim = 64;
  m.query_heads = 8;
  m.kv_heads = 4;
  m.head_size = 8;
  m.ffn_dim = 128;
  return m;
}
inline HardwareSpec gb200_like() {
  HardwareSpec hw;
  hw.name = "gb200-like";
  return hw;
}
// This pool's B200 at the engine's storage precision (bf16): measured copy
// bandwidth and sustained cuBLAS bf16 (MEASURED_PEAKS.json), NVLink 5, 180 GB.
inline HardwareSpec b200_measured() {
  HardwareSpec hw;
  hw.name = "b200-measured";
  hw.mem_bw = 6.5562e12;
  hw.compute_throughput = 1.393e15;
  hw.max_gpus = 8;
  hw.bytes_per_param = 2.0;
  hw.dram_capacity = 180e9;
  return hw;
}
inline std::vector<std::string> model_preset_names() {
  return {"llama405b-like", "deepseek-r1-like", "llama3-8b-like", "tiny-gqa"};
}
inline std::vector<std::string> hardware_preset_names() { return {"gb200-like", "b200-measured"}; }

// ---------------------------------------------------------------- JSON schema (presets.cpp:58-252)
namespace cfg_detail {
using nlohmann::json;
[[noreturn]] inline void fail(const std::string& msg) { throw ConfigError(msg); }
inline void only_keys(const json& j, std::initializer_list<const char*> keys, const std::string& where) {
  if (!j.is_object()) fail(where + ": expected a JSON object");
  const std::set<std::string> ok(keys.begin(), keys.end());
  for (auto it = j.begin(); it != j.end(); ++it)
    if (!ok.count(it.key())) fail(where + ": unknown key '" + it.key() + "'");
}
inline const json& get(const json& j, const char* key, const std::string& where) {
  if (!j.is_object()) fail(where + ": expected a JSON object");
  auto it = j.find(key);
  if (it == j.end()) fail(where + ": missing field '" + key + "'");
  return *it;
}
inline i64 get_int(const json& j, const char* key, const std::string& where) {
  const json& v = get(j, key, where);
  if (!v.is_number_integer()) fail(where + ": field '" + key + "' must be an integer");
  return v.get<i64>();
}
inline double get_num(const json& j, const char* key, const std::string& where) {
  const json& v = get(j, key, where);
  if (!v.is_number()) fail(where + ": field '" + key + "' must be a number");
  return v.get<double>();
}
inline std::string get_str(const json& j, const char* key, const std::string& where) {
  const json& v = get(j, key, where);
  if (!v.is_string()) fail(where + ": field '" + key + "' must be a string");
  return v.get<std::string>();
}
inline json read_file(const std::string& path) {
  std::ifstream in(path, std::ios::binary);
  if (!in) fail("cannot open config file: " + path);
  std::stringstream s;
  s << in.rdbuf();
  json j = json::parse(s.str(), nullptr, false);
  if (j.is_discarded()) fail("malformed JSON in " + path);
  return j;
}
template <class Spec>
Spec validated(Spec s, const std::string& path) {
  try {
    s.validate();
  } catch (const std::invalid_argument& e) {
    fail(path + ": " + e.what());
  }
  return s;
}
}  // namespace cfg_detail

inline nlohmann::json to_json(const ModelSpec& m) {
  nlohmann::json j = {{"name", m.name},
                      {"layers", m.layers},
                      {"hidden_dim", m.hidden_dim},
                      {"query_heads", m.query_heads},
                      {"kv_heads", m.kv_heads},
                      {"head_size", m.head_size},
                      {"ffn_dim", m.ffn_dim},
                      {"ffn_gate_factor", m.ffn_gate_factor},
                      {"attention", m.attention_kind == AttentionKind::MLA ? "mla" : "gqa"},
                      {"kv_latent_dim", m.kv_latent_dim}};
  if (m.moe)
    j["moe"] = {{"total_experts", m.moe->total_experts},
                {"active_experts_per_token", m.moe->active_experts_per_token},
                {"expert_ffn_dim", m.moe->expert_ffn_dim},
                {"shared_expert_ffn_dim", m.moe->shared_expert_ffn_dim}};
  return j;
}
inline nlohmann::json to_json(const HardwareSpec& h) {
  return {{"name", h.name},
          {"mem_bw_bytes_per_s", h.mem_bw},
          {"compute_flops", h.compute_throughput},
          {"link_bw_bytes_per_s", h.link_bw},
          {"link_latency_s", h.link_latency},
          {"max_gpus", h.max_gpus},
          {"bytes_per_param", h.bytes_per_param},
          {"dram_capacity_bytes", h.dram_capacity}};
}
inline nlohmann::json to_json(const WorkloadSpec& w) {
  return {{"batch", w.batch}, {"kv_seq_len", w.kv_seq_len}, {"decode_steps", w.decode_steps}};
}
inline nlohmann::json to_json(const ParallelismConfig& c) {
  return {{"strategy", strategy_name(c.strategy)}, {"tpa", c.tpa}, {"kvp", c.kvp},
          {"tpf", c.tpf},                          {"ep", c.ep},   {"pp", c.pp}};
}

inline ModelSpec model_from_json(const nlohmann::json& j) {
  using namespace cfg_detail;
  const std::string w = "model config";
  only_keys(j, {"name", "layers", "hidden_dim", "query_heads", "kv_heads", "head_size", "ffn_dim",
                "ffn_gate_factor", "attention", "kv_latent_dim", "moe"},
            w);
  ModelSpec m;
  m.name = get_str(j, "name", w);
  m.layers = get_int(j, "layers", w);
  m.hidden_dim = get_int(j, "hidden_dim", w);
  m.query_heads = get_int(j, "query_heads", w);
  m.kv_heads = get_int(j, "kv_heads", w);
  m.head_size = get_int(j, "head_size", w);
  m.ffn_dim = get_int(j, "ffn_dim", w);
  m.ffn_gate_factor = get_int(j, "ffn_gate_factor", w);
  const std::string kind = get_str(j, "attention", w);
  if (kind != "gqa" && kind != "mla") fail(w + ": field 'attention' must be \"gqa\" or \"mla\"");
  m.attention_kind = kind == "mla" ? AttentionKind::MLA : AttentionKind::GQA;
  m.kv_latent_dim = get_int(j, "kv_latent_dim", w);
  if (j.contains("moe")) {
    const nlohmann::json& mj = j.at("moe");
    const std::string mw = "model config: moe";
    only_keys(mj, {"total_experts", "active_experts_per_token", "expert_ffn_dim", "shared_expert_ffn_dim"}, mw);
    m.moe = MoESpec{get_int(mj, "total_experts", mw), get_int(mj, "active_experts_per_token", mw),
                    get_int(mj, "expert_ffn_dim", mw), get_int(mj, "shared_expert_ffn_dim", mw)};
  }
  return m;
}
inline HardwareSpec hardware_from_json(const nlohmann::json& j) {
  using namespace cfg_detail;
  const std::string w = "hardware config";
  only_keys(j, {"name", "mem_bw_bytes_per_s", "compute_flops", "link_bw_bytes_per_s", "link_latency_s", "max_gpus",
                "bytes_per_param", "dram_capacity_bytes"},
            w);
  HardwareSpec h;
  h.name = get_str(j, "name", w);
  h.mem_bw = get_num(j, "mem_bw_bytes_per_s", w);
  h.compute_throughput = get_num(j, "compute_flops", w);
  h.link_bw = get_num(j, "link_bw_bytes_per_s", w);
  h.link_latency = get_num(j, "link_latency_s", w);
  h.max_gpus = get_int(j, "max_gpus", w);
  h.bytes_per_param = get_num(j, "bytes_per_param", w);
  h.dram_capacity = get_num(j, "dram_capacity_bytes", w);
  return h;
}
inline WorkloadSpec workload_from_json(const nlohmann::json& j) {
  using namespace cfg_detail;
  const std::string w = "workload config";
  only_keys(j, {"batch", "kv_seq_len", "decode_steps"}, w);
  WorkloadSpec s;
  s.batch = get_int(j, "batch", w);
  s.kv_seq_len = static_cast<i64>(get_num(j, "kv_seq_len", w));  // "1e6" is accepted, as in the reference
  s.decode_steps = get_int(j, "decode_steps", w);
  return s;
}
inline ParallelismConfig parallelism_from_json(const nlohmann::json& j) {
  using namespace cfg_detail;
  const std::string w = "parallelism config";
  only_keys(j, {"strategy", "tpa", "kvp", "tpf", "ep", "pp"}, w);
  const std::string s = get_str(j, "strategy", w);
  const auto strat = strategy_from_name(s);
  if (!strat) fail(w + ": field 'strategy' has unknown value '" + s + "'");
  ParallelismConfig c;
  c.strategy = *strat;
  c.tpa = get_int(j, "tpa", w);
  c.kvp = get_int(j, "kvp", w);
  c.tpf = get_int(j, "tpf", w);
  c.ep = get_int(j, "ep", w);
  c.pp = get_int(j, "pp", w);
  return c;
}

// Preset name, else a JSON file path; the result is validated (presets.cpp:246-260).
inline ModelSpec load_model(const std::string& name_or_path) {
  if (name_or_path == "llama405b-like") return llama405b_like();
  if (name_or_path == "deepseek-r1-like") return deepseek_r1_like();
  if (name_or_path == "llama3-8b-like") return llama3_8b_like();
  if (name_or_path == "tiny-gqa") return tiny_gqa();
  return cfg_detail::validated(model_from_json(cfg_detail::read_file(name_or_path)), name_or_path);
}
inline HardwareSpec load_hardware(const std::string& name_or_path) {
  if (name_or_path == "gb200-like") return gb200_like();
  if (name_or_path == "b200-measured") return b200_measured();
  return cfg_detail::validated(hardware_from_json(cfg_detail::read_file(name_or_path)), name_or_path);
}
inline WorkloadSpec load_workload(const std::string& path) {
  return cfg_detail::validated(workload_from_json(cfg_detail::read_file(path)), path);
}
inline ParallelismConfig load_parallelism(const std::string& path) {
  return parallelism_from_json(cfg_detail::read_file(path));
}

// ---------------------------------------------------------------- lowering onto the C ABI
// One engine of the Helix pool described by (model, cfg): rank `rank` of
// tpa x kvp (pool = HX_POOL_NCCL / HX_POOL_LOOPBACK) or the whole pool on one
// device (HX_POOL_LOCAL). Throws std::invalid_argument with the reference's
// rule when the layout is not a valid Helix configuration.
struct HxConfig {
  hx_model_config model{};
  hx_parallel_config par{};
};
inline HxConfig to_hx_config(const ModelSpec& m, const ParallelismConfig& c, const HardwareSpec& hw,
                             i64 vocab = 128256, int pool = HX_POOL_LOCAL, int rank = 0) {
  m.validate();
  if (const Validity v = validate_config(c, m, hw); !v)
    throw std::invalid_argument("invalid config " + c.to_string() + ": " + v.rule);
  if (c.strategy != Strategy::Helix) throw std::invalid_argument("the B200 decode engine runs the helix strategy");
  HxConfig out;
  out.model.hidden = m.hidden_dim;
  out.model.query_heads = m.query_heads;
  out.model.kv_heads = m.kv_heads;
  out.model.head_size = m.head_size;
  out.model.ffn = m.moe ? m.moe->shared_expert_ffn_dim : m.ffn_dim;
  out.model.layers = m.layers;
  out.model.vocab = vocab;
  if (m.moe) {
    out.model.n_experts = m.moe->total_experts;
    out.model.top_k = m.moe->active_experts_per_token;
    out.model.expert_ffn = m.moe->expert_ffn_dim;
  }
  if (m.attention_kind == AttentionKind::MLA) out.model.kv_latent = m.kv_latent_dim;
  out.par.tpa = c.tpa;
  out.par.kvp = c.kvp;
  out.par.chunk_size = 16;
  out.par.distributed = pool;
  out.par.rank = rank;
  out.par.ep = c.ep;
  return out;
}

}  // namespace helixsim
