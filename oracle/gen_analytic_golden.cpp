// TEST INFRASTRUCTURE ONLY -- golden values of the reference's analytic layer
// (roofline.hpp:17-48, comm.hpp:28-69, overlap.hpp:37-69, latency.cpp:45-250),
// computed by the REFERENCE'S OWN library (oracle/_ref/libhelixsim_core.a,
// built from /root/reference/proj/src by oracle/Makefile). Pins the product's
// restatement (paper_2507_07120_b200/analytic.py, used by bench.py and
// tools/) in tests/test_analytic.py.
//
//   gen_analytic_golden > tests/golden/analytic.json
#include <cstdio>
#include <string>
#include <vector>

#include "helixsim/comm.hpp"
#include "helixsim/latency.hpp"
#include "helixsim/overlap.hpp"
#include "helixsim/presets.hpp"
#include "helixsim/roofline.hpp"

using namespace helixsim;

namespace {

bool first = true;
void open_row() {
  std::printf(first ? "\n" : ",\n");
  first = false;
}

ModelSpec model(const std::string& n) {
  if (n == "llama3-8b-like") {
    ModelSpec m;
    m.name = n;
    m.layers = 32;
    m.hidden_dim = 4096;
    m.query_heads = 32;
    m.kv_heads = 8;
    m.head_size = 128;
    m.ffn_dim = 14336;
    return m;
  }
  return load_model(n);
}

HardwareSpec hardware(const std::string& n) {
  if (n == "b200-measured") {  // paper_2507_07120_b200/model.py HARDWARE_PRESETS
    HardwareSpec hw;
    hw.name = n;
    hw.mem_bw = 6.5562e12;
    hw.compute_throughput = 1.393e15;
    hw.max_gpus = 8;
    hw.bytes_per_param = 2.0;
    hw.dram_capacity = 180e9;
    return hw;
  }
  return load_hardware(n);
}

const char* strat(Strategy s) { return strategy_name(s); }

void roofline_row(const std::string& m, const std::string& h, i64 batch, i64 s, i64 tpa, i64 kvp, i64 tpf) {
  WorkloadSpec w;
  w.batch = batch;
  w.kv_seq_len = s;
  const ModelSpec mm = model(m);
  const HardwareSpec hw = hardware(h);
  open_row();
  std::printf(
      "{\"fn\": \"roofline\", \"model\": \"%s\", \"hw\": \"%s\", \"batch\": %lld, \"seq\": %lld, \"tpa\": %lld, "
      "\"kvp\": %lld, \"tpf\": %lld, \"kv_read_time\": %.17g, \"weight_read_time\": %.17g}",
      m.c_str(), h.c_str(), (long long)batch, (long long)s, (long long)tpa, (long long)kvp, (long long)tpf,
      kv_read_time(mm, w, tpa, kvp, hw), weight_read_time(mm, tpa, tpf, hw));
}

void a2a_row(const std::string& m, const std::string& h, i64 batch, i64 kvp, i64 tpa) {
  const ModelSpec mm = model(m);
  const HardwareSpec hw = hardware(h);
  open_row();
  std::printf(
      "{\"fn\": \"a2a\", \"model\": \"%s\", \"hw\": \"%s\", \"batch\": %lld, \"kvp\": %lld, \"tpa\": %lld, "
      "\"per_destination\": %.17g, \"total_send\": %.17g}",
      m.c_str(), h.c_str(), (long long)batch, (long long)kvp, (long long)tpa,
      a2a_payload_per_destination(mm, batch, kvp, tpa, hw), a2a_total_send_bytes(mm, batch, kvp, tpa, hw));
}

void comm_row(const std::string& h, CollKind k, i64 g, double payload) {
  const HardwareSpec hw = hardware(h);
  open_row();
  std::printf("{\"fn\": \"comm_time\", \"hw\": \"%s\", \"kind\": \"%s\", \"group\": %lld, \"payload\": %.17g, "
              "\"time\": %.17g}",
              h.c_str(), coll_name(k), (long long)g, payload, comm_time(k, g, payload, hw));
}

void hopb_row(i64 r, double c, double t, bool on) {
  const OverlapTimeline tl = hopb_schedule(r, c, t, on);
  open_row();
  std::printf("{\"fn\": \"hopb_schedule\", \"requests\": %lld, \"compute\": %.17g, \"comm\": %.17g, \"enabled\": %s, "
              "\"total\": %.17g, \"comm_start\": [",
              (long long)r, c, t, on ? "true" : "false", tl.total);
  for (std::size_t i = 0; i < tl.events.size(); ++i) std::printf("%s%.17g", i ? ", " : "", tl.events[i].comm_start);
  std::printf("]}");
}

void ttl_row(const std::string& m, const std::string& h, Strategy s, i64 tpa, i64 kvp, i64 tpf, i64 ep, i64 pp,
             i64 batch, i64 seq, bool hopb) {
  ParallelismConfig c;
  c.strategy = s;
  c.tpa = tpa;
  c.kvp = kvp;
  c.tpf = tpf;
  c.ep = ep;
  c.pp = pp;
  WorkloadSpec w;
  w.batch = batch;
  w.kv_seq_len = seq;
  const ModelSpec mm = model(m);
  HardwareSpec hw = hardware(h);
  hw.max_gpus = 64;
  const LatencyBreakdown b = decode_ttl(c, mm, w, hw, hopb);
  open_row();
  std::printf(
      "{\"fn\": \"decode_ttl\", \"model\": \"%s\", \"hw\": \"%s\", \"strategy\": \"%s\", \"tpa\": %lld, \"kvp\": "
      "%lld, \"tpf\": %lld, \"ep\": %lld, \"pp\": %lld, \"batch\": %lld, \"seq\": %lld, \"hopb\": %s, "
      "\"qkv_proj\": %.17g, \"kv_read\": %.17g, \"attn_compute\": %.17g, \"a2a_comm\": %.17g, \"a2a_exposed\": "
      "%.17g, \"post_proj\": %.17g, \"attn_allreduce\": %.17g, \"ffn_weight_read\": %.17g, \"ffn_compute\": "
      "%.17g, \"moe_comm\": %.17g, \"ttl\": %.17g, \"memory_bytes\": %.17g}",
      m.c_str(), h.c_str(), strat(s), (long long)tpa, (long long)kvp, (long long)tpf, (long long)ep, (long long)pp,
      (long long)batch, (long long)seq, hopb ? "true" : "false", b.qkv_proj, b.kv_read, b.attn_compute, b.a2a_comm,
      b.a2a_exposed, b.post_proj, b.attn_allreduce, b.ffn_weight_read, b.ffn_compute, b.moe_comm, b.ttl,
      per_gpu_memory_bytes(c, mm, w, hw));
}

}  // namespace

int main() {
  std::printf("{\"generator\": \"oracle/gen_analytic_golden.cpp (reference libhelixsim_core)\", \"rows\": [");
  // pinned by the reference's own tests (test_roofline.cpp:41-62, test_comm.cpp:80-85)
  for (const char* h : {"gb200-like", "b200-measured"}) {
    roofline_row("llama405b-like", h, 8, 1000000, 8, 1, 8);
    roofline_row("llama405b-like", h, 8, 1000000, 8, 8, 8);
    roofline_row("llama405b-like", h, 8, 1000000, 8, 1, 64);
    roofline_row("llama405b-like", h, 8, 1000000, 1, 8, 8);
    roofline_row("deepseek-r1-like", h, 8, 1000000, 1, 8, 1);
    roofline_row("deepseek-r1-like", h, 8, 1000000, 1, 1, 1);
    for (i64 n : {1, 2, 4, 8}) roofline_row("llama3-8b-like", h, 8, 131072 * n, 1, n, n);
    a2a_row("llama405b-like", h, 8, 4, 8);
    a2a_row("llama405b-like", h, 8, 8, 1);
    a2a_row("deepseek-r1-like", h, 8, 8, 1);
    for (i64 n : {2, 4, 8}) a2a_row("llama3-8b-like", h, 8, n, 1);
    for (CollKind k : {CollKind::AllToAll, CollKind::AllReduce, CollKind::AllGather, CollKind::Broadcast})
      for (i64 g : {1, 2, 4, 8}) comm_row(h, k, g, 262144.0);
  }
  hopb_row(8, 2.0, 1.2, false);  // PAPER.md:114-115; test_overlap.cpp:12-21 (25.6 / 17.2)
  hopb_row(8, 2.0, 1.2, true);
  hopb_row(8, 0.5, 1.5, true);
  hopb_row(1, 3.0, 1.0, true);
  hopb_row(64, 0.01, 0.003, true);
  // BASELINE configurations on the measured B200, HOP-B on / off
  for (bool hopb : {true, false}) {
    for (i64 n : {1, 2, 4, 8})
      ttl_row("llama3-8b-like", "b200-measured", Strategy::Helix, 1, n, n, 1, 1, 8, 131072 * n, hopb);
    ttl_row("llama405b-like", "b200-measured", Strategy::Helix, 1, 8, 8, 1, 1, 8, 1000000, hopb);
    ttl_row("llama405b-like", "b200-measured", Strategy::Helix, 8, 1, 8, 1, 1, 8, 1000000, hopb);
    ttl_row("deepseek-r1-like", "b200-measured", Strategy::Helix, 1, 8, 1, 8, 1, 8, 1000000, hopb);
    ttl_row("deepseek-r1-like", "b200-measured", Strategy::Helix, 1, 8, 2, 4, 1, 8, 1000000, hopb);
    ttl_row("deepseek-r1-like", "b200-measured", Strategy::Helix, 1, 8, 8, 1, 1, 8, 1000000, hopb);
    ttl_row("llama405b-like", "gb200-like", Strategy::Helix, 8, 8, 64, 1, 1, 32, 1000000, hopb);
    ttl_row("llama405b-like", "gb200-like", Strategy::TP, 8, 1, 8, 1, 1, 8, 1000000, hopb);
    ttl_row("llama405b-like", "gb200-like", Strategy::MedhaKVP, 8, 4, 8, 1, 1, 8, 1000000, hopb);
    ttl_row("deepseek-r1-like", "gb200-like", Strategy::EP_DPAttention, 1, 1, 4, 8, 1, 32, 1000000, hopb);
    ttl_row("llama405b-like", "gb200-like", Strategy::TP_PP, 8, 1, 8, 1, 4, 8, 1000000, hopb);
  }
  std::printf("\n]}\n");
  return 0;
}
