// TEST INFRASTRUCTURE ONLY -- compiled against the REFERENCE's own
// helixsim core (oracle/Makefile, target config_golden) to record what its
// validate_config (types.cpp:86-141) returns over a grid of layouts, so the
// Python mirror (paper_2507_07120_b200/model.py validate_config) is pinned to
// the reference itself: tests/golden/validate_config.json.
#include <cstdio>
#include <string>
#include <vector>

#include "helixsim/types.hpp"

using namespace helixsim;

int main() {
  ModelSpec gqa;
  gqa.name = "gqa";
  gqa.layers = 2;
  gqa.hidden_dim = 16384;
  gqa.query_heads = 128;
  gqa.kv_heads = 8;
  gqa.head_size = 128;
  gqa.ffn_dim = 65536;
  ModelSpec mla = gqa;
  mla.name = "mla";
  mla.kv_heads = 1;
  mla.attention_kind = AttentionKind::MLA;
  mla.kv_latent_dim = 288;
  ModelSpec moe = gqa;
  moe.name = "moe";
  moe.moe = MoESpec{256, 8, 2048, 2048};
  ModelSpec moe_odd = moe;  // experts / expert width that the widths do not divide
  moe_odd.name = "moe_odd";
  moe_odd.moe = MoESpec{6, 2, 24, 0};
  const ModelSpec* models[] = {&gqa, &mla, &moe, &moe_odd};
  const Strategy strats[] = {Strategy::Helix, Strategy::TP, Strategy::TP_PP, Strategy::EP_DPAttention,
                             Strategy::MedhaKVP};
  // compact rows: [model, max_gpus, strategy, tpa, kvp, tpf, ep, pp, total_gpus, ok, rule]
  std::printf("{\"columns\": [\"model\", \"max_gpus\", \"strategy\", \"tpa\", \"kvp\", \"tpf\", \"ep\", "
              "\"pp\", \"total_gpus\", \"ok\", \"rule\"],\n \"rows\": [\n");
  bool first = true;
  for (const ModelSpec* m : models)
    for (i64 maxg : {64})
      for (Strategy s : strats)
        for (i64 tpa : {0, 1, 3, 8, 16})
          for (i64 kvp : {1, 5, 8})
            for (i64 tpf : {1, 8, 24})
              for (i64 ep : {1, 8})
                for (i64 pp : {1, 2}) {
                  HardwareSpec hw;
                  hw.max_gpus = maxg;
                  const ParallelismConfig c{s, tpa, kvp, tpf, ep, pp};
                  const Validity v = validate_config(c, *m, hw);
                  std::printf("%s[\"%s\",%lld,\"%s\",%lld,%lld,%lld,%lld,%lld,%lld,%d,\"%s\"]", first ? "" : ",\n",
                              m->name.c_str(), static_cast<long long>(maxg), strategy_name(s),
                              static_cast<long long>(tpa), static_cast<long long>(kvp), static_cast<long long>(tpf),
                              static_cast<long long>(ep), static_cast<long long>(pp),
                              static_cast<long long>(c.total_gpus()), v.ok ? 1 : 0, v.rule.c_str());
                  first = false;
                }
  std::printf("\n]}\n");
  return 0;
}
