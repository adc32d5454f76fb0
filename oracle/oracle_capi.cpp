// TEST INFRASTRUCTURE ONLY -- ctypes surface over the CPU oracle
// (helix_oracle.hpp) for tests/ and bench.py's cpu_baseline leg.
// Status: 0 ok, 1 invalid_argument (message via oracle_last_error), 2 other.
#include <cstring>
#include <exception>
#include <string>

#include "helix_oracle.hpp"
#include "layer_oracle.hpp"

using namespace helix_oracle;

namespace {
thread_local std::string g_err;
template <class F>
int guard(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return 1;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 2;
  }
}
}  // namespace

extern "C" {

const char* oracle_last_error() { return g_err.c_str(); }

void* oracle_rng_create(std::uint64_t seed) { return new std::mt19937_64(seed); }
void oracle_rng_free(void* r) { delete static_cast<std::mt19937_64*>(r); }
double oracle_rng_unit_draw(void* r) { return unit_draw(*static_cast<std::mt19937_64*>(r)); }
std::uint64_t oracle_rng_next(void* r) { return (*static_cast<std::mt19937_64*>(r))(); }
double oracle_round_bf16(double x) { return round_bf16(x); }
double oracle_round_e4m3(double x) { return round_e4m3(x); }
int oracle_quantize_q_e4m3_pow2(double* q, long long n) { return quantize_q_e4m3_pow2(q, n); }

int oracle_harness_create(i64 q, i64 k, i64 hsz, i64 tpa, i64 kvp, i64 chunk, std::uint64_t seed,
                          int bf16, void** out) {
  return guard([&] {
    *out = new DecodeHarness({q, k, hsz}, tpa, kvp, chunk, seed, bf16 != 0);
  });
}
void oracle_harness_free(void* h) { delete static_cast<DecodeHarness*>(h); }
void oracle_harness_set_kv_fp8(void* h, int on) { static_cast<DecodeHarness*>(h)->set_kv_fp8(on != 0); }
void oracle_harness_set_kv_fp4(void* h, int on) { static_cast<DecodeHarness*>(h)->set_kv_fp4(on != 0); }
void oracle_round_e2m1_block(double* x, i64 n) { round_e2m1_block(x, n); }

int oracle_harness_grow_random(void* h, i64 n, void* rng) {
  return guard([&] {
    static_cast<DecodeHarness*>(h)->grow_random(n, *static_cast<std::mt19937_64*>(rng));
  });
}

int oracle_harness_step(void* hp, const double* x, i64 n, double* out, double* lse) {
  return guard([&] {
    auto* h = static_cast<DecodeHarness*>(hp);
    Mat o = h->step(std::vector<double>(x, x + n));
    std::memcpy(out, o.a.data(), o.a.size() * sizeof(double));
    if (lse) std::memcpy(lse, h->last_lse().data(), h->last_lse().size() * sizeof(double));
  });
}

int oracle_harness_step_append(void* hp, const double* x, i64 n, double* out, double* lse,
                               const double* k, const double* v) {
  return guard([&] {
    auto* h = static_cast<DecodeHarness*>(hp);
    const Dims d = h->dims();
    Mat km(d.kv_heads, d.head_size), vm(d.kv_heads, d.head_size);
    std::memcpy(km.a.data(), k, km.a.size() * sizeof(double));
    std::memcpy(vm.a.data(), v, vm.a.size() * sizeof(double));
    Mat o = h->step_with_append(std::vector<double>(x, x + n), &km, &vm);
    std::memcpy(out, o.a.data(), o.a.size() * sizeof(double));
    if (lse) std::memcpy(lse, h->last_lse().data(), h->last_lse().size() * sizeof(double));
  });
}

int oracle_harness_reference(void* hp, const double* x, i64 n, double* out) {
  return guard([&] {
    Mat o = static_cast<DecodeHarness*>(hp)->reference(std::vector<double>(x, x + n));
    std::memcpy(out, o.a.data(), o.a.size() * sizeof(double));
  });
}

int oracle_harness_append_projected(void* hp, const double* x, i64 n) {
  return guard([&] { static_cast<DecodeHarness*>(hp)->append_projected(std::vector<double>(x, x + n)); });
}

int oracle_harness_project(void* hp, const double* x, i64 n, double* q, double* k, double* v) {
  return guard([&] {
    auto* h = static_cast<DecodeHarness*>(hp);
    std::vector<double> xv(x, x + n);
    std::vector<double> qq = h->project_q(xv);
    std::memcpy(q, qq.data(), qq.size() * sizeof(double));
    Mat kk, vv;
    h->project_kv(xv, kk, vv);
    std::memcpy(k, kk.a.data(), kk.a.size() * sizeof(double));
    std::memcpy(v, vv.a.data(), vv.a.size() * sizeof(double));
  });
}

// which: 0 = W_q, 1 = W_k, 2 = W_v (row-major [hidden x cols])
int oracle_harness_weights(void* hp, int which, double* out) {
  return guard([&] {
    auto* h = static_cast<DecodeHarness*>(hp);
    const Mat& m = which == 0 ? h->wq() : which == 1 ? h->wk() : h->wv();
    std::memcpy(out, m.a.data(), m.a.size() * sizeof(double));
  });
}

i64 oracle_harness_total_tokens(void* hp) {
  return static_cast<DecodeHarness*>(hp)->cache().total_tokens();
}
i64 oracle_harness_effective_tokens(void* hp, i64 rank) {
  return static_cast<DecodeHarness*>(hp)->cache().effective_tokens(rank);
}
i64 oracle_harness_max_min_gap(void* hp) {
  return static_cast<DecodeHarness*>(hp)->cache().max_min_gap();
}

// which: 0 keys, 1 values; rows of (rank, head) in append order
int oracle_harness_cache_rows(void* hp, i64 rank, i64 head, int which, double* out) {
  return guard([&] {
    const auto& c = static_cast<DecodeHarness*>(hp)->cache();
    const Mat& m = which == 0 ? c.keys(rank, head) : c.values(rank, head);
    std::memcpy(out, m.a.data(), m.a.size() * sizeof(double));
  });
}

int oracle_harness_token_order(void* hp, i64* ranks, i64* rows) {
  return guard([&] {
    const auto& o = static_cast<DecodeHarness*>(hp)->cache().token_order();
    for (std::size_t i = 0; i < o.size(); ++i) {
      ranks[i] = o[i].rank;
      rows[i] = o[i].row;
    }
  });
}

i64 oracle_harness_transcript_size(void* hp) {
  return static_cast<i64>(static_cast<DecodeHarness*>(hp)->transcript().size());
}
// out: [n x 5] = kind, src, dst, payload_scalars, lse_scalars
int oracle_harness_transcript(void* hp, i64* out) {
  return guard([&] {
    const auto& t = static_cast<DecodeHarness*>(hp)->transcript();
    for (std::size_t i = 0; i < t.size(); ++i) {
      out[5 * i + 0] = static_cast<i64>(t[i].kind);
      out[5 * i + 1] = t[i].src;
      out[5 * i + 2] = t[i].dst;
      out[5 * i + 3] = t[i].payload_scalars;
      out[5 * i + 4] = t[i].lse_scalars;
    }
  });
}

// Single-head primitives: keys/values row-major [n x w].
int oracle_partial_head_attention(const double* q, const double* keys, const double* values,
                                  i64 n, i64 w, double* out, double* lse) {
  return guard([&] {
    Mat K(n, w), V(n, w);
    std::memcpy(K.a.data(), keys, static_cast<std::size_t>(n * w) * sizeof(double));
    std::memcpy(V.a.data(), values, static_cast<std::size_t>(n * w) * sizeof(double));
    HeadFragment f = partial_head_attention(std::vector<double>(q, q + w), K, V);
    std::memcpy(out, f.out.data(), static_cast<std::size_t>(w) * sizeof(double));
    *lse = f.lse;
  });
}

int oracle_reference_attention(const double* q, const double* keys, const double* values, i64 n,
                               i64 w, double* out) {
  return guard([&] {
    Mat K(n, w), V(n, w);
    std::memcpy(K.a.data(), keys, static_cast<std::size_t>(n * w) * sizeof(double));
    std::memcpy(V.a.data(), values, static_cast<std::size_t>(n * w) * sizeof(double));
    std::vector<double> o = reference_attention(std::vector<double>(q, q + w), K, V);
    std::memcpy(out, o.data(), static_cast<std::size_t>(w) * sizeof(double));
  });
}

// frags: outs [nf x w], lses [nf]
int oracle_merge_head_fragments(i64 nf, i64 w, const double* outs, const double* lses,
                                double* out, double* lse) {
  return guard([&] {
    std::vector<HeadFragment> f(static_cast<std::size_t>(nf));
    for (i64 i = 0; i < nf; ++i) {
      f[static_cast<std::size_t>(i)].out.assign(outs + i * w, outs + (i + 1) * w);
      f[static_cast<std::size_t>(i)].lse = lses[i];
    }
    HeadFragment m = merge_head_fragments(f);
    std::memcpy(out, m.out.data(), static_cast<std::size_t>(w) * sizeof(double));
    *lse = m.lse;
  });
}

}  // extern "C"

// ---- decoder-layer extension (layer_oracle.hpp) ----
extern "C" {

int oracle_model_create(i64 hidden, i64 q, i64 k, i64 hsz, i64 ffn, i64 layers, i64 vocab, i64 tpa,
                        i64 kvp, i64 chunk, i64 batch, std::uint64_t seed, int qkv_hash, int bf16,
                        void** out) {
  return guard([&] {
    *out = new ModelOracle({hidden, q, k, hsz, ffn, layers, vocab}, tpa, kvp, chunk, batch, seed,
                           qkv_hash ? QkvInit::Hash : QkvInit::MT19937, bf16 != 0);
  });
}

// Dense model with FP8 (e4m3, per-output power-of-two scale) GEMV weights.
int oracle_model_create_w8(i64 hidden, i64 q, i64 k, i64 hsz, i64 ffn, i64 layers, i64 vocab, i64 tpa, i64 kvp,
                           i64 chunk, i64 batch, std::uint64_t seed, void** out) {
  return guard([&] {
    ModelDims d{hidden, q, k, hsz, ffn, layers, vocab};
    d.w_fp8 = true;
    *out = new ModelOracle(d, tpa, kvp, chunk, batch, seed, QkvInit::Hash, true);
  });
}

// Any model (dense, MoE and/or MLA as oracle_model_create_ex) with FP8 (wq = 1)
// or FP4 (wq = 2) GEMV weights.
int oracle_model_create_wq(i64 hidden, i64 q, i64 k, i64 hsz, i64 ffn, i64 layers, i64 vocab, i64 n_experts,
                           i64 top_k, i64 expert_ffn, i64 kv_latent, i64 tpa, i64 kvp, i64 chunk, i64 batch,
                           std::uint64_t seed, int wq, void** out) {
  return guard([&] {
    ModelDims d{hidden, q, k, hsz, ffn, layers, vocab};
    d.n_experts = n_experts;
    d.top_k = top_k;
    d.expert_ffn = expert_ffn;
    d.kv_latent = kv_latent;
    d.w_fp8 = wq == 1;
    d.w_fp4 = wq == 2;
    *out = new ModelOracle(d, tpa, kvp, chunk, batch, seed, QkvInit::Hash, true);
  });
}

// Any model (MoE and/or MLA as oracle_model_create_ex) with FP8 GEMV weights.
int oracle_model_create_ex_w8(i64 hidden, i64 q, i64 k, i64 hsz, i64 ffn, i64 layers, i64 vocab, i64 n_experts,
                              i64 top_k, i64 expert_ffn, i64 kv_latent, i64 tpa, i64 kvp, i64 chunk, i64 batch,
                              std::uint64_t seed, void** out) {
  return guard([&] {
    ModelDims d{hidden, q, k, hsz, ffn, layers, vocab};
    d.n_experts = n_experts;
    d.top_k = top_k;
    d.expert_ffn = expert_ffn;
    d.kv_latent = kv_latent;
    d.w_fp8 = true;
    *out = new ModelOracle(d, tpa, kvp, chunk, batch, seed, QkvInit::Hash, true);
  });
}

// MoE model: ffn = shared-expert width (0: none), n_experts / top_k / expert_ffn routed.
int oracle_model_create_moe(i64 hidden, i64 q, i64 k, i64 hsz, i64 shared_ffn, i64 layers, i64 vocab,
                            i64 n_experts, i64 top_k, i64 expert_ffn, i64 tpa, i64 kvp, i64 chunk, i64 batch,
                            std::uint64_t seed, int qkv_hash, int bf16, void** out) {
  return guard([&] {
    ModelDims d{hidden, q, k, hsz, shared_ffn, layers, vocab};
    d.n_experts = n_experts;
    d.top_k = top_k;
    d.expert_ffn = expert_ffn;
    *out = new ModelOracle(d, tpa, kvp, chunk, batch, seed, qkv_hash ? QkvInit::Hash : QkvInit::MT19937,
                           bf16 != 0);
  });
}

// General model: MoE when n_experts > 0, MLA attention when kv_latent > 0.
int oracle_model_create_ex(i64 hidden, i64 q, i64 k, i64 hsz, i64 ffn, i64 layers, i64 vocab, i64 n_experts,
                           i64 top_k, i64 expert_ffn, i64 kv_latent, i64 tpa, i64 kvp, i64 chunk, i64 batch,
                           std::uint64_t seed, int qkv_hash, int bf16, void** out) {
  return guard([&] {
    ModelDims d{hidden, q, k, hsz, ffn, layers, vocab};
    d.n_experts = n_experts;
    d.top_k = top_k;
    d.expert_ffn = expert_ffn;
    d.kv_latent = kv_latent;
    *out = new ModelOracle(d, tpa, kvp, chunk, batch, seed, qkv_hash ? QkvInit::Hash : QkvInit::MT19937,
                           bf16 != 0);
  });
}

// routes of the last step: [layers][B][top_k]
int oracle_model_routes(void* mp, std::int64_t* out) {
  return guard([&] {
    auto* m = static_cast<ModelOracle*>(mp);
    std::size_t o = 0;
    for (const auto& r : m->routes())
      for (i64 e : r) out[o++] = e;
  });
}
// router top-k margins of the last step: [layers][B]
int oracle_model_route_gaps(void* mp, double* out) {
  return guard([&] {
    const auto& g = static_cast<ModelOracle*>(mp)->route_gaps();
    std::copy(g.begin(), g.end(), out);
  });
}
void oracle_model_free(void* m) { delete static_cast<ModelOracle*>(m); }
void oracle_model_set_kv_fp8(void* m, int on) { static_cast<ModelOracle*>(m)->set_kv_fp8(on != 0); }
void oracle_model_set_kv_fp4(void* m, int on) { static_cast<ModelOracle*>(m)->set_kv_fp4(on != 0); }

int oracle_model_grow_random(void* m, i64 layer, i64 request, i64 n, void* rng) {
  return guard([&] {
    static_cast<ModelOracle*>(m)->grow_random(layer, request, n,
                                              *static_cast<std::mt19937_64*>(rng));
  });
}
int oracle_model_grow_hash(void* m, i64 layer, i64 request, i64 n) {
  return guard([&] { static_cast<ModelOracle*>(m)->grow_hash(layer, request, n); });
}

// logits [B x V], hidden [(L+1) x B x H] (nullable), next [B] (nullable)
int oracle_model_step(void* m, const std::int64_t* tokens, i64 batch, double* logits,
                      double* hidden, std::int64_t* next) {
  return guard([&] {
    std::vector<double> hs;
    std::vector<std::int64_t> nx;
    std::vector<double> lg = static_cast<ModelOracle*>(m)->step(
        std::vector<std::int64_t>(tokens, tokens + batch), hidden ? &hs : nullptr, &nx);
    std::memcpy(logits, lg.data(), lg.size() * sizeof(double));
    if (hidden) std::memcpy(hidden, hs.data(), hs.size() * sizeof(double));
    if (next) std::memcpy(next, nx.data(), nx.size() * sizeof(std::int64_t));
  });
}

// which: 0 Wq 1 Wk 2 Wv 3 Wo 4 Wgate 5 Wup 6 Wdown 7 emb 8 lm (row-major, reference orientation)
int oracle_model_weight(void* mp, int which, i64 layer, double* out) {
  return guard([&] {
    auto* m = static_cast<ModelOracle*>(mp);
    const Mat* w = nullptr;
    switch (which) {
      case 0: w = &m->harness(layer, 0).wq(); break;
      case 1: w = &m->harness(layer, 0).wk(); break;
      case 2: w = &m->harness(layer, 0).wv(); break;
      case 3: w = &m->wo(layer); break;
      case 4: w = &m->wgate(layer); break;
      case 5: w = &m->wup(layer); break;
      case 6: w = &m->wdown(layer); break;
      case 7: w = &m->emb(); break;
      case 8: w = &m->lm(); break;
      default: throw std::invalid_argument("unknown weight id");
    }
    std::memcpy(out, w->a.data(), w->a.size() * sizeof(double));
  });
}

double oracle_hash_unit(std::uint64_t seed, std::uint64_t stream, std::uint64_t index) {
  return hash_unit(seed, stream, index);
}

}  // extern "C"
