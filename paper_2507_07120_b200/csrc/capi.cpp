// extern "C" surface (include/helix_b200.h): exceptions never cross the ABI.
#include <cstring>
#include <random>
#include <string>

#include "comm.h"
#include "engine.h"

struct hx_engine {
  hx::Engine* e;
};
struct hx_rng {
  std::mt19937_64 r;
};
struct hx_loopback {
  explicit hx_loopback(int n) : hub(n) {}
  hx::LoopbackHub hub;
};

namespace {
thread_local std::string g_err;

template <class F>
int guard(hx_engine* h, F&& f) {
  try {
    f();
    return HX_OK;
  } catch (const std::invalid_argument& ex) {
    (h ? h->e->last_error : g_err) = ex.what();
    return HX_ERR_INVALID;
  } catch (const hx::CudaError& ex) {
    (h ? h->e->last_error : g_err) = ex.what();
    return HX_ERR_CUDA;
  } catch (const hx::NcclError& ex) {
    (h ? h->e->last_error : g_err) = ex.what();
    return HX_ERR_NCCL;
  } catch (const std::exception& ex) {
    (h ? h->e->last_error : g_err) = ex.what();
    return HX_ERR_STATE;
  }
}
}  // namespace

extern "C" {

const char* hx_version(void) { return "helix-b200 0.1 (sm_100a)"; }

const char* hx_last_error(const hx_engine* e) { return e ? e->e->last_error.c_str() : g_err.c_str(); }

int hx_engine_create(const hx_model_config* m, const hx_parallel_config* p, const hx_runtime_config* r,
                     hx_engine** out) {
  return guard(nullptr, [&] {
    if (!m || !p || !r || !out) throw std::invalid_argument("null argument");
    hx_parallel_config par = *p;
    if (par.loopback) par.loopback = reinterpret_cast<hx_loopback*>(&p->loopback->hub);  // engine sees the hub
    auto* e = new hx::Engine(*m, par, *r);
    *out = new hx_engine{e};
  });
}

void hx_engine_destroy(hx_engine* e) {
  if (!e) return;
  delete e->e;
  delete e;
}

int hx_engine_get_info(const hx_engine* e, hx_engine_info* info) {
  return guard(const_cast<hx_engine*>(e), [&] { e->e->info(info); });
}

int hx_init_weights_mt19937(hx_engine* e, uint64_t seed) {
  return guard(e, [&] { e->e->init_weights_mt19937(seed); });
}
int hx_init_weights_hash(hx_engine* e, uint64_t seed) {
  return guard(e, [&] { e->e->init_weights_hash(seed); });
}

int hx_rng_create(uint64_t seed, hx_rng** out) {
  return guard(nullptr, [&] { *out = new hx_rng{std::mt19937_64(seed)}; });
}
void hx_rng_destroy(hx_rng* r) { delete r; }
double hx_rng_unit_draw(hx_rng* r) {
  const double u = static_cast<double>(r->r() >> 11) * 0x1.0p-53;
  return 2.0 * u - 1.0;
}

int hx_grow_random(hx_engine* e, int64_t layer, int64_t request, int64_t n, hx_rng* rng) {
  return guard(e, [&] { e->e->grow_random(layer, request, n, rng->r); });
}
int hx_append_kv(hx_engine* e, int64_t layer, int64_t request, int64_t n, const float* k, const float* v) {
  return guard(e, [&] { e->e->append_kv(layer, request, n, k, v); });
}
int hx_fill_kv_hash(hx_engine* e, int64_t n, uint64_t seed) {
  return guard(e, [&] { e->e->fill_kv_hash(n, seed); });
}

int64_t hx_total_tokens(const hx_engine* e, int64_t layer, int64_t request) {
  int64_t v = -1;
  guard(const_cast<hx_engine*>(e), [&] { v = e->e->total_tokens(layer, request); });
  return v;
}
int64_t hx_effective_tokens(const hx_engine* e, int64_t layer, int64_t request, int64_t rank) {
  int64_t v = -1;
  guard(const_cast<hx_engine*>(e), [&] { v = e->e->effective_tokens(layer, request, rank); });
  return v;
}
int64_t hx_max_min_gap(const hx_engine* e, int64_t layer, int64_t request) {
  int64_t v = -1;
  guard(const_cast<hx_engine*>(e), [&] { v = e->e->max_min_gap(layer, request); });
  return v;
}
int hx_read_kv(hx_engine* e, int64_t layer, int64_t request, int64_t rank, int64_t head, float* k, float* v) {
  return guard(e, [&] { e->e->read_kv(layer, request, rank, head, k, v); });
}

int hx_harness_step(hx_engine* e, int64_t layer, const float* x, int64_t x_len, float* out, float* lse) {
  return guard(e, [&] { e->e->harness_step(layer, x, x_len, out, lse); });
}
int hx_harness_step_device(hx_engine* e, int64_t layer, const float* x_dev, float* out_dev) {
  return guard(e, [&] { e->e->harness_step_device(layer, x_dev, out_dev); });
}
int hx_decode_step(hx_engine* e, const int32_t* tokens, int32_t* next, float* logits, float* hidden) {
  return guard(e, [&] { e->e->decode_step(tokens, next, logits, hidden); });
}
int hx_decode_step_device(hx_engine* e, const int32_t* tokens_dev, int32_t* next_dev) {
  return guard(e, [&] { e->e->decode_step_device(tokens_dev, next_dev); });
}
int hx_profile_step(hx_engine* e, int64_t reps, double* ms) {
  return guard(e, [&] { e->e->profile_step(reps, ms); });
}
int hx_harness_step_f64(hx_engine* e, int64_t layer, const double* x, int64_t x_len, double* out, double* lse) {
  return guard(e, [&] { e->e->harness_step_f64(layer, x, x_len, out, lse); });
}
int hx_harness_reference_f64(hx_engine* e, int64_t layer, const double* x, int64_t x_len, double* out) {
  return guard(e, [&] { e->e->harness_reference_f64(layer, x, x_len, out); });
}
int hx_append_projected_f64(hx_engine* e, int64_t layer, const double* x, int64_t x_len) {
  return guard(e, [&] { e->e->append_projected_f64(layer, x, x_len); });
}
int hx_append_kv_f64(hx_engine* e, int64_t layer, int64_t request, int64_t n, const double* k, const double* v) {
  return guard(e, [&] { e->e->append_kv_f64(layer, request, n, k, v); });
}
int hx_read_kv_f64(hx_engine* e, int64_t layer, int64_t request, int64_t rank, int64_t head, double* k, double* v) {
  return guard(e, [&] { e->e->read_kv_f64(layer, request, rank, head, k, v); });
}
int hx_attention_f64(const double* q, int64_t n_queries, const double* keys, const double* values, int64_t tokens,
                     int64_t width, double* out, double* lse) {
  return guard(nullptr, [&] { hx::attention_f64(q, n_queries, keys, values, tokens, width, out, lse); });
}
int hx_merge_f64(int64_t n_fragments, int64_t width, const double* outs, const double* lses, double* out,
                 double* lse) {
  return guard(nullptr, [&] { hx::merge_f64(n_fragments, width, outs, lses, out, lse); });
}

int hx_synchronize(hx_engine* e) {
  return guard(e, [&] { e->e->synchronize(); });
}
void* hx_stream(hx_engine* e) { return e ? static_cast<void*>(e->e->stream()) : nullptr; }

int64_t hx_transcript_size(const hx_engine* e) { return static_cast<int64_t>(e->e->transcript().size()); }
int hx_transcript(const hx_engine* e, int64_t* out) {
  return guard(const_cast<hx_engine*>(e), [&] {
    const auto& t = e->e->transcript();
    for (size_t i = 0; i < t.size(); ++i) {
      out[5 * i + 0] = t[i].kind;
      out[5 * i + 1] = t[i].src;
      out[5 * i + 2] = t[i].dst;
      out[5 * i + 3] = t[i].payload;
      out[5 * i + 4] = t[i].lse;
    }
  });
}
int hx_clear_transcript(hx_engine* e) {
  return guard(e, [&] { e->e->clear_transcript(); });
}

int hx_nccl_get_unique_id(void* out128) {
  return guard(nullptr, [&] { hx::nccl_get_unique_id(out128); });
}

int hx_loopback_create(int32_t n, hx_loopback** out) {
  return guard(nullptr, [&] {
    if (n < 1) throw std::invalid_argument("loopback group needs >= 1 rank");
    *out = new hx_loopback(n);
  });
}
void hx_loopback_destroy(hx_loopback* lb) { delete lb; }

}  // extern "C"

extern "C" {
int64_t hx_exchange_layout(int64_t q_per_group, int64_t head_size, int64_t kvp, int64_t* out) {
  int64_t chunk = -1;
  guard(nullptr, [&] { chunk = hx::exchange_layout(q_per_group, head_size, kvp, out); });
  return chunk;
}
int hx_engine_set_flag(hx_engine* e, int32_t flag, int32_t value) {
  return guard(e, [&] { e->e->set_flag(flag, value); });
}
int64_t hx_moe_active_experts(hx_engine* e) {
  int64_t n = -1;
  guard(e, [&] { n = e->e->moe_active_experts(); });
  return n;
}
}  // extern "C"
