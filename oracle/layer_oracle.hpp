// TEST INFRASTRUCTURE ONLY -- see helix_oracle.hpp.
//
// Decoder-layer extension of the reference's attention harness. The
// reference defines only the attention numerics (DecodeHarness::step,
// attention.hpp:460-510); O-projection, FFN, norms and the LM head exist there
// only as analytical shapes (latency.cpp:85-146, types.hpp:27-52). This file
// is the definition the B200 path is held to ("parity unpinned" by the
// reference, "Layer extension"):
//
//   x_0      = E[token]                                  (embedding, U[-1,1))
//   a        = rmsnorm(x_l)                              (no weight, eps 1e-5)
//   attn     = DecodeHarness(seed + l).step(a)           (reference semantics:
//              attend over the sharded cache, merge, then append a's K/V)
//   h        = x_l + attn . W_o                          (W_o: [H x H])
//   f        = rmsnorm(h)
//   x_{l+1}  = h + (silu(f . W_gate) * (f . W_up)) . W_down
//   logits   = rmsnorm(x_L) . W_lm ; next = argmax (lowest index on ties)
//
// W_q/W_k/W_v come from the reference's own mt19937_64 draw (attention.hpp:
// 438-442) with seed + l, or -- for the large bench shapes -- from the
// counter-based hash below (same values on host and device). Extension
// weights always use the hash, scaled by 1/sqrt(fan_in). With bf16 storage
// every weight and KV element is rounded to bf16 exactly as the GPU stores it.
#pragma once

#include <cstdint>
#include <vector>

#include "helix_oracle.hpp"

namespace helix_oracle {

inline std::uint64_t splitmix64(std::uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}
// Counter-based uniform in [-1, 1) with the reference's 53-bit mapping.
inline double hash_unit(std::uint64_t seed, std::uint64_t stream, std::uint64_t index) {
  const std::uint64_t z = splitmix64(splitmix64(seed ^ (stream * 0xD1B54A32D192ED03ull)) + index);
  return 2.0 * (static_cast<double>(z >> 11) * 0x1.0p-53) - 1.0;
}
enum HashKind : std::uint64_t {
  kWq = 1, kWk = 2, kWv = 3, kWo = 4, kWgate = 5, kWup = 6, kWdown = 7, kEmb = 8, kLm = 9,
  kCacheK = 10, kCacheV = 11, kWrouter = 12, kEgate = 13, kEup = 14, kEdown = 15, kWuk = 16, kWuv = 17
};
inline std::uint64_t hash_stream(HashKind kind, std::int64_t layer) {
  return (static_cast<std::uint64_t>(kind) << 32) | static_cast<std::uint64_t>(layer);
}
// Routed-expert weights: one stream per (layer, expert).
inline std::uint64_t expert_stream(HashKind kind, std::int64_t layer, std::int64_t expert) {
  return (static_cast<std::uint64_t>(kind) << 32) | (static_cast<std::uint64_t>(layer) << 16) |
         static_cast<std::uint64_t>(expert);
}

// MoE FFN (types.hpp:19-25 MoESpec; latency.cpp:110-137 analytic shape):
//   f = rmsnorm(h); r = f . W_router [H x E] (scale 1/sqrt(H));
//   top-k experts by r (ties: lower index); w = softmax over the k selected r;
//   y = sum_i w_i * E_i(f) + S(f),  E_i(f) = (silu(f Wg_i) * (f Wu_i)) Wd_i  [H x Fe, Fe x H]
//   S = the dense SwiGLU weights (kWgate/kWup/kWdown) of width shared_ffn (0: none).
struct ModelDims {
  i64 hidden, query_heads, kv_heads, head_size, ffn, layers, vocab;
  i64 n_experts = 0, top_k = 0, expert_ffn = 0;  // n_experts == 0: dense FFN of width `ffn`
  i64 kv_latent = 0;  // > 0: MLA attention (types.hpp:37-49), latent width W = 2 * kv_latent
  // FP8 weights (hash init): every GEMV
  // weight W[k][n] (input k, output n) is stored as e4m3(W / s_n) * s_n with a
  // power-of-two per-output scale s_n = 2^ceil(log2(max_k |W[k][n]| / 448));
  // the embedding (a gather) and the MLA per-head absorptions W_UK / W_UV stay bf16.
  bool w_fp8 = false;
  // FP4 weights (the paper's setting; hash init): every GEMV
  // weight column n is stored in MX-style e2m1 blocks of 32 consecutive inputs k
  // (k0 = 32 i) sharing a power-of-two scale -- round_e2m1_block (helix_oracle.hpp)
  // over W[k0 .. k0+31][n]; same exclusions as w_fp8.
  bool w_fp4 = false;
};

// MLA attention in the weight-absorbed decode form (types.hpp:37-49: K_eff = 1,
// one latent "KV head" of width W = 2 * kv_latent_dim = 576 for
// deepseek-r1-like, 512 latent + 64 rope dims). The projections keep the
// reference's weight shapes (roofline.hpp:17-48 counts W_q as H x Q*Hsz, the
// latent as H x W and W_O as (H/N) x H) plus the two small per-head
// up-projections absorbed at decode time. Per request, with a = rmsnorm(x):
//   n_h = (a . Wq)[h*Hsz:(h+1)*Hsz]     (hash kWq [H x Q*Hsz], scale 1/sqrt(H))
//   q_h = bf16(n_h . Wuk_h)               (W_UK absorbed into the query: hash kWuk
//                                          [Q*Hsz x W] = Q blocks [Hsz x W], scale
//                                          16/sqrt(Hsz); the B200 MMA consumes q in bf16)
//   c   = a . Wdkv                        (hash kWk [H x W], scale 1/sqrt(H); stored bf16)
//   o_h = partial_head_attention / merge_head_fragments (attention.hpp:65-78,
//         :118-137, via shard_attention / merge_fragments) with keys = values =
//         the rank's latent rows, scale logit_scale(W) = 1/sqrt(W); keep
//         o_h[0:DV], DV = W - 64 (the value part of the latent)
//   v_h = o_h . Wuv_h                     (W_UV: hash kWuv [Q*DV x Hsz] = Q blocks
//                                          [DV x Hsz], scale 1/sqrt(DV))
//   h   = x + concat_h(v_h) . Wo          (hash kWo [H x H], scale 1/sqrt(H), as GQA)
// then append c round-robin (attend-then-append, attention.hpp:504-508).
// Cache fill: latent element d of token g of (layer, request) =
//   hash_unit(seed, (kCacheK<<32)|layer, ((request << 32) + g) * W + d).
inline i64 mla_width(i64 kv_latent) { return 2 * kv_latent; }
// FP8-latent MLA query image (the GPU's absorb kernel, mla.cu Q8): one head's
// values scaled by 2^e, e the largest exponent keeping max |q| <= 448, rounded to
// e4m3 (round_e4m3) and scaled back; in place. Returns e.
int quantize_q_e4m3_pow2(double* q, i64 n);
inline i64 mla_value_width(i64 kv_latent) { return 2 * kv_latent - 64; }

enum class QkvInit { MT19937 = 0, Hash = 1 };

class ModelOracle {
 public:
  ModelOracle(ModelDims d, i64 tpa, i64 kvp, i64 chunk, i64 batch, std::uint64_t seed,
              QkvInit qkv_init, bool bf16_storage);
  // Reference-style growth: cache of (layer, request) grown with the
  // reference's V-then-K mt19937_64 draws.
  void grow_random(i64 layer, i64 request, i64 n, std::mt19937_64& rng);
  // Hash growth: token g of (layer, request, kv head h) has
  //   K[d] = hash_unit(seed, (kCacheK<<32)|layer, ((request*K + h)*2^32 + g)*Hsz + d)
  void grow_hash(i64 layer, i64 request, i64 n);
  // One decode step over the batch. tokens: [B]. Returns logits [B x V];
  // hidden: (L+1) x B x H residual stream (x_0 .. x_L).
  std::vector<double> step(const std::vector<std::int64_t>& tokens,
                           std::vector<double>* hidden, std::vector<std::int64_t>* next);
  DecodeHarness& harness(i64 layer, i64 request) {
    return h_[static_cast<std::size_t>(layer * batch_ + request)];
  }
  const Mat& wo(i64 l) const { return wo_[static_cast<std::size_t>(l)]; }
  const Mat& wgate(i64 l) const { return wg_[static_cast<std::size_t>(l)]; }
  const Mat& wup(i64 l) const { return wu_[static_cast<std::size_t>(l)]; }
  const Mat& wdown(i64 l) const { return wd_[static_cast<std::size_t>(l)]; }
  const Mat& emb() const { return emb_; }
  const Mat& lm() const { return lm_; }
  const Mat& router(i64 l) const { return wr_[static_cast<std::size_t>(l)]; }
  // Last step's routing: [B][top_k] expert ids per layer (for kernel parity)
  const std::vector<std::vector<i64>>& routes() const { return routes_; }
  // Last step's router margin per (layer, request): r[k-th] - r[(k+1)-th]
  // (a kernel whose logits differ by more than this may legally pick another set)
  const std::vector<double>& route_gaps() const { return gaps_; }
  // FP8 (e4m3) KV storage: the GQA caches (DecodeHarness::set_kv_fp8) and the MLA
  // latents (with the e4m3 query image, attend_mla).
  void set_kv_fp8(bool on) {
    kv_fp8_ = on;
    for (auto& h : h_) h.set_kv_fp8(on);
  }
  // FP4 (e2m1 blocks) KV storage for the GQA caches (DecodeHarness::set_kv_fp4).
  void set_kv_fp4(bool on) {
    for (auto& h : h_) h.set_kv_fp4(on);
  }

 private:
  ModelDims d_;
  i64 batch_;
  std::uint64_t seed_;
  bool bf16_;
  bool kv_fp8_ = false;
  std::vector<DecodeHarness> h_;
  std::vector<Mat> wo_, wg_, wu_, wd_, wr_;
  std::vector<std::vector<Mat>> eg_, eu_, ed_;  // [layer][expert]
  std::vector<std::vector<i64>> routes_;        // [layer*B + b] -> selected experts
  std::vector<ShardedKVCache> mla_;             // [layer*B + b] latent caches (MLA)
  std::vector<Mat> wq_mla_, wdkv_, wuk_, wuv_;  // [layer]
  std::vector<double> attend_mla(i64 l, i64 b, const std::vector<double>& a);
  std::vector<double> gaps_;                    // [layer*B + b] -> top-k margin
  Mat emb_, lm_;
  std::vector<double> ffn(i64 l, i64 b, const std::vector<double>& f);
};

// Hash-initialised matrix [rows x cols], row-major index r*cols + c, times scale.
Mat hash_matrix(std::uint64_t seed, HashKind kind, i64 layer, i64 rows, i64 cols, double scale,
                bool bf16);
// The same values quantised per column (output feature) to e4m3 with a
// power-of-two scale (ModelDims::w_fp8).
Mat hash_matrix_fp8(std::uint64_t seed, HashKind kind, i64 layer, i64 rows, i64 cols, double scale);
double fp8_pow2_scale(double absmax);
// ModelDims::w_fp4: e2m1 blocks of 32 along the rows (inputs k) of every column.
void quantize_fp4_cols(Mat& m);
void quantize_fp8_cols(Mat& m);  // per column: e4m3(m / s_c) * s_c
std::vector<double> rmsnorm(const std::vector<double>& x, double eps = 1e-5);

}  // namespace helix_oracle
