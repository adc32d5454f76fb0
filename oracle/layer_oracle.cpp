// TEST INFRASTRUCTURE ONLY -- see layer_oracle.hpp.
#include "layer_oracle.hpp"

#include <algorithm>
#include <cmath>
#include <numeric>

namespace helix_oracle {

Mat hash_matrix(std::uint64_t seed, HashKind kind, i64 layer, i64 rows, i64 cols, double scale,
                bool bf16) {
  Mat m(rows, cols);
  const std::uint64_t stream = hash_stream(kind, layer);
  for (i64 r = 0; r < rows; ++r)
    for (i64 c = 0; c < cols; ++c) {
      const double v = hash_unit(seed, stream, static_cast<std::uint64_t>(r * cols + c)) * scale;
      m(r, c) = bf16 ? round_bf16(v) : v;
    }
  return m;
}

double fp8_pow2_scale(double absmax) {
  if (!(absmax > 0.0)) return 1.0;
  int e = 0;
  const double f = std::frexp(absmax / 448.0, &e);  // absmax/448 = f * 2^e, f in [0.5, 1)
  return std::ldexp(1.0, f == 0.5 ? e - 1 : e);     // smallest 2^j >= absmax / 448
}

void quantize_fp8_cols(Mat& m) {
  for (i64 c = 0; c < m.cols; ++c) {
    double mx = 0.0;
    for (i64 r = 0; r < m.rows; ++r) mx = std::max(mx, std::fabs(m(r, c)));
    const double s = fp8_pow2_scale(mx);
    for (i64 r = 0; r < m.rows; ++r) m(r, c) = round_e4m3(m(r, c) / s) * s;
  }
}

void quantize_fp4_cols(Mat& m) {
  double blk[32];
  for (i64 c = 0; c < m.cols; ++c)
    for (i64 r0 = 0; r0 < m.rows; r0 += 32) {
      const i64 n = std::min<i64>(32, m.rows - r0);
      for (i64 i = 0; i < n; ++i) blk[i] = m(r0 + i, c);
      round_e2m1_block(blk, n);
      for (i64 i = 0; i < n; ++i) m(r0 + i, c) = blk[i];
    }
}

Mat hash_matrix_fp8(std::uint64_t seed, HashKind kind, i64 layer, i64 rows, i64 cols, double scale) {
  Mat m = hash_matrix(seed, kind, layer, rows, cols, scale, false);
  quantize_fp8_cols(m);
  return m;
}

std::vector<double> rmsnorm(const std::vector<double>& x, double eps) {
  double ss = 0.0;
  for (double v : x) ss += v * v;
  const double inv = 1.0 / std::sqrt(ss / static_cast<double>(x.size()) + eps);
  std::vector<double> y(x.size());
  for (std::size_t i = 0; i < x.size(); ++i) y[i] = x[i] * inv;
  return y;
}

namespace {
// y = x . W for W [in x out] row-major
std::vector<double> vecmat(const std::vector<double>& x, const Mat& w) {
  std::vector<double> y(static_cast<std::size_t>(w.cols), 0.0);
  for (i64 c = 0; c < w.cols; ++c) {
    double acc = 0.0;
    for (i64 k = 0; k < w.rows; ++k) acc += x[static_cast<std::size_t>(k)] * w(k, c);
    y[static_cast<std::size_t>(c)] = acc;
  }
  return y;
}
}  // namespace

ModelOracle::ModelOracle(ModelDims d, i64 tpa, i64 kvp, i64 chunk, i64 batch, std::uint64_t seed,
                         QkvInit qkv_init, bool bf16)
    : d_(d), batch_(batch), seed_(seed), bf16_(bf16) {
  if (d.hidden != d.query_heads * d.head_size)
    throw std::invalid_argument("hidden_dim must equal query_heads * head_size");
  if (d.n_experts > 0 && (d.top_k < 1 || d.top_k > d.n_experts || d.expert_ffn < 1))
    throw std::invalid_argument("invalid MoE shape");
  const bool mla = d.kv_latent > 0;
  if (mla && (d.kv_heads != 1 || tpa != 1 || mla_width(d.kv_latent) <= 64))
    throw std::invalid_argument("MLA needs kv_heads == 1, tpa == 1 and a latent wider than the 64 rope dims");
  const i64 W = mla ? mla_width(d.kv_latent) : 0, DV = mla ? mla_value_width(d.kv_latent) : 0;
  const double sh = 1.0 / std::sqrt(static_cast<double>(d.hidden));
  const double sf = 1.0 / std::sqrt(static_cast<double>(std::max<i64>(d.ffn, 1)));
  if ((d.w_fp8 || d.w_fp4) && qkv_init != QkvInit::Hash)
    throw std::invalid_argument("FP8 / FP4 weights: hash-initialised weights");
  auto wmat = [&](HashKind kind, i64 l, i64 rows, i64 cols, double sc) {
    if (d.w_fp4) {
      Mat m = hash_matrix(seed, kind, l, rows, cols, sc, false);
      quantize_fp4_cols(m);
      return m;
    }
    return d.w_fp8 ? hash_matrix_fp8(seed, kind, l, rows, cols, sc) : hash_matrix(seed, kind, l, rows, cols, sc, bf16);
  };
  h_.reserve(static_cast<std::size_t>(d.layers * batch));
  for (i64 l = 0; l < d.layers; ++l) {
    if (mla) {
      for (i64 b = 0; b < batch; ++b) mla_.emplace_back(kvp, 1, W, chunk);
      // W_q and the latent down-projection are GEMV weights (FP8 under w_fp8);
      // the per-head absorptions W_UK / W_UV stay bf16
      wq_mla_.push_back(wmat(kWq, l, d.hidden, d.query_heads * d.head_size, sh));
      wuk_.push_back(hash_matrix(seed, kWuk, l, d.query_heads * d.head_size, W,
                                 16.0 / std::sqrt(static_cast<double>(d.head_size)), bf16));
      wdkv_.push_back(wmat(kWk, l, d.hidden, W, sh));
      wuv_.push_back(hash_matrix(seed, kWuv, l, d.query_heads * DV, d.head_size,
                                 1.0 / std::sqrt(static_cast<double>(DV)), bf16));
    }
    for (i64 b = 0; b < batch && !mla; ++b) {
      h_.emplace_back(Dims{d.query_heads, d.kv_heads, d.head_size}, tpa, kvp, chunk,
                      seed + static_cast<std::uint64_t>(l), bf16);
      if (qkv_init == QkvInit::Hash)
        h_.back().set_weights(wmat(kWq, l, d.hidden, d.query_heads * d.head_size, 1.0),
                              wmat(kWk, l, d.hidden, d.kv_heads * d.head_size, 1.0),
                              wmat(kWv, l, d.hidden, d.kv_heads * d.head_size, 1.0));
    }
    wo_.push_back(wmat(kWo, l, d.hidden, d.hidden, sh));
    if (d.ffn > 0) {  // dense FFN, or the MoE shared expert
      wg_.push_back(wmat(kWgate, l, d.hidden, d.ffn, sh));
      wu_.push_back(wmat(kWup, l, d.hidden, d.ffn, sh));
      wd_.push_back(wmat(kWdown, l, d.ffn, d.hidden, sf));
    } else {
      wg_.emplace_back();
      wu_.emplace_back();
      wd_.emplace_back();
    }
    if (d.n_experts > 0) {
      wr_.push_back(wmat(kWrouter, l, d.hidden, d.n_experts, sh));
      const double se = 1.0 / std::sqrt(static_cast<double>(d.expert_ffn));
      eg_.emplace_back();
      eu_.emplace_back();
      ed_.emplace_back();
      for (i64 e = 0; e < d.n_experts; ++e) {
        auto em = [&](HashKind k, i64 rows, i64 cols, double sc) {
          Mat m(rows, cols);
          const std::uint64_t st = expert_stream(k, l, e);
          for (i64 r = 0; r < rows; ++r)
            for (i64 c = 0; c < cols; ++c) {
              const double v = hash_unit(seed, st, static_cast<std::uint64_t>(r * cols + c)) * sc;
              m(r, c) = (bf16 && !d.w_fp8 && !d.w_fp4) ? round_bf16(v) : v;
            }
          if (d.w_fp8) quantize_fp8_cols(m);
          if (d.w_fp4) quantize_fp4_cols(m);
          return m;
        };
        eg_.back().push_back(em(kEgate, d.hidden, d.expert_ffn, sh));
        eu_.back().push_back(em(kEup, d.hidden, d.expert_ffn, sh));
        ed_.back().push_back(em(kEdown, d.expert_ffn, d.hidden, se));
      }
    }
  }
  routes_.assign(static_cast<std::size_t>(d.layers * batch), {});
  gaps_.assign(static_cast<std::size_t>(d.layers * batch), 1e30);
  emb_ = hash_matrix(seed, kEmb, 0, d.vocab, d.hidden, 1.0, bf16);
  lm_ = wmat(kLm, 0, d.hidden, d.vocab, sh);
}

void ModelOracle::grow_random(i64 layer, i64 request, i64 n, std::mt19937_64& rng) {
  if (d_.kv_latent > 0) throw std::invalid_argument("MLA caches are grown with the counter hash");
  harness(layer, request).grow_random(n, rng);
}

void ModelOracle::grow_hash(i64 layer, i64 request, i64 n) {
  if (d_.kv_latent > 0) {
    const i64 W = mla_width(d_.kv_latent);
    ShardedKVCache& c = mla_[static_cast<std::size_t>(layer * batch_ + request)];
    for (i64 i = 0; i < n; ++i) {
      const i64 g = c.total_tokens();
      Mat row(1, W);
      for (i64 dd = 0; dd < W; ++dd) {
        const std::uint64_t idx =
            ((static_cast<std::uint64_t>(request) << 32) + static_cast<std::uint64_t>(g)) *
                static_cast<std::uint64_t>(W) +
            static_cast<std::uint64_t>(dd);
        const double v = hash_unit(seed_, hash_stream(kCacheK, layer), idx);
        row(0, dd) = kv_fp8_ ? round_e4m3(v) : (bf16_ ? round_bf16(v) : v);
      }
      c.append_round_robin(row, row);
    }
    return;
  }
  DecodeHarness& h = harness(layer, request);
  const i64 K = d_.kv_heads, w = d_.head_size;
  for (i64 i = 0; i < n; ++i) {
    const i64 g = h.cache().total_tokens();
    Mat k(K, w), v(K, w);
    for (i64 kh = 0; kh < K; ++kh)
      for (i64 dd = 0; dd < w; ++dd) {
        const std::uint64_t idx =
            ((static_cast<std::uint64_t>(request * K + kh) << 32) + static_cast<std::uint64_t>(g)) *
                static_cast<std::uint64_t>(w) +
            static_cast<std::uint64_t>(dd);
        const double kv = hash_unit(seed_, hash_stream(kCacheK, layer), idx);
        const double vv = hash_unit(seed_, hash_stream(kCacheV, layer), idx);
        k(kh, dd) = kv;
        v(kh, dd) = vv;
      }
    h.round_kv_rows(k);  // the harness's storage rounding (bf16 / e4m3 / e2m1 blocks)
    h.round_kv_rows(v);
    h.cache().append_round_robin(k, v);
  }
}

std::vector<double> ModelOracle::ffn(i64 l, i64 b, const std::vector<double>& f) {
  const i64 H = d_.hidden;
  std::vector<double> y(static_cast<std::size_t>(H), 0.0);
  auto swiglu_ffn = [&](const Mat& wg, const Mat& wu, const Mat& wd, double scale) {
    const std::vector<double> gt = vecmat(f, wg);
    const std::vector<double> up = vecmat(f, wu);
    std::vector<double> m(gt.size());
    for (std::size_t i = 0; i < m.size(); ++i) m[i] = gt[i] / (1.0 + std::exp(-gt[i])) * up[i];
    const std::vector<double> dn = vecmat(m, wd);
    for (i64 i = 0; i < H; ++i) y[static_cast<std::size_t>(i)] += scale * dn[static_cast<std::size_t>(i)];
  };
  if (d_.n_experts > 0) {
    const std::vector<double> r = vecmat(f, wr_[static_cast<std::size_t>(l)]);
    std::vector<i64> idx(static_cast<std::size_t>(d_.n_experts));
    std::iota(idx.begin(), idx.end(), 0);
    std::stable_sort(idx.begin(), idx.end(), [&](i64 a, i64 c) {
      return r[static_cast<std::size_t>(a)] > r[static_cast<std::size_t>(c)];
    });
    gaps_[static_cast<std::size_t>(l * batch_ + b)] =
        d_.top_k < d_.n_experts ? r[static_cast<std::size_t>(idx[static_cast<std::size_t>(d_.top_k - 1)])] -
                                      r[static_cast<std::size_t>(idx[static_cast<std::size_t>(d_.top_k)])]
                                : 1e30;
    idx.resize(static_cast<std::size_t>(d_.top_k));
    const double m = r[static_cast<std::size_t>(idx[0])];
    double z = 0.0;
    for (i64 e : idx) z += std::exp(r[static_cast<std::size_t>(e)] - m);
    for (i64 e : idx) {
      const double w = std::exp(r[static_cast<std::size_t>(e)] - m) / z;
      swiglu_ffn(eg_[static_cast<std::size_t>(l)][static_cast<std::size_t>(e)],
                 eu_[static_cast<std::size_t>(l)][static_cast<std::size_t>(e)],
                 ed_[static_cast<std::size_t>(l)][static_cast<std::size_t>(e)], w);
    }
    routes_[static_cast<std::size_t>(l * batch_ + b)] = idx;
  }
  if (d_.ffn > 0)
    swiglu_ffn(wg_[static_cast<std::size_t>(l)], wu_[static_cast<std::size_t>(l)], wd_[static_cast<std::size_t>(l)],
               1.0);
  return y;
}

int quantize_q_e4m3_pow2(double* q, i64 n) {
  double mx = 0.0;
  for (i64 j = 0; j < n; ++j) mx = std::max(mx, std::fabs(q[j]));
  int e = 0;
  if (mx > 0.0) {
    e = static_cast<int>(std::floor(std::log2(448.0 / mx)));
    while (std::ldexp(mx, e) > 448.0) --e;
    while (std::ldexp(mx, e + 1) <= 448.0) ++e;
  }
  for (i64 j = 0; j < n; ++j) q[j] = std::ldexp(round_e4m3(std::ldexp(q[j], e)), -e);
  return e;
}

std::vector<double> ModelOracle::attend_mla(i64 l, i64 b, const std::vector<double>& a) {
  const i64 Qh = d_.query_heads, W = mla_width(d_.kv_latent), DV = mla_value_width(d_.kv_latent);
  const i64 hs = d_.head_size;
  const std::vector<double> qn = vecmat(a, wq_mla_[static_cast<std::size_t>(l)]);
  const Mat& wuk = wuk_[static_cast<std::size_t>(l)];
  Mat q(Qh, W);
  for (i64 h = 0; h < Qh; ++h)
    for (i64 j = 0; j < W; ++j) {
      double acc = 0.0;
      for (i64 dd = 0; dd < hs; ++dd) acc += qn[static_cast<std::size_t>(h * hs + dd)] * wuk(h * hs + dd, j);
      q(h, j) = round_bf16(acc);
    }
  if (kv_fp8_) {
    // FP8 latents: the query image is e4m3 of q_h * 2^e_h, e_h the largest power
    // of two keeping max |q_h| <= 448 (the GPU's absorb kernel, mla.cu Q8)
    for (i64 h = 0; h < Qh; ++h) {
      Mat qa(1, W);
      double mx = 0.0;
      for (i64 j = 0; j < W; ++j) {
        double acc = 0.0;
        for (i64 dd = 0; dd < hs; ++dd) acc += qn[static_cast<std::size_t>(h * hs + dd)] * wuk(h * hs + dd, j);
        qa(0, j) = acc;
        mx = std::max(mx, std::fabs(acc));
      }
      (void)mx;
      quantize_q_e4m3_pow2(&qa(0, 0), W);
      for (i64 j = 0; j < W; ++j) q(h, j) = qa(0, j);
    }
  }
  ShardedKVCache& cache = mla_[static_cast<std::size_t>(l * batch_ + b)];
  std::vector<AttentionFragment> frags;
  for (i64 r = 0; r < cache.kvp(); ++r) frags.push_back(shard_attention(q, cache, r, 0, 1, Qh));
  const AttentionFragment m = merge_fragments(frags);
  const Mat& wuv = wuv_[static_cast<std::size_t>(l)];
  std::vector<double> att(static_cast<std::size_t>(Qh * hs));
  for (i64 h = 0; h < Qh; ++h)
    for (i64 j = 0; j < hs; ++j) {
      double acc = 0.0;
      for (i64 dd = 0; dd < DV; ++dd) acc += m.out(h, dd) * wuv(h * DV + dd, j);
      att[static_cast<std::size_t>(h * hs + j)] = acc;
    }
  // attend-then-append: this token's latent joins the cache after the merge
  const std::vector<double> c = vecmat(a, wdkv_[static_cast<std::size_t>(l)]);
  Mat row(1, W);
  for (i64 dd = 0; dd < W; ++dd) {
    const double cv = c[static_cast<std::size_t>(dd)];
    row(0, dd) = kv_fp8_ ? round_e4m3(cv) : (bf16_ ? round_bf16(cv) : cv);
  }
  cache.append_round_robin(row, row);
  return att;
}

std::vector<double> ModelOracle::step(const std::vector<std::int64_t>& tokens,
                                      std::vector<double>* hidden,
                                      std::vector<std::int64_t>* next) {
  if (static_cast<i64>(tokens.size()) != batch_)
    throw std::invalid_argument("token batch has wrong size");
  const i64 H = d_.hidden;
  std::vector<double> logits(static_cast<std::size_t>(batch_ * d_.vocab));
  if (hidden) hidden->assign(static_cast<std::size_t>((d_.layers + 1) * batch_ * H), 0.0);
  if (next) next->assign(static_cast<std::size_t>(batch_), 0);
  for (i64 b = 0; b < batch_; ++b) {
    const std::int64_t tok = tokens[static_cast<std::size_t>(b)];
    if (tok < 0 || tok >= d_.vocab) throw std::invalid_argument("token id out of range");
    std::vector<double> x(emb_.row(tok), emb_.row(tok) + H);
    if (hidden) std::copy(x.begin(), x.end(), hidden->begin() + b * H);
    for (i64 l = 0; l < d_.layers; ++l) {
      const std::vector<double> a = rmsnorm(x);
      // [Q x Hsz] == flattened [H] (MLA: after the per-head W_UV)
      const std::vector<double> att = d_.kv_latent > 0 ? attend_mla(l, b, a) : harness(l, b).step(a).a;
      const std::vector<double> o = vecmat(att, wo_[static_cast<std::size_t>(l)]);
      std::vector<double> h(static_cast<std::size_t>(H));
      for (i64 i = 0; i < H; ++i) h[static_cast<std::size_t>(i)] = x[static_cast<std::size_t>(i)] + o[static_cast<std::size_t>(i)];
      const std::vector<double> dn = ffn(l, b, rmsnorm(h));
      for (i64 i = 0; i < H; ++i) x[static_cast<std::size_t>(i)] = h[static_cast<std::size_t>(i)] + dn[static_cast<std::size_t>(i)];
      if (hidden)
        std::copy(x.begin(), x.end(), hidden->begin() + ((l + 1) * batch_ + b) * H);
    }
    const std::vector<double> lg = vecmat(rmsnorm(x), lm_);
    std::copy(lg.begin(), lg.end(), logits.begin() + b * d_.vocab);
    if (next)
      (*next)[static_cast<std::size_t>(b)] =
          static_cast<std::int64_t>(std::max_element(lg.begin(), lg.end()) - lg.begin());
  }
  return logits;
}

}  // namespace helix_oracle
