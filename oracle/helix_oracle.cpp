// TEST INFRASTRUCTURE ONLY -- see helix_oracle.hpp.
#include "helix_oracle.hpp"

#include <algorithm>
#include <numeric>

namespace helix_oracle {

double unit_draw(std::mt19937_64& rng) {
  // attention.hpp:549-552
  const double u = static_cast<double>(rng() >> 11) * 0x1.0p-53;
  return 2.0 * u - 1.0;
}

Mat random_matrix(std::mt19937_64& rng, i64 rows, i64 cols) {
  // attention.hpp:541-546: for r, for c -> m(r, c)
  Mat m(rows, cols);
  for (i64 r = 0; r < rows; ++r)
    for (i64 c = 0; c < cols; ++c) m(r, c) = unit_draw(rng);
  return m;
}

double round_bf16(double x) {
  if (x == 0.0 || !std::isfinite(x)) return x;
  int e = 0;
  const double m = std::frexp(x, &e);            // x = m * 2^e, 0.5 <= |m| < 1
  const double r = std::nearbyint(std::ldexp(m, 8));  // 8 significant bits, RNE
  return std::ldexp(r, e - 8);
}

double round_e4m3(double x) {
  if (x == 0.0 || std::isnan(x)) return x;
  const double a = std::fabs(x);
  int e = 0;
  std::frexp(a, &e);                                   // a in [2^(e-1), 2^e)
  const int unb = std::max(e - 1, -6);                 // subnormals share the 2^-6 quantum
  const double q = std::ldexp(1.0, unb - 3);           // 3 mantissa bits
  double r = std::nearbyint(a / q) * q;                // RNE (default rounding mode)
  if (r > 448.0) r = 448.0;                            // satfinite
  return std::copysign(r, x);
}

void round_e2m1_block(double* x, i64 n) {
  double amax = 0.0;
  for (i64 i = 0; i < n; ++i) amax = std::max(amax, std::fabs(x[i]));
  int e = 0;
  if (amax > 0.0) {
    int k = 0;
    const double m = std::frexp(amax / 6.0, &k);  // amax / 6 = m 2^k, m in [0.5, 1)
    e = (m == 0.5) ? k - 1 : k;                   // smallest e with 6 2^e >= amax
    e = std::min(13, std::max(-14, e));
  }
  static const double grid[8] = {0.0, 0.5, 1.0, 1.5, 2.0, 3.0, 4.0, 6.0};
  for (i64 i = 0; i < n; ++i) {
    const double t = std::ldexp(std::fabs(x[i]), -e);
    int best = 0;
    for (int c = 1; c < 8; ++c) {  // nearest grid point; a tie goes to the even code
      const double dc = std::fabs(t - grid[c]), db = std::fabs(t - grid[best]);
      if (dc < db || (dc == db && (c & 1) == 0)) best = c;
    }
    x[i] = std::copysign(std::ldexp(grid[best], e), x[i]);
  }
}

void DecodeHarness::round_kv_rows(Mat& m) const {
  if (!kv_fp4_) {
    for (double& e : m.a) e = round_kv(e);
    return;
  }
  for (i64 r = 0; r < m.rows; ++r)
    for (i64 c0 = 0; c0 < m.cols; c0 += 32) round_e2m1_block(m.row(r) + c0, std::min<i64>(32, m.cols - c0));
}

double logit_scale(i64 width) { return 1.0 / std::sqrt(static_cast<double>(width)); }

namespace {
std::vector<double> logits_of(const std::vector<double>& q, const Mat& keys) {
  // (keys * q) * logit_scale  (attention.hpp:49, :71)
  const double s = logit_scale(static_cast<i64>(q.size()));
  std::vector<double> l(static_cast<std::size_t>(keys.rows));
  for (i64 t = 0; t < keys.rows; ++t) {
    double acc = 0.0;
    const double* k = keys.row(t);
    for (i64 d = 0; d < keys.cols; ++d) acc += k[d] * q[static_cast<std::size_t>(d)];
    l[static_cast<std::size_t>(t)] = acc * s;
  }
  return l;
}
}  // namespace

std::vector<double> reference_attention(const std::vector<double>& q, const Mat& keys,
                                        const Mat& values) {
  // attention.hpp:43-53
  if (keys.rows == 0) throw std::invalid_argument("attention needs >= 1 context token");
  if (keys.rows != values.rows || keys.cols != static_cast<i64>(q.size()) ||
      values.cols != static_cast<i64>(q.size()))
    throw std::invalid_argument("mismatched attention operand shapes");
  std::vector<double> l = logits_of(q, keys);
  const double m = *std::max_element(l.begin(), l.end());
  double z = 0.0;
  for (double& v : l) v = std::exp(v - m);
  for (double v : l) z += v;
  std::vector<double> out(q.size(), 0.0);
  for (i64 d = 0; d < values.cols; ++d) {
    double acc = 0.0;
    for (i64 t = 0; t < values.rows; ++t) acc += values(t, d) * l[static_cast<std::size_t>(t)];
    out[static_cast<std::size_t>(d)] = acc / z;
  }
  return out;
}

HeadFragment partial_head_attention(const std::vector<double>& q, const Mat& keys,
                                    const Mat& values) {
  // attention.hpp:65-78: empty shard -> (0, -inf)
  HeadFragment f;
  f.out.assign(q.size(), 0.0);
  if (keys.rows == 0) return f;
  std::vector<double> l = logits_of(q, keys);
  const double m = *std::max_element(l.begin(), l.end());
  for (double& v : l) v = std::exp(v - m);
  double z = 0.0;
  for (double v : l) z += v;
  for (i64 d = 0; d < values.cols; ++d) {
    double acc = 0.0;
    for (i64 t = 0; t < values.rows; ++t) acc += values(t, d) * l[static_cast<std::size_t>(t)];
    f.out[static_cast<std::size_t>(d)] = acc / z;
  }
  f.lse = m + std::log(z);
  return f;
}

std::vector<std::size_t> canonical_order(std::span<const HeadFragment> frags) {
  // attention.hpp:90-102: descending lse, ties by first differing coefficient
  std::vector<std::size_t> idx(frags.size());
  std::iota(idx.begin(), idx.end(), std::size_t{0});
  std::sort(idx.begin(), idx.end(), [&](std::size_t a, std::size_t b) {
    if (frags[a].lse != frags[b].lse) return frags[a].lse > frags[b].lse;
    const auto& oa = frags[a].out;
    const auto& ob = frags[b].out;
    for (std::size_t i = 0; i < oa.size() && i < ob.size(); ++i)
      if (oa[i] != ob[i]) return oa[i] < ob[i];
    return oa.size() < ob.size();
  });
  return idx;
}

HeadFragment merge_head_fragments(std::span<const HeadFragment> frags) {
  // attention.hpp:118-137
  if (frags.empty()) throw std::invalid_argument("merge needs >= 1 fragment");
  const std::vector<std::size_t> order = canonical_order(frags);
  const double m = frags[order.front()].lse;
  if (m == neg_inf()) throw std::invalid_argument("all fragments empty: nothing to merge");
  const std::size_t width = frags[order.front()].out.size();
  std::vector<double> acc(width, 0.0);
  double z = 0.0;
  for (std::size_t i : order) {
    if (frags[i].out.size() != width) throw std::invalid_argument("fragment widths differ");
    if (frags[i].lse == neg_inf()) continue;
    const double w = std::exp(frags[i].lse - m);
    for (std::size_t d = 0; d < width; ++d) acc[d] += w * frags[i].out[d];
    z += w;
  }
  HeadFragment out;
  out.out.resize(width);
  for (std::size_t d = 0; d < width; ++d) out.out[d] = acc[d] / z;
  out.lse = m + std::log(z);
  return out;
}

// ---------------------------------------------------------------------------

ShardedKVCache::ShardedKVCache(i64 kvp, i64 kv_heads, i64 head_width, i64 chunk_size)
    : kvp_(kvp), kv_heads_(kv_heads), w_(head_width), chunk_(chunk_size) {
  // attention.hpp:235-248
  if (kvp < 1 || kv_heads < 1 || head_width < 1 || chunk_size < 1)
    throw std::invalid_argument("cache dimensions must be >= 1");
  k_.assign(static_cast<std::size_t>(kvp * kv_heads), Mat(0, head_width));
  v_.assign(static_cast<std::size_t>(kvp * kv_heads), Mat(0, head_width));
  counts_.assign(static_cast<std::size_t>(kvp), 0);
}

void ShardedKVCache::push_row(i64 rank, i64 head, const double* k, const double* v) {
  Mat& K = k_[idx(rank, head)];
  Mat& V = v_[idx(rank, head)];
  K.a.insert(K.a.end(), k, k + w_);
  V.a.insert(V.a.end(), v, v + w_);
  ++K.rows;
  ++V.rows;
}

void ShardedKVCache::append_round_robin(const Mat& k, const Mat& v) {
  // attention.hpp:262-282. Chunks are a storage detail of the reference; the
  // observable state is the per-rank row order, the cursor and token_order.
  if (k.rows != kv_heads_ || v.rows != kv_heads_ || k.cols != w_ || v.cols != w_)
    throw std::invalid_argument("appended token has wrong shape");
  for (i64 h = 0; h < kv_heads_; ++h) push_row(cursor_, h, k.row(h), v.row(h));
  order_.push_back({cursor_, counts_[static_cast<std::size_t>(cursor_)]++});
  ++fill_;
  if (fill_ == chunk_) {
    fill_ = 0;
    cursor_ = (cursor_ + 1) % kvp_;
  }
}

i64 ShardedKVCache::max_min_gap() const {
  // attention.hpp:286-294
  i64 lo = std::numeric_limits<i64>::max(), hi = 0;
  for (i64 c : counts_) {
    lo = std::min(lo, c);
    hi = std::max(hi, c);
  }
  return hi - lo;
}

void ShardedKVCache::global_context(i64 head, Mat& keys, Mat& values) const {
  // attention.hpp:312-327
  keys = Mat(total_tokens(), w_);
  values = Mat(total_tokens(), w_);
  std::vector<i64> next(static_cast<std::size_t>(kvp_), 0);
  for (i64 g = 0; g < total_tokens(); ++g) {
    const TokenRef& t = order_[static_cast<std::size_t>(g)];
    const i64 row = next[static_cast<std::size_t>(t.rank)]++;
    const Mat& K = k_[idx(t.rank, head)];
    const Mat& V = v_[idx(t.rank, head)];
    std::copy(K.row(row), K.row(row) + w_, keys.row(g));
    std::copy(V.row(row), V.row(row) + w_, values.row(g));
  }
}

ShardedKVCache ShardedKVCache::from_partition(i64 kvp, const std::vector<Mat>& keys,
                                              const std::vector<Mat>& values,
                                              const std::vector<i64>& rank_of_token,
                                              i64 chunk) {
  // attention.hpp:332-359
  if (keys.empty() || keys.size() != values.size())
    throw std::invalid_argument("need matching per-head key/value matrices");
  ShardedKVCache c(kvp, static_cast<i64>(keys.size()), keys.front().cols, chunk);
  for (std::size_t g = 0; g < rank_of_token.size(); ++g) {
    const i64 r = rank_of_token[g];
    if (r < 0 || r >= kvp) throw std::invalid_argument("token rank out of range");
    for (i64 h = 0; h < c.kv_heads_; ++h)
      c.push_row(r, h, keys[static_cast<std::size_t>(h)].row(static_cast<i64>(g)),
                 values[static_cast<std::size_t>(h)].row(static_cast<i64>(g)));
    c.order_.push_back({r, c.counts_[static_cast<std::size_t>(r)]++});
  }
  return c;
}

AttentionFragment shard_attention(const Mat& queries, const ShardedKVCache& cache, i64 rank,
                                  i64 kv_head_offset, i64 kv_head_count, i64 q_per_kv) {
  // attention.hpp:375-396
  if (queries.rows != kv_head_count * q_per_kv)
    throw std::invalid_argument("query rows must equal kv_head_count * q_per_kv");
  AttentionFragment f;
  f.out = Mat(queries.rows, queries.cols);
  f.lse.assign(static_cast<std::size_t>(queries.rows), neg_inf());
  for (i64 h = 0; h < kv_head_count; ++h) {
    const Mat& K = cache.keys(rank, kv_head_offset + h);
    const Mat& V = cache.values(rank, kv_head_offset + h);
    for (i64 qi = 0; qi < q_per_kv; ++qi) {
      const i64 row = h * q_per_kv + qi;
      std::vector<double> q(queries.row(row), queries.row(row) + queries.cols);
      HeadFragment hf = partial_head_attention(q, K, V);
      std::copy(hf.out.begin(), hf.out.end(), f.out.row(row));
      f.lse[static_cast<std::size_t>(row)] = hf.lse;
    }
  }
  return f;
}

AttentionFragment merge_fragments(std::span<const AttentionFragment> frags) {
  // attention.hpp:155-175
  if (frags.empty()) throw std::invalid_argument("merge needs >= 1 fragment");
  const i64 heads = frags.front().out.rows, width = frags.front().out.cols;
  AttentionFragment m;
  m.out = Mat(heads, width);
  m.lse.resize(static_cast<std::size_t>(heads));
  std::vector<HeadFragment> per_head(frags.size());
  for (i64 h = 0; h < heads; ++h) {
    for (std::size_t i = 0; i < frags.size(); ++i) {
      if (frags[i].out.rows != heads || static_cast<i64>(frags[i].lse.size()) != heads)
        throw std::invalid_argument("fragment head counts differ");
      per_head[i].out.assign(frags[i].out.row(h), frags[i].out.row(h) + frags[i].out.cols);
      per_head[i].lse = frags[i].lse[static_cast<std::size_t>(h)];
    }
    HeadFragment hm = merge_head_fragments(per_head);
    std::copy(hm.out.begin(), hm.out.end(), m.out.row(h));
    m.lse[static_cast<std::size_t>(h)] = hm.lse;
  }
  return m;
}

// ---------------------------------------------------------------------------

namespace {
void maybe_round(Mat& m, bool on) {
  if (on)
    for (double& v : m.a) v = round_bf16(v);
}
}  // namespace

DecodeHarness::DecodeHarness(Dims dims, i64 tpa, i64 kvp, i64 chunk_size, std::uint64_t seed,
                             bool bf16_storage)
    : dims_(dims), tpa_(tpa), kvp_(kvp), bf16_(bf16_storage),
      cache_(kvp, dims.kv_heads, dims.head_size, chunk_size) {
  // attention.hpp:428-443 (the cache ctor above validates the cache dims first)
  if (tpa < 1 || kvp < 1) throw std::invalid_argument("tpa and kvp must be >= 1");
  if (dims.query_heads % dims.kv_heads != 0)
    throw std::invalid_argument("query_heads must be a multiple of kv_heads");
  if (dims.kv_heads % tpa != 0) throw std::invalid_argument("tpa must divide kv_heads");
  if (dims.hidden() % (tpa * kvp) != 0)
    throw std::invalid_argument("tpa*kvp must divide the hidden width");
  std::mt19937_64 rng(seed);
  const i64 h = dims.hidden();
  wq_ = random_matrix(rng, h, dims.query_heads * dims.head_size);
  wk_ = random_matrix(rng, h, dims.kv_heads * dims.head_size);
  wv_ = random_matrix(rng, h, dims.kv_heads * dims.head_size);
  maybe_round(wq_, bf16_);
  maybe_round(wk_, bf16_);
  maybe_round(wv_, bf16_);
}

void DecodeHarness::grow_random(i64 n, std::mt19937_64& rng) {
  // attention.hpp:452-456. The reference writes
  //   append_round_robin(random_matrix(rng,..), random_matrix(rng,..))
  // and g++ evaluates the two arguments right to left, so V is drawn
  // BEFORE K for every token (verified against the reference build in
  // tests/test_oracle_golden.py). This order is part of the contract.
  for (i64 i = 0; i < n; ++i) {
    Mat v = random_matrix(rng, dims_.kv_heads, dims_.head_size);
    Mat k = random_matrix(rng, dims_.kv_heads, dims_.head_size);
    round_kv_rows(k);
    round_kv_rows(v);
    cache_.append_round_robin(k, v);
  }
}

std::vector<double> DecodeHarness::project_q(const std::vector<double>& x) const {
  // q_head = x^T W_q[:, head*Hsz:(head+1)*Hsz] for every head (attention.hpp:479-484)
  const i64 h = dims_.hidden(), n = dims_.query_heads * dims_.head_size;
  std::vector<double> q(static_cast<std::size_t>(n), 0.0);
  for (i64 c = 0; c < n; ++c) {
    double acc = 0.0;
    for (i64 k = 0; k < h; ++k) acc += x[static_cast<std::size_t>(k)] * wq_(k, c);
    q[static_cast<std::size_t>(c)] = acc;
  }
  return q;
}

void DecodeHarness::project_kv(const std::vector<double>& x, Mat& k, Mat& v) const {
  // attention.hpp:531-538
  const i64 h = dims_.hidden();
  k = Mat(dims_.kv_heads, dims_.head_size);
  v = Mat(dims_.kv_heads, dims_.head_size);
  for (i64 kh = 0; kh < dims_.kv_heads; ++kh)
    for (i64 d = 0; d < dims_.head_size; ++d) {
      const i64 c = kh * dims_.head_size + d;
      double ak = 0.0, av = 0.0;
      for (i64 i = 0; i < h; ++i) {
        ak += x[static_cast<std::size_t>(i)] * wk_(i, c);
        av += x[static_cast<std::size_t>(i)] * wv_(i, c);
      }
      k(kh, d) = ak;
      v(kh, d) = av;
    }
}

void DecodeHarness::append_projected(const std::vector<double>& x) {
  Mat k, v;
  project_kv(x, k, v);
  round_kv_rows(k);
  round_kv_rows(v);
  cache_.append_round_robin(k, v);
}

Mat DecodeHarness::step(const std::vector<double>& x) { return step_with_append(x, nullptr, nullptr); }

Mat DecodeHarness::step_with_append(const std::vector<double>& x, const Mat* k_over, const Mat* v_over) {
  // attention.hpp:460-510 -- attend, exchange, merge, THEN append
  if (static_cast<i64>(x.size()) != dims_.hidden())
    throw std::invalid_argument("hidden state has wrong width");
  if (cache_.total_tokens() == 0) throw std::invalid_argument("decode needs a nonempty context");
  for (i64 r = 1; r < pool(); ++r)
    transcript_.push_back({MsgKind::Broadcast, 0, r, dims_.hidden(), 0});

  const i64 kv_per_group = dims_.kv_heads / tpa_;
  const i64 q_per_kv = dims_.query_heads / dims_.kv_heads;
  const i64 q_per_group = kv_per_group * q_per_kv;
  const i64 group_width = q_per_group * dims_.head_size;
  const i64 slice = group_width / kvp_;
  const std::vector<double> qall = project_q(x);

  Mat out(dims_.query_heads, dims_.head_size);
  last_lse_.assign(static_cast<std::size_t>(dims_.query_heads), neg_inf());
  for (i64 g = 0; g < tpa_; ++g) {
    Mat queries(q_per_group, dims_.head_size);
    for (i64 qi = 0; qi < q_per_group; ++qi) {
      const i64 head = g * q_per_group + qi;
      for (i64 d = 0; d < dims_.head_size; ++d)
        queries(qi, d) = qall[static_cast<std::size_t>(head * dims_.head_size + d)];
    }
    std::vector<AttentionFragment> frags;
    for (i64 r = 0; r < kvp_; ++r)
      frags.push_back(shard_attention(queries, cache_, r, g * kv_per_group, kv_per_group, q_per_kv));
    for (i64 r = 0; r < kvp_; ++r)
      for (i64 p = 0; p < kvp_; ++p) {
        if (p == r) continue;
        const i64 first_head = p * slice / dims_.head_size;
        const i64 last_head = ((p + 1) * slice - 1) / dims_.head_size;
        transcript_.push_back(
            {MsgKind::AllToAll, rank_id(r, g), rank_id(p, g), slice, last_head - first_head + 1});
      }
    AttentionFragment merged = merge_fragments(frags);
    for (i64 qi = 0; qi < q_per_group; ++qi) {
      std::copy(merged.out.row(qi), merged.out.row(qi) + dims_.head_size,
                out.row(g * q_per_group + qi));
      last_lse_[static_cast<std::size_t>(g * q_per_group + qi)] =
          merged.lse[static_cast<std::size_t>(qi)];
    }
  }
  if (k_over && v_over)
    cache_.append_round_robin(*k_over, *v_over);
  else
    append_projected(x);
  return out;
}

Mat DecodeHarness::reference(const std::vector<double>& x) const {
  // attention.hpp:514-529
  Mat out(dims_.query_heads, dims_.head_size);
  const i64 q_per_kv = dims_.query_heads / dims_.kv_heads;
  const std::vector<double> qall = project_q(x);
  for (i64 kh = 0; kh < dims_.kv_heads; ++kh) {
    Mat K, V;
    cache_.global_context(kh, K, V);
    for (i64 qi = 0; qi < q_per_kv; ++qi) {
      const i64 head = kh * q_per_kv + qi;
      std::vector<double> q(qall.begin() + head * dims_.head_size,
                            qall.begin() + (head + 1) * dims_.head_size);
      std::vector<double> o = reference_attention(q, K, V);
      std::copy(o.begin(), o.end(), out.row(head));
    }
  }
  return out;
}

}  // namespace helix_oracle
