// helixsim/exact_b200.hpp -- drop-in C++ surface of the reference's
// helixsim::exact decode path (/root/reference/proj/include/helixsim/
// attention.hpp:20-563) backed by the B200 library (include/helix_b200.h,
// libhelix_b200.so).
//
// Swap `#include "helixsim/attention.hpp"` for this header (or put a
// one-line helixsim/attention.hpp that includes it ahead of the reference's on
// the include path, as tests/cpp/dropin/ does) and link libhelix_b200.so:
// the names, argument meaning, value semantics of the results and the
// std::invalid_argument messages are the reference's. Every numeric operation
// runs on the GPU:
//   * free functions (reference_attention, partial_head_attention,
//     merge_head_fragments, merge_fragments, shard_attention) -> the fp64
//     kernels behind hx_attention_f64 / hx_merge_f64;
//   * DecodeHarness<Scalar> -> a device-resident engine. Storage::exact
//     (default) keeps weights, KV shards, projections and merges in fp64
//     (HX_KV_F64), i.e. the reference's precision and tolerances;
//     Storage::bf16 is the production decode path (bf16 pages, fp32
//     accumulation; reference() / append_projected() need Storage::exact).
// ShardedKVCache is the reference's host-side container semantics (round-robin
// bookkeeping, trimmed per-rank contexts, global order); DecodeHarness::cache()
// returns a snapshot of the engine's device-resident cache in that form.
// Like the reference, Matrix/Vector are Eigen types (Eigen 3.3+).
#pragma once

#include <Eigen/Dense>
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <limits>
#include <memory>
#include <random>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "../helix_b200.h"

namespace helixsim {
using i64 = std::int64_t;

namespace exact {

template <class Scalar>
using Matrix = Eigen::Matrix<Scalar, Eigen::Dynamic, Eigen::Dynamic>;
template <class Scalar>
using Vector = Eigen::Matrix<Scalar, Eigen::Dynamic, 1>;

template <class Scalar>
constexpr Scalar neg_inf() {
  return -std::numeric_limits<Scalar>::infinity();
}

template <class Scalar>
Scalar logit_scale(Eigen::Index head_width) {
  return Scalar(1) / std::sqrt(static_cast<Scalar>(head_width));
}

namespace b200 {
inline void check(int rc, const hx_engine* e) {
  if (rc == HX_OK) return;
  const std::string msg = hx_last_error(e);
  if (rc == HX_ERR_INVALID) throw std::invalid_argument(msg);  // the reference's exceptions
  throw std::runtime_error(msg);
}
// Row-major fp64 image of any Eigen expression (rows x cols).
template <class M>
std::vector<double> row_major(const M& m) {
  std::vector<double> out(static_cast<std::size_t>(m.rows() * m.cols()));
  for (Eigen::Index r = 0; r < m.rows(); ++r)
    for (Eigen::Index c = 0; c < m.cols(); ++c)
      out[static_cast<std::size_t>(r * m.cols() + c)] = static_cast<double>(m(r, c));
  return out;
}
template <class Scalar>
Matrix<Scalar> from_row_major(const double* p, i64 rows, i64 cols) {
  Matrix<Scalar> m(rows, cols);
  for (i64 r = 0; r < rows; ++r)
    for (i64 c = 0; c < cols; ++c) m(r, c) = static_cast<Scalar>(p[r * cols + c]);
  return m;
}
// nq queries (rows of q_rows, q_rows x w) over one K/V (tokens x w) on the GPU.
template <class Scalar>
void attend(const std::vector<double>& q_rows, i64 nq, const Matrix<Scalar>& keys, const Matrix<Scalar>& values,
            i64 w, std::vector<double>& out, std::vector<double>& lse) {
  const std::vector<double> k = row_major(keys), v = row_major(values);
  out.assign(static_cast<std::size_t>(nq * w), 0.0);
  lse.assign(static_cast<std::size_t>(nq), 0.0);
  check(hx_attention_f64(q_rows.data(), nq, k.data(), v.data(), keys.rows(), w, out.data(), lse.data()), nullptr);
}
}  // namespace b200

// ---------------------------------------------------------------------------
// Single-head primitives (attention.hpp:35-78)

template <class Scalar>
Vector<Scalar> reference_attention(const Vector<Scalar>& q, const Matrix<Scalar>& keys,
                                   const Matrix<Scalar>& values) {
  if (keys.rows() == 0) throw std::invalid_argument("attention needs >= 1 context token");
  if (keys.rows() != values.rows() || keys.cols() != q.size() || values.cols() != q.size())
    throw std::invalid_argument("mismatched attention operand shapes");
  std::vector<double> out, lse;
  b200::attend<Scalar>(b200::row_major(q), 1, keys, values, q.size(), out, lse);
  return b200::from_row_major<Scalar>(out.data(), q.size(), 1);
}

template <class Scalar>
struct HeadFragment {
  Vector<Scalar> partial_out;
  Scalar lse = neg_inf<Scalar>();
};

template <class Scalar>
HeadFragment<Scalar> partial_head_attention(const Vector<Scalar>& q, const Matrix<Scalar>& keys,
                                            const Matrix<Scalar>& values) {
  HeadFragment<Scalar> frag;
  frag.partial_out = Vector<Scalar>::Zero(q.size());
  if (keys.rows() == 0) return frag;  // identity element: (0, -inf)
  if (keys.rows() != values.rows() || keys.cols() != q.size() || values.cols() != q.size())
    throw std::invalid_argument("mismatched attention operand shapes");
  std::vector<double> out, lse;
  b200::attend<Scalar>(b200::row_major(q), 1, keys, values, q.size(), out, lse);
  frag.partial_out = b200::from_row_major<Scalar>(out.data(), q.size(), 1);
  frag.lse = static_cast<Scalar>(lse[0]);
  return frag;
}

// ---------------------------------------------------------------------------
// Merging (attention.hpp:80-175): canonical order on the GPU (descending lse,
// ties by the first differing coefficient), so the result is a pure function
// of the fragment set.

template <class Scalar>
struct MergedHead {
  Vector<Scalar> out;
  Scalar lse = neg_inf<Scalar>();
};

template <class Scalar>
MergedHead<Scalar> merge_head_fragments(std::span<const HeadFragment<Scalar>> frags) {
  if (frags.empty()) throw std::invalid_argument("merge needs >= 1 fragment");
  bool any = false;
  for (const auto& f : frags) any |= f.lse != neg_inf<Scalar>();
  if (!any) throw std::invalid_argument("all fragments empty: nothing to merge");
  const Eigen::Index width = frags.front().partial_out.size();
  for (const auto& f : frags)
    if (f.partial_out.size() != width) throw std::invalid_argument("fragment widths differ");
  std::vector<double> outs, lses;
  for (const auto& f : frags) {
    for (Eigen::Index i = 0; i < width; ++i) outs.push_back(static_cast<double>(f.partial_out[i]));
    lses.push_back(static_cast<double>(f.lse));
  }
  std::vector<double> out(static_cast<std::size_t>(width));
  double lse = 0.0;
  b200::check(hx_merge_f64(static_cast<i64>(frags.size()), width, outs.data(), lses.data(), out.data(), &lse),
              nullptr);
  return {b200::from_row_major<Scalar>(out.data(), width, 1), static_cast<Scalar>(lse)};
}

template <class Scalar>
struct AttentionFragment {
  Matrix<Scalar> partial_out;  // query heads x head size
  Vector<Scalar> lse;          // one scalar per query head
};

template <class Scalar>
struct MergedAttention {
  Matrix<Scalar> out;
  Vector<Scalar> lse;
};

template <class Scalar>
MergedAttention<Scalar> merge_fragments(std::span<const AttentionFragment<Scalar>> frags) {
  if (frags.empty()) throw std::invalid_argument("merge needs >= 1 fragment");
  const Eigen::Index heads = frags.front().partial_out.rows();
  const Eigen::Index width = frags.front().partial_out.cols();
  for (const auto& f : frags)
    if (f.partial_out.rows() != heads || f.lse.size() != heads)
      throw std::invalid_argument("fragment head counts differ");
  MergedAttention<Scalar> merged;
  merged.out.resize(heads, width);
  merged.lse.resize(heads);
  std::vector<HeadFragment<Scalar>> per_head(frags.size());
  for (Eigen::Index h = 0; h < heads; ++h) {
    for (std::size_t i = 0; i < frags.size(); ++i) {
      per_head[i].partial_out = frags[i].partial_out.row(h).transpose();
      per_head[i].lse = frags[i].lse[h];
    }
    const MergedHead<Scalar> m = merge_head_fragments<Scalar>(per_head);
    merged.out.row(h) = m.out.transpose();
    merged.lse[h] = m.lse;
  }
  return merged;
}

// ---------------------------------------------------------------------------
// Sharded KV cache (attention.hpp:182-369): host-side container with the
// reference's round-robin semantics. Each (rank, head) keeps its rows in
// append order, row-major.

template <class Scalar>
struct KvChunk {
  Matrix<Scalar> keys;    // tokens x width
  Matrix<Scalar> values;  // tokens x width
};

struct TokenRef {
  i64 rank;
  i64 row;  // position within the shard's concatenated sequence
};

template <class Scalar>
class DecodeHarness;

template <class Scalar>
class ShardedKVCache {
 public:
  ShardedKVCache(i64 kvp, i64 kv_heads, i64 head_width, i64 chunk_size = 16)
      : kvp_(kvp), heads_(kv_heads), width_(head_width), chunk_(chunk_size) {
    if (kvp < 1 || kv_heads < 1 || head_width < 1 || chunk_size < 1)
      throw std::invalid_argument("cache dimensions must be >= 1");
    k_.assign(static_cast<std::size_t>(kvp * kv_heads), {});
    v_.assign(static_cast<std::size_t>(kvp * kv_heads), {});
    count_.assign(static_cast<std::size_t>(kvp), 0);
  }

  i64 kvp() const { return kvp_; }
  i64 kv_heads() const { return heads_; }
  i64 head_width() const { return width_; }
  i64 chunk_size() const { return chunk_; }
  i64 total_tokens() const { return static_cast<i64>(order_.size()); }
  const std::vector<TokenRef>& token_order() const { return order_; }
  i64 effective_tokens(i64 rank) const { return count_.at(static_cast<std::size_t>(rank)); }

  // Row h of k / v feeds KV head h; chunk_size tokens per rank, then the next rank.
  void append_round_robin(const Matrix<Scalar>& k, const Matrix<Scalar>& v) {
    if (k.rows() != heads_ || v.rows() != heads_ || k.cols() != width_ || v.cols() != width_)
      throw std::invalid_argument("appended token has wrong shape");
    push(cursor_, k, v);
    if (++fill_ == chunk_) {
      fill_ = 0;
      cursor_ = (cursor_ + 1) % kvp_;
    }
  }

  i64 max_min_gap() const {
    const auto [lo, hi] = std::minmax_element(count_.begin(), count_.end());
    return *hi - *lo;
  }

  KvChunk<Scalar> context(i64 rank, i64 head) const {
    if (rank < 0 || rank >= kvp_ || head < 0 || head >= heads_) throw std::out_of_range("rank or head out of range");
    const std::size_t s = slot(rank, head);
    const i64 n = count_[static_cast<std::size_t>(rank)];
    return {b200::from_row_major<Scalar>(k_[s].data(), n, width_),
            b200::from_row_major<Scalar>(v_[s].data(), n, width_)};
  }

  KvChunk<Scalar> global_context(i64 head) const {
    KvChunk<Scalar> out{Matrix<Scalar>(total_tokens(), width_), Matrix<Scalar>(total_tokens(), width_)};
    for (i64 g = 0; g < total_tokens(); ++g) {
      const TokenRef& t = order_[static_cast<std::size_t>(g)];
      const std::size_t s = slot(t.rank, head);
      for (i64 d = 0; d < width_; ++d) {
        out.keys(g, d) = static_cast<Scalar>(k_[s][static_cast<std::size_t>(t.row * width_ + d)]);
        out.values(g, d) = static_cast<Scalar>(v_[s][static_cast<std::size_t>(t.row * width_ + d)]);
      }
    }
    return out;
  }

  // Explicit token -> rank assignment; keys/values: one matrix per KV head, rows in global order.
  static ShardedKVCache from_partition(i64 kvp, std::span<const Matrix<Scalar>> keys,
                                       std::span<const Matrix<Scalar>> values, std::span<const i64> rank_of_token,
                                       i64 chunk_size = 16) {
    if (keys.empty() || keys.size() != values.size())
      throw std::invalid_argument("need matching per-head key/value matrices");
    ShardedKVCache cache(kvp, static_cast<i64>(keys.size()), keys.front().cols(), chunk_size);
    Matrix<Scalar> k(cache.heads_, cache.width_), v(cache.heads_, cache.width_);
    for (std::size_t g = 0; g < rank_of_token.size(); ++g) {
      const i64 r = rank_of_token[g];
      if (r < 0 || r >= kvp) throw std::invalid_argument("token rank out of range");
      for (i64 h = 0; h < cache.heads_; ++h) {
        k.row(h) = keys[static_cast<std::size_t>(h)].row(static_cast<Eigen::Index>(g));
        v.row(h) = values[static_cast<std::size_t>(h)].row(static_cast<Eigen::Index>(g));
      }
      cache.push(r, k, v);
    }
    return cache;
  }

 private:
  friend class DecodeHarness<Scalar>;
  std::size_t slot(i64 rank, i64 head) const { return static_cast<std::size_t>(rank * heads_ + head); }
  void push(i64 rank, const Matrix<Scalar>& k, const Matrix<Scalar>& v) {
    for (i64 h = 0; h < heads_; ++h)
      for (i64 d = 0; d < width_; ++d) {
        k_[slot(rank, h)].push_back(static_cast<double>(k(h, d)));
        v_[slot(rank, h)].push_back(static_cast<double>(v(h, d)));
      }
    order_.push_back({rank, count_[static_cast<std::size_t>(rank)]++});
  }
  i64 kvp_, heads_, width_, chunk_;
  i64 cursor_ = 0, fill_ = 0;
  std::vector<std::vector<double>> k_, v_;  // [rank][head] -> rows x width
  std::vector<i64> count_;
  std::vector<TokenRef> order_;
};

// One rank's shard attention for a contiguous group of query heads (attention.hpp:375-396).
template <class Scalar>
AttentionFragment<Scalar> shard_attention(const Matrix<Scalar>& queries, const ShardedKVCache<Scalar>& cache,
                                          i64 rank, i64 kv_head_offset, i64 kv_head_count, i64 q_per_kv) {
  if (queries.rows() != kv_head_count * q_per_kv)
    throw std::invalid_argument("query rows must equal kv_head_count * q_per_kv");
  AttentionFragment<Scalar> frag;
  frag.partial_out = Matrix<Scalar>::Zero(queries.rows(), queries.cols());
  frag.lse.resize(queries.rows());
  const i64 w = queries.cols();
  for (i64 h = 0; h < kv_head_count; ++h) {
    const KvChunk<Scalar> ctx = cache.context(rank, kv_head_offset + h);
    if (ctx.keys.rows() == 0) {
      for (i64 qi = 0; qi < q_per_kv; ++qi) frag.lse[h * q_per_kv + qi] = neg_inf<Scalar>();
      continue;
    }
    std::vector<double> q = b200::row_major(queries.middleRows(h * q_per_kv, q_per_kv));
    std::vector<double> out, lse;
    b200::attend<Scalar>(q, q_per_kv, ctx.keys, ctx.values, w, out, lse);
    for (i64 qi = 0; qi < q_per_kv; ++qi) {
      for (i64 d = 0; d < w; ++d)
        frag.partial_out(h * q_per_kv + qi, d) = static_cast<Scalar>(out[static_cast<std::size_t>(qi * w + d)]);
      frag.lse[h * q_per_kv + qi] = static_cast<Scalar>(lse[static_cast<std::size_t>(qi)]);
    }
  }
  return frag;
}

// ---------------------------------------------------------------------------
// Decode-step harness (attention.hpp:398-563)

enum class MsgKind { Broadcast, AllToAll };

struct Message {
  MsgKind kind;
  i64 src;
  i64 dst;
  i64 payload_scalars;
  i64 lse_scalars;
};

enum class Storage { exact, bf16 };

struct HarnessOptions {
  Storage storage = Storage::exact;  // exact: fp64 on the GPU (HX_KV_F64); bf16: production pages
  i64 capacity = 1 << 16;            // max context tokens (the reference grows without bound)
  int device = 0;
};

template <class Scalar>
class DecodeHarness {
 public:
  struct Dims {
    i64 query_heads;
    i64 kv_heads;
    i64 head_size;
    i64 hidden() const { return query_heads * head_size; }
  };

  DecodeHarness(Dims dims, i64 tpa, i64 kvp, i64 chunk_size, std::uint64_t seed, HarnessOptions opt = {})
      : dims_(dims), tpa_(tpa), kvp_(kvp), chunk_(chunk_size), opt_(opt) {
    hx_model_config m{};
    m.hidden = dims.hidden();
    m.query_heads = dims.query_heads;
    m.kv_heads = dims.kv_heads;
    m.head_size = dims.head_size;
    m.ffn = 16;
    m.layers = 1;
    m.vocab = 1;
    m.attention_only = 1;
    hx_parallel_config p{};
    p.tpa = tpa;
    p.kvp = kvp;
    p.chunk_size = chunk_size;
    hx_runtime_config r{};
    r.batch = 1;
    r.capacity_tokens = opt.capacity;
    r.device = opt.device;
    r.kv_dtype = opt.storage == Storage::exact ? HX_KV_F64 : HX_KV_BF16;
    b200::check(hx_engine_create(&m, &p, &r, &e_), nullptr);
    // W_q, W_k, W_v drawn from mt19937_64(seed) in that order (attention.hpp:438-442)
    b200::check(hx_init_weights_mt19937(e_, seed), e_);
  }
  ~DecodeHarness() { hx_engine_destroy(e_); }
  DecodeHarness(const DecodeHarness&) = delete;
  DecodeHarness& operator=(const DecodeHarness&) = delete;

  i64 pool() const { return tpa_ * kvp_; }

  // Snapshot of the device-resident cache in the reference's container form.
  const ShardedKVCache<Scalar>& cache() const {
    snapshot_ = make_snapshot();  // detached copy: appending to it does not touch the engine
    return *snapshot_;
  }

  const std::vector<Message>& transcript() const {
    const i64 n = hx_transcript_size(e_);
    std::vector<std::int64_t> raw(static_cast<std::size_t>(5 * n));
    if (n) b200::check(hx_transcript(e_, raw.data()), e_);
    transcript_.clear();
    for (i64 i = 0; i < n; ++i) {
      const std::int64_t* r = raw.data() + 5 * i;
      transcript_.push_back({r[0] == 0 ? MsgKind::Broadcast : MsgKind::AllToAll, r[1], r[2], r[3], r[4]});
    }
    return transcript_;
  }

  // n random tokens, V drawn before K for each (attention.hpp:452-456 under g++),
  // from the caller's generator -- which advances exactly as the reference's does.
  void grow_random(i64 n, std::mt19937_64& rng) {
    const i64 per = dims_.kv_heads * dims_.head_size;
    const i64 block = 4096;
    std::vector<double> k, v;
    for (i64 done = 0; done < n; done += block) {
      const i64 m = std::min(block, n - done);
      k.resize(static_cast<std::size_t>(m * per));
      v.resize(static_cast<std::size_t>(m * per));
      for (i64 t = 0; t < m; ++t) {
        for (i64 j = 0; j < per; ++j) v[static_cast<std::size_t>(t * per + j)] = unit_draw(rng);
        for (i64 j = 0; j < per; ++j) k[static_cast<std::size_t>(t * per + j)] = unit_draw(rng);
      }
      append_rows(m, k.data(), v.data());
    }
  }

  // attention.hpp:460-510: merged attention output (query heads x head size),
  // then x's projected K/V is appended (attend-then-append).
  Matrix<Scalar> step(const Vector<Scalar>& x) {
    const std::vector<double> xd = b200::row_major(x);
    std::vector<double> out(static_cast<std::size_t>(dims_.hidden()));
    if (opt_.storage == Storage::exact) {
      b200::check(hx_harness_step_f64(e_, 0, xd.data(), x.size(), out.data(), nullptr), e_);
    } else {
      std::vector<float> xf(xd.begin(), xd.end()), of(out.size());
      b200::check(hx_harness_step(e_, 0, xf.data(), x.size(), of.data(), nullptr), e_);
      std::copy(of.begin(), of.end(), out.begin());
    }
    return b200::from_row_major<Scalar>(out.data(), dims_.query_heads, dims_.head_size);
  }

  // attention.hpp:514-529: monolithic attention over the global context, no append.
  Matrix<Scalar> reference(const Vector<Scalar>& x) const {
    require_exact("reference");
    const std::vector<double> xd = b200::row_major(x);
    std::vector<double> out(static_cast<std::size_t>(dims_.hidden()));
    b200::check(hx_harness_reference_f64(e_, 0, xd.data(), x.size(), out.data()), e_);
    return b200::from_row_major<Scalar>(out.data(), dims_.query_heads, dims_.head_size);
  }

  // attention.hpp:531-539
  void append_projected(const Vector<Scalar>& x) {
    require_exact("append_projected");
    const std::vector<double> xd = b200::row_major(x);
    b200::check(hx_append_projected_f64(e_, 0, xd.data(), x.size()), e_);
  }

  static Matrix<Scalar> random_matrix(std::mt19937_64& rng, i64 rows, i64 cols) {
    Matrix<Scalar> m(rows, cols);
    for (i64 r = 0; r < rows; ++r)
      for (i64 c = 0; c < cols; ++c) m(r, c) = unit_draw(rng);
    return m;
  }

  // Fixed 53-bit mapping to [-1, 1) (attention.hpp:549-552).
  static Scalar unit_draw(std::mt19937_64& rng) {
    const double u = static_cast<double>(rng() >> 11) * 0x1.0p-53;
    return static_cast<Scalar>(2.0 * u - 1.0);
  }

  hx_engine* engine() { return e_; }

 private:
  void require_exact(const char* what) const {
    if (opt_.storage != Storage::exact)
      throw std::logic_error(std::string(what) + "() needs Storage::exact (fp64 weights and shards)");
  }
  void append_rows(i64 n, const double* k, const double* v) {
    if (opt_.storage == Storage::exact) {
      b200::check(hx_append_kv_f64(e_, 0, 0, n, k, v), e_);
    } else {  // bf16 pages: the engine rounds the fp32 rows to bf16
      const std::size_t cnt = static_cast<std::size_t>(n * dims_.kv_heads * dims_.head_size);
      std::vector<float> kf(k, k + cnt), vf(v, v + cnt);
      b200::check(hx_append_kv(e_, 0, 0, n, kf.data(), vf.data()), e_);
    }
  }
  std::unique_ptr<ShardedKVCache<Scalar>> make_snapshot() const {
    auto c = std::make_unique<ShardedKVCache<Scalar>>(kvp_, dims_.kv_heads, dims_.head_size, chunk_);
    const i64 total = hx_total_tokens(e_, 0, 0), w = dims_.head_size;
    for (i64 r = 0; r < kvp_; ++r) {
      const i64 n = hx_effective_tokens(e_, 0, 0, r);
      c->count_[static_cast<std::size_t>(r)] = n;
      for (i64 h = 0; h < dims_.kv_heads; ++h) {
        std::vector<double>& k = c->k_[c->slot(r, h)];
        std::vector<double>& v = c->v_[c->slot(r, h)];
        k.resize(static_cast<std::size_t>(n * w));
        v.resize(static_cast<std::size_t>(n * w));
        if (!n) continue;
        if (opt_.storage == Storage::exact) {
          b200::check(hx_read_kv_f64(e_, 0, 0, r, h, k.data(), v.data()), e_);
        } else {
          std::vector<float> kf(k.size()), vf(v.size());
          b200::check(hx_read_kv(e_, 0, 0, r, h, kf.data(), vf.data()), e_);
          std::copy(kf.begin(), kf.end(), k.begin());
          std::copy(vf.begin(), vf.end(), v.begin());
        }
      }
    }
    // global order: token g -> rank (g / c) mod kvp, row (g / (c kvp)) c + g mod c (attention.hpp:262-282)
    for (i64 g = 0; g < total; ++g)
      c->order_.push_back({(g / chunk_) % kvp_, (g / (chunk_ * kvp_)) * chunk_ + g % chunk_});
    c->cursor_ = (total / chunk_) % kvp_;
    c->fill_ = total % chunk_;
    return c;
  }

  Dims dims_;
  i64 tpa_, kvp_, chunk_;
  HarnessOptions opt_;
  hx_engine* e_ = nullptr;
  mutable std::vector<Message> transcript_;
  mutable std::unique_ptr<ShardedKVCache<Scalar>> snapshot_;
};

}  // namespace exact
}  // namespace helixsim
