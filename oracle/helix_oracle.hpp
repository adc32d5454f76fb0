// TEST INFRASTRUCTURE ONLY. This CPU oracle is the parity checker for the
// B200 decode path: only tests/, __graft_entry__.smoke() and bench.py's
// cpu_baseline leg may load it. The product library never links it.
//
// Clean-room restatement, in plain C++20 doubles (no Eigen), of the
// reference's exact-attention harness
//   /root/reference/proj/include/helixsim/attention.hpp
// Every function cites the reference lines it follows. Pinning: the
// restatement is checked against golden vectors produced by the reference
// header itself (compiled unmodified against oracle/shims, see
// oracle/gen_golden.cpp and tests/test_oracle_golden.py).
//
// Beyond the reference (which stops at the merged attention output,
// SPEC.md:94), the oracle defines the rest of the decode layer that the
// north star asks for (O-projection, RMSNorm, SwiGLU FFN, LM head, greedy
// argmax). Those parts are "parity unpinned" by the reference; their
// definition lives here and in DESIGN.md section "Layer extension".
#pragma once

#include <cmath>
#include <cstdint>
#include <limits>
#include <random>
#include <span>
#include <stdexcept>
#include <vector>

namespace helix_oracle {

using i64 = std::int64_t;

constexpr double neg_inf() { return -std::numeric_limits<double>::infinity(); }

// Row-major dense matrix (rows = tokens / heads as in the reference).
struct Mat {
  i64 rows = 0, cols = 0;
  std::vector<double> a;
  Mat() = default;
  Mat(i64 r, i64 c) : rows(r), cols(c), a(static_cast<std::size_t>(r * c), 0.0) {}
  double& operator()(i64 r, i64 c) { return a[static_cast<std::size_t>(r * cols + c)]; }
  double operator()(i64 r, i64 c) const { return a[static_cast<std::size_t>(r * cols + c)]; }
  const double* row(i64 r) const { return a.data() + r * cols; }
  double* row(i64 r) { return a.data() + r * cols; }
};

// attention.hpp:549-552 -- portable uniform in [-1, 1).
double unit_draw(std::mt19937_64& rng);
// attention.hpp:541-546 -- row-major fill order.
Mat random_matrix(std::mt19937_64& rng, i64 rows, i64 cols);

// Round to the nearest bf16 value (round-to-nearest-even on the double).
// Models the B200 path's bf16 storage of weights and KV.
double round_bf16(double x);
// Round to the nearest FP8 E4M3 ("e4m3fn": bias 7, 3 mantissa bits, max finite
// 448, no infinities) value, ties to even, saturating at +-448 -- the B200
// path's optional FP8 KV storage.
double round_e4m3(double x);
// FP4 E2M1 block storage (PAPER.md:158 evaluates at FP4): the n values of one
// block share a power-of-two scale 2^e, e = the smallest exponent with
// 6 * 2^e >= max |x| (clamped to [-14, 13]); each value is rounded to the
// nearest e2m1 grid point {0, 0.5, 1, 1.5, 2, 3, 4, 6} * 2^e, ties to the even
// code, saturating at 6 * 2^e. In place; blocks are 32 dims of one token's row.
void round_e2m1_block(double* x, i64 n);

// ---- single-head primitives (attention.hpp:35-78) ----
struct HeadFragment {
  std::vector<double> out;  // partial_out, width w
  double lse = neg_inf();
};
double logit_scale(i64 width);                                    // :36-38
std::vector<double> reference_attention(const std::vector<double>& q, const Mat& keys,
                                        const Mat& values);       // :43-53
HeadFragment partial_head_attention(const std::vector<double>& q, const Mat& keys,
                                    const Mat& values);           // :65-78

// ---- merging (attention.hpp:85-175) ----
std::vector<std::size_t> canonical_order(std::span<const HeadFragment> frags);  // :90-102
HeadFragment merge_head_fragments(std::span<const HeadFragment> frags);         // :118-137

// ---- sharded KV cache (attention.hpp:229-369) ----
struct TokenRef {
  i64 rank, row;
};
class ShardedKVCache {
 public:
  ShardedKVCache(i64 kvp, i64 kv_heads, i64 head_width, i64 chunk_size);
  i64 kvp() const { return kvp_; }
  i64 kv_heads() const { return kv_heads_; }
  i64 head_width() const { return w_; }
  i64 chunk_size() const { return chunk_; }
  i64 total_tokens() const { return static_cast<i64>(order_.size()); }
  const std::vector<TokenRef>& token_order() const { return order_; }
  i64 effective_tokens(i64 rank) const { return counts_.at(static_cast<std::size_t>(rank)); }
  i64 max_min_gap() const;  // :286-294
  // :262-282 -- k, v are [kv_heads x w] row-major
  void append_round_robin(const Mat& k, const Mat& v);
  // Rows of one rank for one head, append order, open chunk trimmed (:303-309)
  const Mat& keys(i64 rank, i64 head) const { return k_[idx(rank, head)]; }
  const Mat& values(i64 rank, i64 head) const { return v_[idx(rank, head)]; }
  // :312-327 -- global append order
  void global_context(i64 head, Mat& keys, Mat& values) const;
  // :332-359 -- explicit token->rank assignment (chunking only affects storage)
  static ShardedKVCache from_partition(i64 kvp, const std::vector<Mat>& keys,
                                       const std::vector<Mat>& values,
                                       const std::vector<i64>& rank_of_token, i64 chunk);
  i64 cursor() const { return cursor_; }
  i64 fill() const { return fill_; }

 private:
  std::size_t idx(i64 rank, i64 head) const {
    return static_cast<std::size_t>(rank * kv_heads_ + head);
  }
  void push_row(i64 rank, i64 head, const double* k, const double* v);
  i64 kvp_, kv_heads_, w_, chunk_;
  std::vector<Mat> k_, v_;
  std::vector<i64> counts_;
  std::vector<TokenRef> order_;
  i64 cursor_ = 0, fill_ = 0;
};

// :375-396 -- queries [kv_head_count*q_per_kv x w] -> fragment rows
struct AttentionFragment {
  Mat out;                  // heads x w
  std::vector<double> lse;  // per head
};
AttentionFragment shard_attention(const Mat& queries, const ShardedKVCache& cache, i64 rank,
                                  i64 kv_head_offset, i64 kv_head_count, i64 q_per_kv);
// :155-175
AttentionFragment merge_fragments(std::span<const AttentionFragment> frags);

// ---- decode harness (attention.hpp:401-563) ----
enum class MsgKind { Broadcast = 0, AllToAll = 1 };
struct Message {
  MsgKind kind;
  i64 src, dst, payload_scalars, lse_scalars;
};

struct Dims {
  i64 query_heads, kv_heads, head_size;
  i64 hidden() const { return query_heads * head_size; }
};

class DecodeHarness {
 public:
  // bf16_storage=false reproduces the reference bit-for-bit in intent
  // (double weights and KV). bf16_storage=true rounds weights, grown KV and
  // appended KV to bf16 -- the operands the B200 path actually stores.
  DecodeHarness(Dims dims, i64 tpa, i64 kvp, i64 chunk_size, std::uint64_t seed,
                bool bf16_storage = false);
  void grow_random(i64 n, std::mt19937_64& rng);              // :452-456
  Mat step(const std::vector<double>& x);                     // :460-510
  // step() whose final append uses the given rows (k, v: [kv_heads x w])
  // instead of this harness's own projection -- lets a parity test feed the
  // exact bf16 rows the GPU stored, isolating attention arithmetic.
  Mat step_with_append(const std::vector<double>& x, const Mat* k, const Mat* v);
  Mat reference(const std::vector<double>& x) const;          // :514-529
  void append_projected(const std::vector<double>& x);        // :531-539
  std::vector<double> project_q(const std::vector<double>& x) const;  // x^T W_q, all heads
  void project_kv(const std::vector<double>& x, Mat& k, Mat& v) const;
  const ShardedKVCache& cache() const { return cache_; }
  ShardedKVCache& cache() { return cache_; }
  const std::vector<Message>& transcript() const { return transcript_; }
  i64 pool() const { return tpa_ * kvp_; }
  const Mat& wq() const { return wq_; }
  const Mat& wk() const { return wk_; }
  const Mat& wv() const { return wv_; }
  Dims dims() const { return dims_; }
  // Replace the drawn W_q/W_k/W_v (hash-initialised model layers).
  void set_weights(Mat wq, Mat wk, Mat wv) {
    wq_ = std::move(wq);
    wk_ = std::move(wk);
    wv_ = std::move(wv);
  }
  bool bf16_storage() const { return bf16_; }
  // KV storage rounding: bf16 (bf16_storage) or, with kv_fp8, e4m3 (round_e4m3);
  // weights stay bf16. Applies to KV grown or appended after the call.
  void set_kv_fp8(bool on) { kv_fp8_ = on; }
  bool kv_fp8() const { return kv_fp8_; }
  // FP4 (e2m1, blocks of 32 dims of a token's K or V row per KV head)
  void set_kv_fp4(bool on) { kv_fp4_ = on; }
  double round_kv(double x) const { return kv_fp8_ ? round_e4m3(x) : (bf16_ ? round_bf16(x) : x); }
  // Storage rounding of one token's K or V rows [kv heads x width].
  void round_kv_rows(Mat& m) const;
  // Last step's merged lse per query head (natural log), for kernel parity.
  const std::vector<double>& last_lse() const { return last_lse_; }

 private:
  i64 rank_id(i64 kvp_rank, i64 group) const { return group * kvp_ + kvp_rank; }
  Dims dims_;
  i64 tpa_, kvp_;
  bool bf16_;
  bool kv_fp8_ = false;
  bool kv_fp4_ = false;
  Mat wq_, wk_, wv_;
  ShardedKVCache cache_;
  std::vector<Message> transcript_;
  std::vector<double> last_lse_;
};

}  // namespace helix_oracle
