// helixsim/exact_b200.hpp -- drop-in C++ mirror of the reference's
// helixsim::exact decode harness (/root/reference/proj/include/helixsim/
// attention.hpp:401-563) backed by the B200 library (include/helix_b200.h).
//
// Swap `#include "helixsim/attention.hpp"` for this header and link
// libhelix_b200.so: DecodeHarness, its Dims, grow_random, step, cache views,
// transcript, Message/MsgKind keep the reference's names, argument meaning and
// std::invalid_argument messages. Differences, all documented in DESIGN.md:
//   * the matrix types are helixsim::exact::Matrix/Vector below (row-major,
//     Eigen-like accessors) unless Eigen is included first, in which case the
//     reference's Eigen aliases are used;
//   * weights/KV are stored in bf16 on the GPU, x is rounded to fp32;
//   * DecodeHarness takes an optional request batch (one reference harness per
//     request, identical seeded weights) and a context capacity.
#pragma once

#include <cstdint>
#include <random>
#include <stdexcept>
#include <string>
#include <vector>

#include "../helix_b200.h"

namespace helixsim {
using i64 = std::int64_t;

namespace exact {

#ifndef EIGEN_WORLD_VERSION
// Minimal dense row-major matrix with the Eigen accessors the reference API uses.
template <class Scalar>
class Matrix {
 public:
  Matrix() = default;
  Matrix(i64 rows, i64 cols) : rows_(rows), cols_(cols), a_(static_cast<std::size_t>(rows * cols)) {}
  i64 rows() const { return rows_; }
  i64 cols() const { return cols_; }
  i64 size() const { return rows_ * cols_; }
  Scalar& operator()(i64 r, i64 c) { return a_[static_cast<std::size_t>(r * cols_ + c)]; }
  Scalar operator()(i64 r, i64 c) const { return a_[static_cast<std::size_t>(r * cols_ + c)]; }
  Scalar& operator[](i64 i) { return a_[static_cast<std::size_t>(i)]; }
  Scalar operator[](i64 i) const { return a_[static_cast<std::size_t>(i)]; }
  Scalar* data() { return a_.data(); }
  const Scalar* data() const { return a_.data(); }

 private:
  i64 rows_ = 0, cols_ = 0;
  std::vector<Scalar> a_;
};
template <class Scalar>
class Vector : public Matrix<Scalar> {
 public:
  Vector() = default;
  explicit Vector(i64 n) : Matrix<Scalar>(n, 1) {}
};
#else
template <class Scalar>
using Matrix = Eigen::Matrix<Scalar, Eigen::Dynamic, Eigen::Dynamic, Eigen::RowMajor>;
template <class Scalar>
using Vector = Eigen::Matrix<Scalar, Eigen::Dynamic, 1>;
#endif

// attention.hpp:401-411
enum class MsgKind { Broadcast, AllToAll };
struct Message {
  MsgKind kind;
  i64 src;
  i64 dst;
  i64 payload_scalars;
  i64 lse_scalars;
};

namespace detail {
inline void check(int rc, const hx_engine* e) {
  if (rc == HX_OK) return;
  const std::string msg = hx_last_error(e);
  if (rc == HX_ERR_INVALID) throw std::invalid_argument(msg);  // the reference's exceptions
  throw std::runtime_error(msg);
}
}  // namespace detail

// Random stream for grow_random: std::mt19937_64 semantics (attention.hpp:452-456, 549-552).
class Rng {
 public:
  explicit Rng(std::uint64_t seed) { detail::check(hx_rng_create(seed, &r_), nullptr); }
  ~Rng() { hx_rng_destroy(r_); }
  Rng(const Rng&) = delete;
  Rng& operator=(const Rng&) = delete;
  double unit_draw() { return hx_rng_unit_draw(r_); }
  hx_rng* handle() { return r_; }

 private:
  hx_rng* r_ = nullptr;
};

// DecodeHarness on the B200 (attention.hpp:419-563). Scalar is the host type of
// x and of the returned output; the GPU computes in bf16-stored / fp32 arithmetic.
template <class Scalar>
class DecodeHarness {
 public:
  struct Dims {
    i64 query_heads;
    i64 kv_heads;
    i64 head_size;
    i64 hidden() const { return query_heads * head_size; }
  };

  DecodeHarness(Dims dims, i64 tpa, i64 kvp, i64 chunk_size, std::uint64_t seed, i64 batch = 1,
                i64 capacity = 1 << 16, int device = 0)
      : dims_(dims), tpa_(tpa), kvp_(kvp), batch_(batch) {
    hx_model_config m{dims.hidden(), dims.query_heads, dims.kv_heads, dims.head_size, 16, 1, 1, 1, 0};
    hx_parallel_config p{tpa, kvp, chunk_size, 0, 0, nullptr};
    hx_runtime_config r{batch, capacity, device, 0, 0, 0};
    detail::check(hx_engine_create(&m, &p, &r, &e_), nullptr);
    detail::check(hx_init_weights_mt19937(e_, seed), e_);
  }
  ~DecodeHarness() { hx_engine_destroy(e_); }
  DecodeHarness(const DecodeHarness&) = delete;
  DecodeHarness& operator=(const DecodeHarness&) = delete;

  i64 pool() const { return tpa_ * kvp_; }

  // attention.hpp:452-456 (request 0 unless given)
  void grow_random(i64 n, Rng& rng, i64 request = 0) {
    detail::check(hx_grow_random(e_, 0, request, n, rng.handle()), e_);
  }

  // attention.hpp:460-510: returns query_heads x head_size for request 0
  // (batch 1), appends x's projected K/V afterwards.
  Matrix<Scalar> step(const Vector<Scalar>& x) {
    std::vector<float> xf(static_cast<std::size_t>(x.size()));
    for (i64 i = 0; i < x.size(); ++i) xf[static_cast<std::size_t>(i)] = static_cast<float>(x[i]);
    std::vector<float> out(static_cast<std::size_t>(batch_ * dims_.hidden()));
    detail::check(hx_harness_step(e_, 0, xf.data(), static_cast<i64>(xf.size()), out.data(), nullptr), e_);
    Matrix<Scalar> o(dims_.query_heads, dims_.head_size);
    for (i64 h = 0; h < dims_.query_heads; ++h)
      for (i64 d = 0; d < dims_.head_size; ++d)
        o(h, d) = static_cast<Scalar>(out[static_cast<std::size_t>(h * dims_.head_size + d)]);
    return o;
  }

  // ShardedKVCache views (attention.hpp:286-309)
  i64 total_tokens(i64 request = 0) const { return hx_total_tokens(e_, 0, request); }
  i64 effective_tokens(i64 rank, i64 request = 0) const { return hx_effective_tokens(e_, 0, request, rank); }
  i64 max_min_gap(i64 request = 0) const { return hx_max_min_gap(e_, 0, request); }

  std::vector<Message> transcript() const {
    const i64 n = hx_transcript_size(e_);
    std::vector<std::int64_t> raw(static_cast<std::size_t>(5 * n));
    if (n) detail::check(hx_transcript(e_, raw.data()), e_);
    std::vector<Message> t;
    for (i64 i = 0; i < n; ++i) {
      const std::int64_t* r = raw.data() + 5 * i;
      t.push_back({r[0] == 0 ? MsgKind::Broadcast : MsgKind::AllToAll, r[1], r[2], r[3], r[4]});
    }
    return t;
  }

  hx_engine* engine() { return e_; }

 private:
  Dims dims_;
  i64 tpa_, kvp_, batch_;
  hx_engine* e_ = nullptr;
};

}  // namespace exact
}  // namespace helixsim
