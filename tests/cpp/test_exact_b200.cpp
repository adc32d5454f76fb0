// C++ parity driver for include/helixsim/exact_b200.hpp beyond the reference's
// own test file (which oracle/Makefile compiles unmodified against the header:
// oracle/_ref/test_attention_b200): the production bf16 storage of the harness
// against the CPU oracle (oracle/helix_oracle.hpp, bf16-storage mode), the
// fp64 harness against the oracle's double harness, and the cache snapshot.
#define DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
#include <doctest.h>

#include <cmath>
#include <random>
#include <vector>

#include "helix_oracle.hpp"
#include "helixsim/exact_b200.hpp"

using namespace helixsim;
namespace ex = helixsim::exact;
namespace orc = helix_oracle;

namespace {
double rel_err(const ex::Matrix<double>& got, const orc::Mat& want) {
  double scale = 1e-12, err = 0.0;
  for (i64 r = 0; r < want.rows; ++r)
    for (i64 c = 0; c < want.cols; ++c) {
      scale = std::max(scale, std::abs(want(r, c)));
      err = std::max(err, std::abs(got(r, c) - want(r, c)));
    }
  return err / scale;
}
}  // namespace

TEST_CASE("bf16 storage: decode steps match the bf16-storage oracle on the worked shape") {
  // test_attention.cpp:293-305: {4,2,8}, tpa 2, kvp 4, chunk 16, seed 42, 48 tokens
  ex::HarnessOptions opt;
  opt.storage = ex::Storage::bf16;
  opt.capacity = 256;
  ex::DecodeHarness<double> h({4, 2, 8}, 2, 4, 16, 42, opt);
  orc::DecodeHarness o({4, 2, 8}, 2, 4, 16, 42, /*bf16_storage=*/true);
  std::mt19937_64 rng(112), orng(112);
  h.grow_random(48, rng);
  o.grow_random(48, orng);
  for (int step = 0; step < 3; ++step) {
    ex::Vector<double> x(32);
    std::vector<double> xo(32);
    for (i64 i = 0; i < 32; ++i) {
      const double v = ex::DecodeHarness<double>::unit_draw(rng);
      CHECK(v == orc::unit_draw(orng));  // identical stream
      x[i] = static_cast<float>(v);
      xo[static_cast<std::size_t>(i)] = static_cast<float>(v);
    }
    const ex::Matrix<double> got = h.step(x);
    const orc::Mat want = o.step(xo);
    CHECK(rel_err(got, want) <= 1e-3);  // appended K/V may differ by 1 bf16 ulp
  }
  CHECK(h.cache().total_tokens() == 51);
  CHECK_THROWS_AS(h.reference(ex::Vector<double>::Zero(32)), std::logic_error);
}

TEST_CASE("exact storage: steps match the double oracle at 1e-10, Hsz 128, GQA 4") {
  ex::HarnessOptions opt;
  opt.capacity = 4096;
  ex::DecodeHarness<double> h({16, 4, 128}, 2, 2, 16, 9, opt);
  orc::DecodeHarness o({16, 4, 128}, 2, 2, 16, 9, /*bf16_storage=*/false);
  std::mt19937_64 rng(500), orng(500);
  h.grow_random(1000, rng);
  o.grow_random(1000, orng);
  for (int step = 0; step < 3; ++step) {
    ex::Vector<double> x(2048);
    std::vector<double> xo(2048);
    for (i64 i = 0; i < 2048; ++i) {
      const double v = orc::unit_draw(orng);
      x[i] = v;
      xo[static_cast<std::size_t>(i)] = v;
    }
    CHECK(rel_err(h.step(x), o.step(xo)) <= 1e-10);
  }
}

TEST_CASE("the cache snapshot reproduces the reference container") {
  ex::DecodeHarness<double> h({6, 2, 8}, 1, 3, 5, 3);  // hidden 48: tpa*kvp = 3 divides it
  ex::ShardedKVCache<double> host(3, 2, 8, 5);
  std::mt19937_64 rng(108), hr(108);
  for (i64 i = 0; i < 41; ++i) {
    h.grow_random(1, rng);
    const auto v = ex::DecodeHarness<double>::random_matrix(hr, 2, 8);  // V first (attention.hpp:454-455)
    const auto k = ex::DecodeHarness<double>::random_matrix(hr, 2, 8);
    host.append_round_robin(k, v);
    CHECK(h.cache().max_min_gap() <= 5);
  }
  const auto& c = h.cache();
  CHECK(c.total_tokens() == 41);
  for (i64 r = 0; r < 3; ++r) {
    CHECK(c.effective_tokens(r) == host.effective_tokens(r));
    for (i64 head = 0; head < 2; ++head) {
      CHECK(c.context(r, head).keys == host.context(r, head).keys);
      CHECK(c.context(r, head).values == host.context(r, head).values);
    }
  }
  for (i64 head = 0; head < 2; ++head) CHECK(c.global_context(head).keys == host.global_context(head).keys);
  for (std::size_t g = 0; g < 41; ++g) {
    CHECK(c.token_order()[g].rank == host.token_order()[g].rank);
    CHECK(c.token_order()[g].row == host.token_order()[g].row);
  }
}

TEST_CASE("append_projected then reference equals the reference of the grown cache") {
  ex::DecodeHarness<double> a({4, 2, 8}, 1, 2, 16, 5), b({4, 2, 8}, 1, 2, 16, 5);
  std::mt19937_64 ra(7), rb(7), rx(8);
  a.grow_random(30, ra);
  b.grow_random(30, rb);
  const ex::Vector<double> x = ex::DecodeHarness<double>::random_matrix(rx, 32, 1);
  const ex::Vector<double> y = ex::DecodeHarness<double>::random_matrix(rx, 32, 1);
  a.append_projected(x);
  b.step(x);  // attend, then the same append
  CHECK(a.reference(y) == b.reference(y));
  CHECK(a.cache().total_tokens() == 31);
}
