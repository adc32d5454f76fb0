// C++ parity driver for include/helixsim/exact_b200.hpp, written like the
// reference's tests/test_attention.cpp (doctest-style checks, same shapes and
// seeds) but running on the B200 library. Compiled against the in-repo doctest
// shim; the CPU oracle (oracle/helix_oracle.hpp, bf16-storage mode) is the checker.
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

TEST_CASE("decode steps match the monolithic oracle on the worked shape (GPU)") {
  // test_attention.cpp:293-305: {4,2,8}, tpa 2, kvp 4, chunk 16, seed 42, 48 tokens
  ex::DecodeHarness<double> h({4, 2, 8}, 2, 4, 16, 42, 1, 256);
  orc::DecodeHarness o({4, 2, 8}, 2, 4, 16, 42, /*bf16_storage=*/true);
  ex::Rng rng(112);
  std::mt19937_64 orng(112);
  h.grow_random(48, rng);
  o.grow_random(48, orng);
  for (int step = 0; step < 3; ++step) {
    ex::Vector<double> x(32);
    std::vector<double> xo(32);
    for (i64 i = 0; i < 32; ++i) {
      const double v = rng.unit_draw();
      CHECK(v == orc::unit_draw(orng));  // identical stream
      x[i] = static_cast<float>(v);
      xo[static_cast<std::size_t>(i)] = static_cast<float>(v);
    }
    const ex::Matrix<double> got = h.step(x);
    const orc::Mat want = o.step(xo);
    CHECK(rel_err(got, want) <= 1e-3);  // appended K/V may differ by 1 bf16 ulp
  }
  CHECK(h.total_tokens() == 51);
}

TEST_CASE("the transcript records exactly the expected transfers (GPU)") {
  // test_attention.cpp:318-348
  ex::DecodeHarness<double> h({4, 2, 8}, 2, 4, 16, 42, 1, 256);
  ex::Rng rng(113);
  h.grow_random(48, rng);
  ex::Vector<double> x(32);
  for (i64 i = 0; i < 32; ++i) x[i] = rng.unit_draw();
  h.step(x);
  i64 bcast = 0, a2a = 0;
  for (const ex::Message& m : h.transcript()) {
    if (m.kind == ex::MsgKind::Broadcast) {
      ++bcast;
      CHECK(m.src == 0);
      CHECK(m.payload_scalars == 32);
    } else {
      ++a2a;
      CHECK(m.payload_scalars == 4);
      CHECK(m.lse_scalars == 1);
    }
  }
  CHECK(bcast == h.pool() - 1);
  CHECK(a2a == 2 * 4 * 3);
}

TEST_CASE("round-robin growth stays balanced at every prefix (GPU)") {
  // test_attention.cpp:195-223 through the harness cache views
  ex::DecodeHarness<double> h({8, 2, 8}, 1, 4, 16, 3, 1, 256);
  ex::Rng rng(108);
  for (i64 i = 0; i < 70; ++i) {
    h.grow_random(1, rng);
    CHECK(h.max_min_gap() <= 16);
  }
  CHECK(h.total_tokens() == 70);
  CHECK(h.effective_tokens(0) == 22);
  CHECK(h.effective_tokens(1) == 16);
}

TEST_CASE("harness shape constraints are enforced (GPU)") {
  // test_attention.cpp:382-395
  CHECK_THROWS_AS(ex::DecodeHarness<double>({4, 3, 8}, 1, 1, 16, 1), std::invalid_argument);
  CHECK_THROWS_AS(ex::DecodeHarness<double>({4, 2, 8}, 4, 1, 16, 1), std::invalid_argument);
  CHECK_THROWS_AS(ex::DecodeHarness<double>({4, 2, 8}, 2, 3, 16, 1), std::invalid_argument);
  ex::DecodeHarness<double> ok({4, 2, 8}, 2, 2, 16, 1);
  ex::Vector<double> x(32);
  CHECK_THROWS_AS(ok.step(x), std::invalid_argument);  // empty context
  ex::Rng rng(116);
  ok.grow_random(4, rng);
  ex::Vector<double> bad(31);
  CHECK_THROWS_AS(ok.step(bad), std::invalid_argument);
}
