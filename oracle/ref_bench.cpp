// TEST INFRASTRUCTURE ONLY -- bench.py's CPU baseline ("kind": "reference").
// Times the REFERENCE's own DecodeHarness<double>::step (attention.hpp:460-510,
// unmodified, compiled against oracle/shims/Eigen) on host cores. Each thread
// owns an independent harness (one request of the batch), as the reference
// runs one request per harness. Construction and KV growth are untimed.
//
//   ref_bench Q K Hsz tpa kvp context steps threads [warmup]
// prints one JSON line.
#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <random>
#include <thread>
#include <vector>

#include "helixsim/attention.hpp"

using namespace helixsim;
using namespace helixsim::exact;

int main(int argc, char** argv) {
  if (argc < 9) {
    std::fprintf(stderr, "usage: ref_bench Q K Hsz tpa kvp context steps threads\n");
    return 2;
  }
  const i64 Q = std::atoll(argv[1]), K = std::atoll(argv[2]), Hsz = std::atoll(argv[3]);
  const i64 tpa = std::atoll(argv[4]), kvp = std::atoll(argv[5]);
  const i64 context = std::atoll(argv[6]);
  const int steps = std::atoi(argv[7]), threads = std::atoi(argv[8]);
  const int warmup = argc > 9 ? std::atoi(argv[9]) : 0;

  std::atomic<int> ready{0};
  std::atomic<bool> go{false};
  std::vector<double> seconds(static_cast<std::size_t>(threads), 0.0);
  std::vector<double> checksum(static_cast<std::size_t>(threads), 0.0);
  std::vector<std::thread> pool;
  for (int t = 0; t < threads; ++t)
    pool.emplace_back([&, t] {
      DecodeHarness<double> h({Q, K, Hsz}, tpa, kvp, 16, 42);
      std::mt19937_64 rng(1000 + static_cast<std::uint64_t>(t));
      h.grow_random(context, rng);
      std::vector<Vector<double>> xs;
      for (int s = 0; s < steps + warmup; ++s) {
        Vector<double> x(Q * Hsz);
        for (i64 i = 0; i < Q * Hsz; ++i) x[i] = DecodeHarness<double>::unit_draw(rng);
        xs.push_back(x);
      }
      for (int s = 0; s < warmup; ++s) h.step(xs[static_cast<std::size_t>(steps + s)]);
      ready.fetch_add(1);
      while (!go.load()) std::this_thread::yield();
      const auto t0 = std::chrono::steady_clock::now();
      double cs = 0.0;
      for (int s = 0; s < steps; ++s) cs += h.step(xs[static_cast<std::size_t>(s)])(0, 0);
      const auto t1 = std::chrono::steady_clock::now();
      seconds[static_cast<std::size_t>(t)] = std::chrono::duration<double>(t1 - t0).count();
      checksum[static_cast<std::size_t>(t)] = cs;
    });
  while (ready.load() < threads) std::this_thread::sleep_for(std::chrono::milliseconds(5));
  const auto w0 = std::chrono::steady_clock::now();
  go.store(true);
  for (auto& th : pool) th.join();
  const double wall = std::chrono::duration<double>(std::chrono::steady_clock::now() - w0).count();
  double worst = 0.0, cs = 0.0;
  for (int t = 0; t < threads; ++t) {
    worst = std::max(worst, seconds[static_cast<std::size_t>(t)]);
    cs += checksum[static_cast<std::size_t>(t)];
  }
  std::printf(
      "{\"threads\": %d, \"steps\": %d, \"context\": %lld, \"wall_s\": %.6f, "
      "\"max_thread_s\": %.6f, \"seconds_per_step_per_request\": %.9g, "
      "\"request_steps_per_s\": %.9g, \"checksum\": %.17g}\n",
      threads, steps, static_cast<long long>(context), wall, worst, worst / steps,
      static_cast<double>(threads) * steps / worst, cs);
  return 0;
}
