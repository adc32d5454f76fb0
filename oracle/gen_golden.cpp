// TEST INFRASTRUCTURE ONLY. Generates tests/golden/*.json by running the
// REFERENCE's own header-only harness (/root/reference/proj/include/helixsim/
// attention.hpp, unmodified) compiled against oracle/shims/Eigen. Built and
// run by `make -C oracle golden` in the development container (the reference
// tree does not exist on the GPU box; the fixtures are committed).
#include <cstdio>
#include <fstream>
#include <random>
#include <sstream>
#include <string>
#include <vector>

#include "helixsim/attention.hpp"

using namespace helixsim;
using namespace helixsim::exact;
using Mat = Matrix<double>;
using Vec = Vector<double>;

namespace {

std::string num(double v) {
  if (std::isinf(v)) return v < 0 ? "\"-inf\"" : "\"inf\"";
  char buf[64];
  std::snprintf(buf, sizeof buf, "%.17g", v);
  return buf;
}
// Row-major flattening (the reference matrices are rows = heads / tokens).
std::string arr(const Eigen::Dense<double>& m) {
  std::ostringstream o;
  o << "[";
  for (Eigen::Index r = 0; r < m.rows(); ++r)
    for (Eigen::Index c = 0; c < m.cols(); ++c)
      o << (r || c ? "," : "") << num(m(r, c));
  o << "]";
  return o.str();
}
std::string arr(const std::vector<double>& v) {
  std::ostringstream o;
  o << "[";
  for (std::size_t i = 0; i < v.size(); ++i) o << (i ? "," : "") << num(v[i]);
  o << "]";
  return o.str();
}
std::string iarr(const std::vector<i64>& v) {
  std::ostringstream o;
  o << "[";
  for (std::size_t i = 0; i < v.size(); ++i) o << (i ? "," : "") << v[i];
  o << "]";
  return o.str();
}

// One decode-harness case: construct, grow with rng(grow_seed), then `steps`
// decode steps with x = random_matrix(rng, hidden, 1) from the same rng
// (test_attention.cpp:293-305 pattern).
std::string harness_case(const std::string& name, DecodeHarness<double>::Dims dims, i64 tpa,
                         i64 kvp, i64 chunk, std::uint64_t seed, std::uint64_t grow_seed,
                         i64 context, int steps) {
  DecodeHarness<double> h(dims, tpa, kvp, chunk, seed);
  std::mt19937_64 rng(grow_seed);
  h.grow_random(context, rng);
  std::ostringstream o;
  o << "{\"name\":\"" << name << "\",\"query_heads\":" << dims.query_heads
    << ",\"kv_heads\":" << dims.kv_heads << ",\"head_size\":" << dims.head_size
    << ",\"tpa\":" << tpa << ",\"kvp\":" << kvp << ",\"chunk\":" << chunk << ",\"seed\":" << seed
    << ",\"grow_seed\":" << grow_seed << ",\"context\":" << context << ",\"steps\":[";
  for (int s = 0; s < steps; ++s) {
    const Vec x = DecodeHarness<double>::random_matrix(rng, dims.hidden(), 1);
    const Mat want = h.reference(x);
    const Mat got = h.step(x);
    o << (s ? "," : "") << "{\"x\":" << arr(x) << ",\"step\":" << arr(got)
      << ",\"reference\":" << arr(want) << "}";
  }
  std::vector<i64> counts, order_rank;
  for (i64 r = 0; r < kvp; ++r) counts.push_back(h.cache().effective_tokens(r));
  for (const TokenRef& t : h.cache().token_order()) order_rank.push_back(t.rank);
  std::vector<i64> tr;
  for (const Message& m : h.transcript()) {
    tr.push_back(m.kind == MsgKind::Broadcast ? 0 : 1);
    tr.push_back(m.src);
    tr.push_back(m.dst);
    tr.push_back(m.payload_scalars);
    tr.push_back(m.lse_scalars);
  }
  // Final cache contents of rank 0 / head 0 (keys), append order.
  const KvChunk<double> ctx = h.cache().context(0, 0);
  o << "],\"effective_tokens\":" << iarr(counts) << ",\"token_rank\":" << iarr(order_rank)
    << ",\"max_min_gap\":" << h.cache().max_min_gap() << ",\"transcript\":" << iarr(tr)
    << ",\"rank0_head0_keys\":" << arr(ctx.keys) << ",\"rank0_head0_values\":" << arr(ctx.values)
    << "}";
  return o.str();
}

std::string merge_case() {
  // test_attention.cpp:108-126 shapes: fragments of {40,1,17,0,64,0,5} tokens.
  std::mt19937_64 rng(104);
  const i64 width = 16;
  const Vec q = DecodeHarness<double>::random_matrix(rng, width, 1);
  std::vector<HeadFragment<double>> frags;
  std::vector<Mat> keys, values;
  for (i64 tokens : {40, 1, 17, 0, 64, 0, 5}) {
    keys.push_back(DecodeHarness<double>::random_matrix(rng, tokens, width));
    values.push_back(DecodeHarness<double>::random_matrix(rng, tokens, width));
    frags.push_back(partial_head_attention<double>(q, keys.back(), values.back()));
  }
  const MergedHead<double> m = merge_head_fragments<double>(frags);
  std::ostringstream o;
  o << "{\"name\":\"merge\",\"width\":" << width << ",\"q\":" << arr(q) << ",\"fragments\":[";
  for (std::size_t i = 0; i < frags.size(); ++i)
    o << (i ? "," : "") << "{\"keys\":" << arr(keys[i]) << ",\"values\":" << arr(values[i])
      << ",\"out\":" << arr(frags[i].partial_out) << ",\"lse\":" << num(frags[i].lse) << "}";
  Mat allk(0, width), allv(0, width);
  for (std::size_t i = 0; i < keys.size(); ++i) {
    const Eigen::Index r0 = allk.rows();
    allk.conservativeResize(r0 + keys[i].rows(), Eigen::NoChange);
    allv.conservativeResize(r0 + keys[i].rows(), Eigen::NoChange);
    if (keys[i].rows()) {
      allk.middleRows(r0, keys[i].rows()) = keys[i];
      allv.middleRows(r0, keys[i].rows()) = values[i];
    }
  }
  o << "],\"merged_out\":" << arr(m.out) << ",\"merged_lse\":" << num(m.lse)
    << ",\"reference\":" << arr(reference_attention<double>(q, allk, allv)) << "}";
  return o.str();
}

}  // namespace

int main(int argc, char** argv) {
  const std::string dir = argc > 1 ? argv[1] : "tests/golden";
  std::vector<std::string> cases;
  // The reference's worked decode shape (test_attention.cpp:293-305).
  cases.push_back(harness_case("worked", {4, 2, 8}, 2, 4, 16, 42, 112, 48, 3));
  // Single-GPU pool (test_attention.cpp:350-359).
  cases.push_back(harness_case("pool1", {4, 2, 8}, 1, 1, 16, 3, 114, 10, 1));
  // tiny-gqa preset (H=64, Q=8, K=4, Hsz=8) at every Helix width <= 8.
  const std::pair<i64, i64> widths[] = {{1, 1}, {1, 2}, {2, 2}, {1, 8}, {2, 4}, {4, 2}, {4, 1}};
  for (auto [tpa, kvp] : widths)
    cases.push_back(harness_case("tiny_gqa_tpa" + std::to_string(tpa) + "_kvp" + std::to_string(kvp),
                                 {8, 4, 8}, tpa, kvp, 16, 7, 1000 + tpa * 10 + kvp, 40, 3));
  // Odd chunk size and ragged shards.
  cases.push_back(harness_case("odd_chunk", {4, 2, 8}, 1, 4, 5, 11, 77, 37, 3));
  // Head size 128 with GQA factor 4 (Llama-3 head geometry, 4 KV heads).
  cases.push_back(harness_case("hsz128_gqa4", {16, 4, 128}, 1, 2, 16, 5, 55, 70, 2));
  // Head size 128, GQA factor 16 (Llama-405B geometry, 1 KV head group).
  cases.push_back(harness_case("hsz128_gqa16", {16, 1, 128}, 1, 4, 16, 6, 66, 90, 2));

  std::ofstream f(dir + "/reference_harness.json");
  f << "{\"generator\":\"oracle/gen_golden.cpp over /root/reference/proj/include/helixsim/"
       "attention.hpp (unmodified) + oracle/shims/Eigen\",\"cases\":[";
  for (std::size_t i = 0; i < cases.size(); ++i) f << (i ? ",\n" : "\n") << cases[i];
  f << "\n],\"merge\":" << merge_case() << "}\n";
  std::printf("wrote %zu harness cases to %s/reference_harness.json\n", cases.size(), dir.c_str());
  return 0;
}
