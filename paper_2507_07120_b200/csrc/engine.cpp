// Host runtime: allocation, weight init, round-robin KV bookkeeping, the
// per-layer launch sequence and CUDA-graph capture of the whole decode step.
#include "engine.h"

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "comm.h"
#include "kv_layout.cuh"

namespace hx {

int64_t exchange_layout(int64_t q_per_group, int64_t head_size, int64_t kvp, int64_t* out) {
  if (q_per_group < 1 || head_size < 1 || kvp < 1) throw std::invalid_argument("layout dims must be >= 1");
  const int64_t width = q_per_group * head_size;
  if (width % kvp) throw std::invalid_argument("tpa*kvp must divide the hidden width");
  const int64_t slice = width / kvp;
  int64_t nh_max = 0;
  for (int64_t p = 0; p < kvp; ++p) {
    const int64_t first = p * slice / head_size, last = ((p + 1) * slice - 1) / head_size;
    if (out) {
      out[4 * p + 0] = p * slice;
      out[4 * p + 1] = slice;
      out[4 * p + 2] = first;
      out[4 * p + 3] = last - first + 1;
    }
    nh_max = std::max(nh_max, last - first + 1);
  }
  return (slice + nh_max + 3) / 4 * 4;
}

void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess)
    throw CudaError(std::string(what) + ": " + cudaGetErrorName(e) + " (" + cudaGetErrorString(e) + ")");
}

namespace {

template <class T>
T* dalloc(size_t n, const char* what) {
  void* p = nullptr;
  cuda_check(cudaMalloc(&p, n * sizeof(T) + 16), what);
  // cudaMemset runs on the legacy default stream, which does NOT order against
  // the engine's non-blocking streams: wait for it, or a large clear (the KV
  // pool: tens of GB, milliseconds) can land after the first kernels' writes
  cuda_check(cudaMemset(p, 0, n * sizeof(T) + 16), what);
  cuda_check(cudaDeviceSynchronize(), what);
  return static_cast<T*>(p);
}

// bf16 RNE of a double -- identical to oracle round_bf16 / device double_to_bf16_rne.
uint16_t bf16_bits_from_double(double x) {
  uint64_t b;
  std::memcpy(&b, &x, 8);
  const uint64_t lsb = (b >> 45) & 1ull;
  b += 0x0FFFFFFFFFFFull + lsb;
  b &= ~0x1FFFFFFFFFFFull;
  double r;
  std::memcpy(&r, &b, 8);
  const float f = static_cast<float>(r);  // exact: <= 8 significant bits
  uint32_t u;
  std::memcpy(&u, &f, 4);
  return static_cast<uint16_t>(u >> 16);
}
uint16_t bf16_bits_from_float(float f) {
  uint32_t u;
  std::memcpy(&u, &f, 4);
  if ((u & 0x7F800000u) == 0x7F800000u) return static_cast<uint16_t>(u >> 16);
  u += 0x7FFFu + ((u >> 16) & 1u);
  return static_cast<uint16_t>(u >> 16);
}
float float_from_bf16_bits(uint16_t h) {
  const uint32_t u = static_cast<uint32_t>(h) << 16;
  float f;
  std::memcpy(&f, &u, 4);
  return f;
}

double unit_draw(std::mt19937_64& rng) {  // attention.hpp:549-552
  const double u = static_cast<double>(rng() >> 11) * 0x1.0p-53;
  return 2.0 * u - 1.0;
}

// Byte offset of W^T[n][k] in the CTA-tile-major fragment layout of gemv.cu:
// [128-row block nb][k-step ks][n-tile nt (8)][lane][16 B].
// tcgen05 GEMV image (gemv_tc.cu): per (row block, k-step) 4 KB of K-major core
// matrices [row group 16][k-half 2][row 8][8 k]
size_t wtc_offset_host(int n, int k, int kst) {
  const int nb = n >> 7, rg = (n & 127) >> 3, r = n & 7, ks = k >> 4, kh = (k & 15) >> 3;
  return ((static_cast<size_t>(nb) * kst + ks) * 256 + (rg * 2 + kh) * 8 + r) * 16 + (k & 7) * 2;
}
size_t wfrag_offset_host(int n, int k, int kst) {
  const int nb = n >> 7, nt = (n >> 4) & 7, rn = n & 15, ks = k >> 4, rk = k & 15;
  const int g = rn & 7, rowhalf = rn >> 3;
  const int c = (rk & 7) >> 1, khalf = rk >> 3, elem = rk & 1;
  const int reg = khalf * 2 + rowhalf;
  const int lane = g * 4 + c;
  return (((static_cast<size_t>(nb) * kst + ks) * 8 + nt) * 32 + lane) * 16 + reg * 4 + elem * 2;
}

int round_up(int64_t a, int64_t b) { return static_cast<int>((a + b - 1) / b * b); }

uint64_t hash_stream(uint64_t kind, int64_t layer) { return (kind << 32) | static_cast<uint64_t>(layer); }
enum : uint64_t { kWq = 1, kWk = 2, kWv = 3, kWo = 4, kWgate = 5, kWup = 6, kWdown = 7, kEmb = 8, kLm = 9,
                  kCacheK = 10, kCacheV = 11, kWrouter = 12, kEgate = 13, kEup = 14, kEdown = 15,
                  kWuk = 16, kWuv = 17 };
// routed-expert weights: one stream per (layer, expert) -- oracle/layer_oracle.hpp expert_stream
uint64_t expert_stream(uint64_t kind, int64_t layer, int64_t expert) {
  return (kind << 32) | (static_cast<uint64_t>(layer) << 16) | static_cast<uint64_t>(expert);
}

}  // namespace

// ---------------------------------------------------------------------------
Engine::Engine(const hx_model_config& m, const hx_parallel_config& par, const hx_runtime_config& rt)
    : H_(m.hidden), Qh_(m.query_heads), Kh_(m.kv_heads), D_(m.head_size), F_(m.ffn), L_(m.layers),
      V_(m.vocab), attn_only_(m.attention_only != 0), tpa_(static_cast<int>(par.tpa)),
      kvp_(static_cast<int>(par.kvp)), chunk_(static_cast<int>(par.chunk_size)),
      distributed_(par.distributed != 0), rank_(par.rank), B_(static_cast<int>(rt.batch)),
      cap_(rt.capacity_tokens), device_(rt.device), hopb_(rt.hopb != 0), graphs_(rt.use_graphs != 0) {
  validate_reference_dims();
  // the merge kernels hold one (lse, coefficient) pair per KVP rank (merge.cuh);
  // validate_config caps a Helix pool at max_gpus = 64 (types.hpp:63)
  if (kvp_ > kMaxKvp) throw std::invalid_argument("kvp > 64 is not supported (validate_config max_gpus = 64)");
  if (H_ != Qh_ * D_) throw std::invalid_argument("hidden_dim must equal query_heads * head_size");
  if (L_ < 1) throw std::invalid_argument("layers must be >= 1");
  if (B_ < 1 || B_ > 64) throw std::invalid_argument("batch must be in [1, 64] for the B200 decode kernels");
  if (cap_ < 1) throw std::invalid_argument("capacity_tokens must be >= 1");
  mla_ = m.kv_latent > 0;
  if (rt.kv_dtype != HX_KV_BF16 && rt.kv_dtype != HX_KV_FP8_E4M3 && rt.kv_dtype != HX_KV_F64 &&
      rt.kv_dtype != HX_KV_FP4_E2M1)
    throw std::invalid_argument("unknown kv_dtype");
  kv8_ = rt.kv_dtype == HX_KV_FP8_E4M3;
  kv4_ = rt.kv_dtype == HX_KV_FP4_E2M1;
  f64_ = rt.kv_dtype == HX_KV_F64;
  if (f64_ && (!attn_only_ || par.distributed != HX_POOL_LOCAL))
    throw std::invalid_argument("the exact fp64 harness (HX_KV_F64) is the attention-only local pool "
                                "(DecodeHarness<double>)");
  if (kv4_ && mla_)
    throw std::invalid_argument("FP4 KV pages are implemented for GQA caches (MLA latents: bf16 or FP8)");
  if (kv4_ && m.head_size != 32 && m.head_size != 64 && m.head_size != 128)
    throw std::invalid_argument("FP4 KV blocks are 32 dims: head_size must be 32, 64 or 128");
  if (rt.w_dtype != HX_W_BF16 && rt.w_dtype != HX_W_FP8_E4M3 && rt.w_dtype != HX_W_FP4_E2M1)
    throw std::invalid_argument("unknown w_dtype");
  w8_ = rt.w_dtype == HX_W_FP8_E4M3;
  w4_ = rt.w_dtype == HX_W_FP4_E2M1;
  if ((w8_ || w4_) && B_ > 16) throw std::invalid_argument("FP8 / FP4 weights run the mma.sync GEMV: batch <= 16");
  if (mla_) {
    // types.hpp:43-49: MLA keeps one latent KV head; Helix needs tpa <= K_eff = 1 (types.cpp:122-139)
    W_ = static_cast<int>(2 * m.kv_latent);
    DV_ = W_ - 64;
    if (W_ != kMlaW) throw std::invalid_argument("MLA kernel supports kv_latent_dim = 288 (576-wide latent)");
    if (Kh_ != 1) throw std::invalid_argument("MLA keeps a single latent KV head");
    if (tpa_ != 1) throw std::invalid_argument("MLA needs tpa = 1 (tpa <= effective KV heads)");
    if (Qh_ > kMlaHeads) throw std::invalid_argument("MLA kernel supports at most 128 query heads");
    if (m.attention_only) throw std::invalid_argument("the attention-only harness is GQA (DecodeHarness)");
    if (par.distributed != HX_POOL_LOCAL && Qh_ % par.kvp)
      throw std::invalid_argument("MLA needs kvp to divide query_heads (the O-projection shards whole heads)");
  } else if (D_ > 128) {
    throw std::invalid_argument("head_size > 128 is not supported by the GQA decode kernel");
  }
  if (H_ % 16) throw std::invalid_argument("hidden width must be a multiple of 16");
  moe_ = !attn_only_ && m.n_experts > 0;
  if (moe_) {
    E_ = m.n_experts;
    topk_ = m.top_k;
    Fe_ = m.expert_ffn;
    if (topk_ < 1 || topk_ > 16 || topk_ > E_) throw std::invalid_argument("moe top_k must be in [1, min(16, experts)]");
    if (Fe_ < 16 || Fe_ % 16) throw std::invalid_argument("moe expert_ffn_dim must be a positive multiple of 16");
    if (E_ > 512) throw std::invalid_argument("at most 512 experts (register-resident routing)");
  }
  if (!attn_only_) {
    const bool shared_ok = moe_ && F_ == 0;  // MoE without a shared expert
    if (!shared_ok && (F_ < 16 || F_ % 16)) throw std::invalid_argument("ffn_dim must be a positive multiple of 16");
    if (V_ < 1) throw std::invalid_argument("vocab must be >= 1");
  }
  dist_mode_ = par.distributed;
  if (dist_mode_ != HX_POOL_LOCAL && dist_mode_ != HX_POOL_NCCL && dist_mode_ != HX_POOL_LOOPBACK)
    throw std::invalid_argument("unknown pool mode");

  DP_ = D_ <= 32 ? 32 : (D_ <= 64 ? 64 : 128);
  AD_ = mla_ ? DV_ : static_cast<int>(D_);   // per-head attention output width
  ADP_ = mla_ ? DV_ : DP_;                    // its stride in the fragment buffers
  G_ = static_cast<int>(Qh_ / Kh_);
  q_rows_ = G_ > 8 ? 16 : 8;  // a GQA group of 9-16 query heads shares one pass over its KV head
  q_chunks_ = mla_ ? 1 : (G_ + q_rows_ - 1) / q_rows_;
  kvh_per_slot_ = static_cast<int>(Kh_ / tpa_);
  q_per_slot_ = static_cast<int>(Qh_ / tpa_);
  N_ = tpa_ * kvp_;
  F_local_ = static_cast<int>(F_);
  V_local_ = static_cast<int>(V_);
  if (moe_) {  // expert parallelism (types.hpp:100): ep x tpf = tpa x kvp in a distributed pool
    ep_ = dist_mode_ == HX_POOL_LOCAL ? 1 : static_cast<int>(std::max<int64_t>(1, par.ep));
    if (N_ % ep_) throw std::invalid_argument("helix re-provisions one pool: kvp*tpa must equal tpf*ep");
    tpf_ = dist_mode_ == HX_POOL_LOCAL ? 1 : N_ / ep_;
    if (E_ % ep_) throw std::invalid_argument("ep must divide total_experts");
    if (Fe_ % tpf_ || (Fe_ / tpf_) % 16) throw std::invalid_argument("tpf must divide expert_ffn_dim (x16)");
    if (dist_mode_ != HX_POOL_LOCAL) {
      ep_rank_ = rank_ / tpf_;
      tpf_rank_ = rank_ % tpf_;
    }
    E_local_ = static_cast<int>(E_ / ep_);
    e_begin_ = ep_rank_ * E_local_;
    Fe_local_ = static_cast<int>(Fe_ / tpf_);
    n_groups_max_ = static_cast<int>(std::min<int64_t>(E_local_, static_cast<int64_t>(B_) * topk_));
  }
  if (dist_mode_ == HX_POOL_LOCAL) {
    n_slots_ = N_;
    slot_base_ = 0;
  } else {
    // One rank (r, g) of the Helix pool: its KV shard, its group's QKV slice,
    // its H/N slice of the exchange, 1/N of O-proj/FFN/LM head (latency.cpp:45-146).
    if (rank_ < 0 || rank_ >= N_) throw std::invalid_argument("rank out of range for tpa*kvp");
    grp_ = rank_ / kvp_;
    r_ = rank_ % kvp_;
    n_slots_ = 1;
    slot_base_ = rank_;
    slice_ = static_cast<int>(q_per_slot_ * AD_ / kvp_);
    if ((q_per_slot_ * AD_) % kvp_ || slice_ % 16)
      throw std::invalid_argument("distributed Helix needs hidden/(tpa*kvp) to be a multiple of 16");
    xchunk_ = static_cast<int>(exchange_layout(q_per_slot_, AD_, kvp_, nullptr));
    if (mla_) {
      uv_heads_ = static_cast<int>(Qh_ / kvp_);
      uv_h0_ = r_ * uv_heads_;
    }
    if (!attn_only_) {
      if (F_ % N_ || (F_ > 0 && (F_ / N_) % 16))
        throw std::invalid_argument("ffn_dim/(tpa*kvp) must be a multiple of 16");
      F_local_ = static_cast<int>(F_ / N_);
      V_local_ = static_cast<int>((V_ + N_ - 1) / N_);
    }
  }
  if (mla_ && dist_mode_ == HX_POOL_LOCAL) uv_heads_ = static_cast<int>(Qh_);
  // O-projection input: GQA the merged heads (all, or this rank's exchanged slice);
  // MLA the W_UV outputs of the heads held here (H, or H/N)
  K_o_ = mla_ ? uv_heads_ * static_cast<int>(D_)
              : (dist_mode_ == HX_POOL_LOCAL ? static_cast<int>(Qh_) * AD_ : slice_);
  const int64_t per_rank_max = ((cap_ + static_cast<int64_t>(chunk_) * kvp_ - 1) /
                                (static_cast<int64_t>(chunk_) * kvp_)) * chunk_;
  if (mla_) {
    page_cap_ = static_cast<int>((per_rank_max + kMlaPageRows - 1) / kMlaPageRows + 1);
    page_bytes_ = mla_page_bytes(kv8_);
  } else {
    page_cap_ = static_cast<int>((per_rank_max + 15) / 16 + 1);
    page_bytes_ = kv4_ ? page_bytes_kv4(DP_) : page_bytes_kv(DP_, kv8_);
  }
  if (f64_) {  // fp64 shards instead of bf16 pages (exact64.cu)
    rows_cap64_ = per_rank_max;
    page_cap_ = 1;
  }

  if (std::getenv("HX_NO_PDL")) set_pdl(false);  // debugging: serialise every launch
  // batches above 16 make the GEMV contraction dense enough for tcgen05 (gemv_tc.cu);
  // HX_TC_GEMV=0 keeps the mma.sync path (A/B measurements)
  tc_ = B_ > 16 && !(std::getenv("HX_TC_GEMV") && std::getenv("HX_TC_GEMV")[0] == '0');
  cuda_check(cudaSetDevice(device_), "cudaSetDevice");
  cudaDeviceProp prop{};
  cuda_check(cudaGetDeviceProperties(&prop, device_), "cudaGetDeviceProperties");
  if (prop.major < 10)
    throw CudaError("device is not sm_100 class (Blackwell); this build targets sm_100a only");
  num_sms_ = prop.multiProcessorCount;
  cuda_check(cudaStreamCreateWithFlags(&stream_, cudaStreamNonBlocking), "cudaStreamCreate");
  if (dist_mode_ == HX_POOL_NCCL) {
    if (!par.nccl_unique_id) throw std::invalid_argument("NCCL pool needs nccl_unique_id");
    transport_ = make_nccl_transport(par.nccl_unique_id, rank_, tpa_, kvp_);
  } else if (dist_mode_ == HX_POOL_LOOPBACK) {
    if (!par.loopback) throw std::invalid_argument("loopback pool needs a loopback group");
    transport_ = make_loopback_transport(reinterpret_cast<LoopbackHub*>(par.loopback), rank_, tpa_, kvp_);
    // host barriers inside the loopback collectives cannot be captured; graphs
    // stay possible only while both collectives are switched off (measurement)
    loopback_ = true;
  }
  if (dist_mode_ != HX_POOL_LOCAL) {
    // the largest collective: the [B x H] fp32 TP partials (loopback scratch allocated now, not mid-step)
    transport_->reserve(static_cast<size_t>(B_) * H_ * sizeof(float));
    cuda_check(cudaStreamCreateWithFlags(&comm_stream_, cudaStreamNonBlocking), "comm stream");
    hop_events_.resize(static_cast<size_t>(B_) + 1);
    for (auto& e : hop_events_) cuda_check(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
  }
  alloc();
  plan_gemvs();
}

Engine::~Engine() {
  drop_graphs();
  auto f = [](void* p) {
    if (p) cudaFree(p);
  };
  for (auto* p : kv_) f(p);
  for (auto* p : w_qkv_) f(p);
  for (auto* p : w_o_) f(p);
  for (auto* p : w_gu_) f(p);
  for (auto* p : w_down_) f(p);
  for (auto* p : w_router_) f(p);
  for (auto* p : w_egu_) f(p);
  for (auto* p : w_edown_) f(p);
  f(d_qimg_);
  f(d_att_);
  for (auto* p : w_uk_) f(p);
  for (auto* p : w_uv_) f(p);
  f(d_rlog_); f(d_route_w_); f(d_gids_); f(d_gcount_); f(d_xf_em_); f(d_moe_y_);
  f(w_lm_); f(emb_); f(d_total_); f(d_q_); f(d_part_o_); f(d_part_lse_); f(d_work_);
  f(d_frag_o_); f(d_frag_lse_); f(d_ypart_); f(d_counters_); f(d_x_); f(d_ss_); f(d_m_);
  f(d_logits_); f(d_best_); f(d_tokens_); f(d_next_); f(d_out_); f(d_out_lse_); f(d_hidden_);
  f(d_stream_done_); f(d_pushed_); f(d_flags_); f(d_peer_recv_); f(d_peer_flag_); f(d_self_recv_); f(d_self_flag_);
  f(d_segs_); f(d_send_); f(d_recv_); f(d_parth_); f(d_xf_resid_); f(d_xf_attn_); f(d_xf_m_); f(d_plan_ctr_);
  for (auto* p : k64_) f(p);
  for (auto* p : v64_) f(p);
  for (auto* p : w64_) f(p);
  f(d_x64_); f(d_qkv64_); f(d_frag64_o_); f(d_frag64_lse_); f(d_out64_); f(d_lse64_);
  for (auto& e : hop_events_) cudaEventDestroy(e);
  delete transport_;
  if (comm_stream_) cudaStreamDestroy(comm_stream_);
  if (stream_) cudaStreamDestroy(stream_);
}

void Engine::validate_reference_dims() const {
  // Same checks, same order, same messages as the reference:
  // ShardedKVCache ctor (attention.hpp:239-240) then DecodeHarness ctor (:431-437).
  if (kvp_ < 1 || Kh_ < 1 || D_ < 1 || chunk_ < 1)
    throw std::invalid_argument("cache dimensions must be >= 1");
  if (tpa_ < 1 || kvp_ < 1) throw std::invalid_argument("tpa and kvp must be >= 1");
  if (Qh_ % Kh_ != 0) throw std::invalid_argument("query_heads must be a multiple of kv_heads");
  if (Kh_ % tpa_ != 0) throw std::invalid_argument("tpa must divide kv_heads");
  if ((Qh_ * D_) % (static_cast<int64_t>(tpa_) * kvp_) != 0)
    throw std::invalid_argument("tpa*kvp must divide the hidden width");
}

// Splits per stream for `pages` pages of KV per stream.
// GQA: equal-size items pulled by one persistent CTA per SM cost waves x
// (pages per item + per-item overhead ~16 pages: query staging and the
// cross-warp combine), waves = ceil(items / SMs); minimised over the split
// count with items >= 32 pages (256 KB at Hsz 128: below that the per-item
// overhead dominates -- one 131k-token request of the 405B-like shard 0.196 ->
// 0.131 ms). An item count that is a multiple of the SM count leaves no tail
// (configs[1]: 64 streams x 37 splits = 16 x 148; 20.5 -> 20.0 ms of attention
// per step vs 19 splits). MLA: one item per CTA pair, statically strided.
int Engine::plan_splits(int streams, int pages) const {
  if (mla_) return std::max(1, std::min((num_sms_ / 2) / streams, std::max(1, pages / 2)));
  const int smax = std::max(1, pages / std::max(1, min_pages_));
  if (split_env_) return std::max(1, std::min((num_sms_ * std::max(1, ips_) + streams - 1) / streams, smax));
  int best = 1;
  double best_cost = 1e300;
  for (int sp = 1; sp <= smax && sp <= 8192; ++sp) {
    const long long waves = (static_cast<long long>(streams) * sp + num_sms_ - 1) / num_sms_;
    const double cost = static_cast<double>(waves) * ((pages + sp - 1) / sp + 16.0);
    if (cost < best_cost) {
      best_cost = cost;
      best = sp;
    }
  }
  return best;
}

// Splits for a launch over `layer`'s live context (pages of the fullest rank --
// rank 0 -- rounded up to a power of two, so a growing context re-plans, and
// re-captures the step graph, only log2 times), never above the capacity plan
// the partial buffers are sized for.
int Engine::live_splits(int64_t layer, bool per_request) const {
  int64_t tmax = 0;
  for (int b = 0; b < B_; ++b) tmax = std::max(tmax, h_total_[static_cast<size_t>(layer * B_ + b)]);
  const int64_t rows = rr_count(tmax, 0, chunk_, kvp_);
  const int64_t unit = mla_ ? kMlaPageRows : 16;
  int pages = 1;
  while (pages < (rows + unit - 1) / unit && pages < page_cap_) pages *= 2;
  pages = std::min(pages, page_cap_);
  const int streams = per_request ? n_streams_ / B_ : n_streams_;
  return std::min(plan_splits(streams, pages), per_request ? splits_req_ : splits_);
}

void Engine::alloc() {
  const size_t pool = static_cast<size_t>(n_slots_) * B_ * kvh_per_slot_ * page_cap_ * page_bytes_;
  for (int64_t l = 0; l < L_; ++l) kv_.push_back(dalloc<uint8_t>(pool, "kv pool"));
  if (mla_) {  // 2-SM TMA views of each layer's latent pool (mla.cu)
    mla_tm_.resize(static_cast<size_t>(L_));
    for (int64_t l = 0; l < L_; ++l)
      cuda_check(make_mla_tensor_maps(kv_[l], pool, mla_tm_[l].s, mla_tm_[l].v, kv8_), "mla tensor maps");
  }
  d_total_ = dalloc<int>(static_cast<size_t>(L_) * B_, "totals");
  h_total_.assign(static_cast<size_t>(L_ * B_), 0);
  const int qh_buf = dist_mode_ == HX_POOL_LOCAL ? static_cast<int>(Qh_) : q_per_slot_;
  d_q_ = dalloc<float>(static_cast<size_t>(B_) * qh_buf * DP_, "q");

  // attention work decomposition: balanced page ranges ("splits") per stream.
  // Buffers are sized for the capacity; every launch re-plans from the LIVE
  // context (plan_splits / live_splits), so short contexts in a large engine
  // keep items of useful size.
  const char* split_env = std::getenv("HX_ATTN_SPLIT");  // "items_per_sm,min_pages_per_item" (tuning)
  if (split_env) {
    split_env_ = true;
    std::sscanf(split_env, "%d,%d", &ips_, &min_pages_);
  }
  // tcgen05 kernel for quantised pages: opt-in (HX_ATTN_TC=1) -- the e4m3 / e2m1
  // widening it still pays on the CUDA cores keeps it behind the legacy kernel
  // (K1-TC)
  attn_tc_ = !mla_ && kv8_ && DP_ == 128 && q_chunks_ == 1 && std::getenv("HX_ATTN_TC") &&
             std::getenv("HX_ATTN_TC")[0] == '1';
  // the tcgen05 kernel reads K straight from its pages (kind::f8f6f4): FP8 pages
  // in the tensor-core layout, which only it reads -- so no in-kernel HOP-B reduce
  kv8tc_ = attn_tc_;
  n_streams_ = n_slots_ * B_ * kvh_per_slot_ * q_chunks_;
  const int req_streams = n_slots_ * kvh_per_slot_ * q_chunks_;
  splits_ = plan_splits(n_streams_, page_cap_);
  splits_req_ = plan_splits(req_streams, page_cap_);
  n_items_ = std::max(n_streams_ * splits_, req_streams * splits_req_);
  if (mla_) {
    d_qimg_ = dalloc<uint8_t>(static_cast<size_t>(B_) * mla_q_bytes(kv8_), "mla query images");
    d_att_ = dalloc<float>(static_cast<size_t>(B_) * (dist_mode_ == HX_POOL_LOCAL ? Qh_ * DV_ : slice_),
                           "mla merged latent output");
  }
  attn_grid_ = std::min(mla_ ? num_sms_ / 2 : num_sms_, n_items_);  // MLA: CTA pairs
  if (std::getenv("HX_FUSED_REDUCE") && std::getenv("HX_FUSED_REDUCE")[0] == '0') fused_ = false;
  hopb_inkernel_ = !kv8tc_ && std::getenv("HX_HOPB_INKERNEL") && std::getenv("HX_HOPB_INKERNEL")[0] == '1';
  local_stream_reduce_ = std::getenv("HX_LOCAL_STREAM_REDUCE") && std::getenv("HX_LOCAL_STREAM_REDUCE")[0] == '1';
  if (std::getenv("HX_HOPB_GROUP")) hopb_group_ = std::max(1, std::atoi(std::getenv("HX_HOPB_GROUP")));
  if (std::getenv("HX_A2A_NCCL") && std::getenv("HX_A2A_NCCL")[0] == '1') nccl_a2a_ = true;
  // [n_streams] finished splits, [n_streams] finished reducer chunks (HOP-B stream reducer)
  d_stream_done_ = dalloc<int>(2 * static_cast<size_t>(std::max(n_streams_, 1)), "stream done counters");
  d_pushed_ = dalloc<int>(1, "pushed counter");
  if (dist_mode_ != HX_POOL_LOCAL) {
    d_flags_ = dalloc<unsigned>(static_cast<size_t>(kvp_), "exchange flags");
    d_peer_recv_ = dalloc<float*>(static_cast<size_t>(kvp_), "peer recv table");
    d_peer_flag_ = dalloc<unsigned*>(static_cast<size_t>(kvp_), "peer flag table");
    d_self_recv_ = dalloc<float*>(static_cast<size_t>(kvp_), "self recv table");
    d_self_flag_ = dalloc<unsigned*>(static_cast<size_t>(kvp_), "self flag table");
    d_send_ = dalloc<float>(static_cast<size_t>(kvp_) * B_ * xchunk_, "exchange send");
    d_recv_ = dalloc<float>(static_cast<size_t>(kvp_) * B_ * xchunk_, "exchange recv");
    // HX_FLAG_SKIP_COMM stand-ins of the peer tables: every slice and flag stays on this rank
    const std::vector<float*> sr(static_cast<size_t>(kvp_), d_recv_);
    const std::vector<unsigned*> sf(static_cast<size_t>(kvp_), d_flags_ + r_);
    cuda_check(cudaMemcpy(d_self_recv_, sr.data(), sr.size() * sizeof(float*), cudaMemcpyHostToDevice), "self table");
    cuda_check(cudaMemcpy(d_self_flag_, sf.data(), sf.size() * sizeof(unsigned*), cudaMemcpyHostToDevice), "self table");
    d_parth_ = dalloc<float>(static_cast<size_t>(B_) * H_, "tp partial");
  }
  const size_t part_rows = mla_ ? static_cast<size_t>(kMlaHeads) : static_cast<size_t>(q_rows_);  // rows per item
  const size_t part_w = mla_ ? static_cast<size_t>(DV_) : static_cast<size_t>(DP_);
  d_part_o_ = dalloc<float>(static_cast<size_t>(n_items_) * part_rows * part_w, "part_o");
  d_part_lse_ = dalloc<float>(static_cast<size_t>(n_items_) * part_rows, "part_lse");
  d_work_ = dalloc<int>(4, "work counters");
  d_frag_o_ = dalloc<float>(static_cast<size_t>(n_slots_) * B_ * q_per_slot_ * ADP_, "frag_o");
  d_frag_lse_ = dalloc<float>(static_cast<size_t>(n_slots_) * B_ * q_per_slot_, "frag_lse");
  d_x_ = dalloc<float>(static_cast<size_t>(B_) * H_, "x");
  d_out_ = dalloc<float>(static_cast<size_t>(B_) * Qh_ * D_, "out");
  d_out_lse_ = dalloc<float>(static_cast<size_t>(B_) * Qh_, "out_lse");
  d_tokens_ = dalloc<int>(B_, "tokens");
  d_next_ = dalloc<int>(B_, "next");
  d_best_ = dalloc<unsigned long long>(B_, "best");
  d_segs_ = dalloc<WSeg>(16, "segs");
  if (f64_) {
    const size_t shard = static_cast<size_t>(n_slots_) * B_ * kvh_per_slot_ * rows_cap64_ * D_;
    const size_t ncols = static_cast<size_t>(Qh_ + 2 * Kh_) * D_;
    for (int64_t l = 0; l < L_; ++l) {
      k64_.push_back(dalloc<double>(shard, "f64 K shards"));
      v64_.push_back(dalloc<double>(shard, "f64 V shards"));
      w64_.push_back(dalloc<double>(static_cast<size_t>(H_) * ncols, "f64 qkv weights"));
    }
    d_x64_ = dalloc<double>(static_cast<size_t>(B_) * H_, "f64 x");
    d_qkv64_ = dalloc<double>(static_cast<size_t>(B_) * ncols, "f64 qkv");
    d_frag64_o_ = dalloc<double>(static_cast<size_t>(n_slots_) * B_ * q_per_slot_ * D_, "f64 frag_o");
    d_frag64_lse_ = dalloc<double>(static_cast<size_t>(n_slots_) * B_ * q_per_slot_, "f64 frag_lse");
    d_out64_ = dalloc<double>(static_cast<size_t>(B_) * Qh_ * D_, "f64 out");
    d_lse64_ = dalloc<double>(static_cast<size_t>(B_) * Qh_, "f64 lse");
  }
}

// ---------------------------------------------------------------------------
void Engine::plan_gemvs() {
  one_src_merge_ = dist_mode_ == HX_POOL_LOCAL && !mla_ && !attn_only_ && kvp_ == 1 &&
                   !(std::getenv("HX_ONE_SRC_MERGE") && std::getenv("HX_ONE_SRC_MERGE")[0] == '0');
  // fused LSE combine in the O-projection (GQA; the tcgen05 GEMV and MLA keep the merge kernel)
  fused_combine_ = !mla_ && !attn_only_ && !tc_ && !one_src_merge_ &&
                   !(std::getenv("HX_FUSED_COMBINE") && std::getenv("HX_FUSED_COMBINE")[0] == '0');
  d_plan_ctr_ = dalloc<int>(static_cast<size_t>(2 * (7 * L_ + 2) + L_), "plan counters");
  int plan_idx = 0;
  // groups: expected concurrent weight blocks (MoE: active experts) for tile sizing
  auto make = [&](int N, int Npad, int K, int norm, int em, int groups = 1) {
    GemvPlan g;
    GemvParams& p = g.p;
    if (tc_) {  // tcgen05 tiles are row-block PAIRS over k-chunks of whole 4-k-step x blocks
      Npad = round_up(Npad, 256);
      if (K % 64) throw std::invalid_argument("batches above 16 need GEMV input widths that are multiples of 64");
    }
    p.N = N;
    p.Npad = Npad;
    p.K = K;
    p.batch = B_;
    // Persistent GEMV: tiles = (128-row block, k-chunk of kr k-steps) pulled
    // from a queue by one CTA per SM. kr shrinks until there are >= 2 tiles per
    // SM (dynamic balance, <= one short tile of tail); kr >= 8 keeps a tile >= 32 KB,
    // and <= 32 k-chunks keep the epilogue's split-K sum short for narrow outputs
    // (router, sharded LM head: a few row blocks over a long K).
    const int kst = K / 16;
    const int nblk = Npad / 128;
    const int tile_blks = tc_ ? nblk / 2 : nblk;  // row blocks (tc: pairs) per k-chunk
    // tcgen05 plans (batch > 16): the split-K partials grow with the batch
    // (ksplit x B x Npad fp32), so cap them at ~1/4 of the weight bytes
    // (ksplit <= K / (8 B)) and let a tile span the whole K when that suffices
    const int max_ks = tc_ ? std::max(1, std::min(32, static_cast<int>(K / (8 * B_)))) : 32;
    // >= 2 tiles per SM: measured against 4 and 1 at configs[1] (O-proj 0.95 -> 0.75 ms and
    // down 1.27 -> 1.13 ms per step: fewer split-K partials for the epilogue to reduce)
    int tiles_per_sm = 2;  // HX_GEMV_TILES="tiles_per_sm" (tuning experiments)
    if (const char* e = std::getenv("HX_GEMV_TILES")) tiles_per_sm = std::max(1, std::atoi(e));
    const int target = tiles_per_sm * num_sms_;
    int kr = tc_ ? kst : std::min(64, kst);
    while (kr > 8 && (!tc_ || (kr / 2) % 4 == 0) && (kst + kr / 2 - 1) / (kr / 2) <= max_ks &&
           static_cast<int64_t>(tile_blks) * groups * ((kst + kr - 1) / kr) < target)
      kr /= 2;
    if (w4_) {  // FP4 weights stream in 32-input blocks (2 k-steps): even chunks
      if (K % 32) throw std::invalid_argument("FP4 weights: GEMV input widths must be multiples of 32");
      kr += kr & 1;
    }
    const int ksplit = (kst + kr - 1) / kr;
    p.ksplit = ksplit;
    p.kr_steps = kr;
    p.n_tiles = tile_blks * ksplit;
    p.work_counter = d_plan_ctr_ + 2 * plan_idx++;
    p.eps = 1e-5f;
    p.kvp = kvp_;
    p.head_dim = static_cast<int>(D_);
    p.dp = DP_;
    p.tc = tc_ ? 1 : 0;
    p.w8 = w4_ ? 2 : (w8_ ? 1 : 0);  // FP8: wscale is wired by the weight init
    p.xf16 = xf16_();
    p.prefetch_stages = 4;  // weight stages before griddepcontrol.wait; HX_GEMV_PREFETCH: A/B experiments
    if (const char* e = std::getenv("HX_GEMV_PREFETCH")) p.prefetch_stages = std::atoi(e);
    g.xmode = norm;
    g.emode = em;
    ypart_elems_ = std::max(ypart_elems_, static_cast<size_t>(groups) * ksplit * B_ * Npad);
    max_counters_ = std::max(max_counters_, nblk);
    return g;
  };
  const bool dist = dist_mode_ != HX_POOL_LOCAL;
  // MLA: q (head_size per head, absorbed into the latent by mla_absorb_q) + one latent row
  const int nq = static_cast<int>((dist ? q_per_slot_ : Qh_) * D_);
  const int nk = mla_ ? W_ : static_cast<int>((dist ? kvh_per_slot_ : Kh_) * D_);
  const int Nqkv = nq + (mla_ ? 1 : 2) * nk;
  const int Hh = static_cast<int>(H_);
  const int F = F_local_;
  for (int64_t l = 0; l < L_; ++l) {
    GemvPlan q = make(Nqkv, round_up(Nqkv, 128), Hh, attn_only_ ? 0 : 1, E_QKV);
    q.p.nq = nq;
    q.p.nk = nk;
    q.p.kv_heads = mla_ ? 1 : nk / static_cast<int>(D_);
    q.p.mla = mla_ ? 1 : 0;
    q.p.kv_head_base = dist ? grp_ * kvh_per_slot_ : 0;
    q.p.kvh_per_slot = kvh_per_slot_;
    q.p.rr_chunk = chunk_;
    q.p.page_cap = page_cap_;
    q.p.slot_base = slot_base_;
    q.p.n_local_slots = n_slots_;
    q.p.append = 1;
    q.p.kv8 = kv8_fmt();
    q.p.kv4 = kv4_ ? 1 : 0;
    plan_qkv_.push_back(q);
    if (!attn_only_) {
      if (dist) {
        // O-proj: this rank's exchanged slice of its group's heads x its rows of W_O
        plan_o_.push_back(make(Hh, round_up(Hh, 128), K_o_, 0, E_STORE));
      } else {
        plan_o_.push_back(make(Hh, round_up(Hh, 128), K_o_, 0, E_RESID));
      }
      if (F > 0) {  // dense FFN, or the MoE shared expert
        plan_gu_.push_back(make(2 * F, round_up(F, 64) * 2, Hh, 1, E_SWIGLU));
        plan_down_.push_back(make(Hh, round_up(Hh, 128), F, 0, dist ? E_STORE : E_RESID));
      }
    }
  }
  if (moe_) {
    // router -> top-k -> grouped expert GEMVs whose tile queue covers only the
    // experts some request selected (group list written by the routing kernel)
    const int E = static_cast<int>(E_), Fe = Fe_local_, G = n_groups_max_;
    const int nb8 = xf_nb8(B_);
    const long long xfe = static_cast<long long>(Fe / 16) * 3 * nb8 * 256;
    const bool shared = F_ > 0;
    for (int64_t l = 0; l < L_; ++l) {
      GemvPlan r = make(E, round_up(E, 128), Hh, 1, E_STORE);
      r.p.out_stride = E;
      plan_router_.push_back(r);
      GemvPlan gu = make(2 * Fe, round_up(Fe, 64) * 2, Hh, 1, E_SWIGLU, G);
      GemvPlan dn = make(Hh, round_up(Hh, 128), Fe, 0, (dist || shared) ? E_STORE : E_RESID, G);
      for (GemvPlan* g : {&gu, &dn}) {
        GemvParams& p = g->p;
        p.tiles_per_group = p.n_tiles;
        p.n_groups_max = G;
        p.group_base = e_begin_;
        p.w_group_stride = static_cast<long long>(weight_bytes(p.Npad, p.K));
        p.part_group_stride = static_cast<long long>(p.ksplit) * B_ * p.Npad;
        p.n_experts = E;
      }
      gu.p.xf_group_stride = 0;  // every expert reads the same normalised h
      gu.p.xf_out_group_stride = xfe;
      dn.p.xf_group_stride = xfe;
      plan_egu_.push_back(gu);
      plan_edown_.push_back(dn);
    }
    d_rlog_ = dalloc<float>(static_cast<size_t>(B_) * E, "router logits");
    d_route_w_ = dalloc<float>(static_cast<size_t>(B_) * E, "route weights");
    d_gids_ = dalloc<int>(static_cast<size_t>(std::max(G, 1)), "expert list");
    d_gcount_ = dalloc<int>(1, "expert count");
    d_xf_em_ = dalloc<uint8_t>(static_cast<size_t>(std::max(G, 1)) * xfe, "expert xf");
    if (shared) d_moe_y_ = dalloc<float>(static_cast<size_t>(B_) * H_, "moe y");
  }
  if (!attn_only_) {
    plan_lm_ = make(V_local_, round_up(V_local_, 128), Hh, 1, E_LOGITS);
    plan_lm_.p.n_offset = dist ? rank_ * V_local_ : 0;
  }

  d_ypart_ = dalloc<float>(ypart_elems_, "ypart");
  {
    const int nb8 = xf_nb8(B_);
    auto xf_alloc = [&](int K) { return dalloc<uint8_t>(static_cast<size_t>(K / 16) * 3 * nb8 * 256, "xf"); };
    d_xf_resid_ = xf_alloc(static_cast<int>(H_));
    d_xf_attn_ = xf_alloc(K_o_);
    d_xf_m_ = xf_alloc(std::max(16, F_local_));
  }
  d_counters_ = dalloc<int>(static_cast<size_t>(max_counters_), "counters");
  const int hblk = round_up(Hh, 128) / 128;
  d_ss_ = dalloc<float>(static_cast<size_t>(std::max(hblk, 1)) * B_, "ss");
  if (!attn_only_) {
    d_m_ = dalloc<float>(static_cast<size_t>(B_) * F_local_, "m");
    d_logits_ = dalloc<float>(static_cast<size_t>(B_) * V_local_, "logits");
    d_hidden_ = dalloc<float>(static_cast<size_t>(L_ + 1) * B_ * H_, "hidden");
  }
}

// Kernel launches of one step as the engine enqueues it now (each GEMV =
// streaming kernel + epilogue kernel; NCCL's own kernels not counted).
int64_t Engine::launches_per_step() const {
  const int64_t ffn_k = moe_ ? 7 + (F_ > 0 ? 4 : 0) : 4;  // dense 4; MoE router 2 + route + experts 4 (+ shared 4)
  const int64_t sr = 1;                                    // split-reduce kernel (fused under device_exchange())
  if (attn_only_) return f64_ ? 3 + 2 * B_ : 4 + sr + 1;  // xprep, qkv x2, attention, split-reduce, merge
  const int64_t head = 1 + 3;                              // embed; LM head x2 + argmax finish
  const int64_t mla_k = mla_ ? 2 : 0;                      // W_UK absorption, W_UV
  if (dist_mode_ == HX_POOL_LOCAL)
    return head + L_ * (2 + 1 + sr + (one_src_merge_ || fused_combine_ ? 0 : 1) + mla_k + 2 + ffn_k);
  const int64_t attn = device_exchange() ? (hopb_ && fused_ && hopb_inkernel_ ? 2 : 3)  // attention, reduce + push, flag wait
                                         : (hopb_ ? B_ : 1) * (2 + sr);  // [per request] attention, sr, pack
  return head + L_ * (2 + attn + (fused_combine_ ? 0 : 1) + mla_k + 2 + 1 + ffn_k + 1);  // + merge, O x2, residual, FFN, residual
}

// ---------------------------------------------------------------------------
void Engine::build_weights_common(uint64_t seed, bool qkv_hash) {
  const bool dist = dist_mode_ != HX_POOL_LOCAL;
  const int Hh = static_cast<int>(H_);
  // columns of W_q / W_k / W_v held here (all, or this rank's TPA group's heads)
  const int nq = static_cast<int>((dist ? q_per_slot_ : Qh_) * D_);
  const int nk = static_cast<int>((dist ? kvh_per_slot_ : Kh_) * D_);
  const int q0 = dist ? grp_ * nq : 0, k0 = dist ? grp_ * nk : 0;
  const int F = F_local_, f0 = dist ? rank_ * F_local_ : 0;
  const int v0 = dist ? rank_ * V_local_ : 0;
  const int vrows = static_cast<int>(std::min<int64_t>(V_local_, V_ - v0));
  auto wchunks = [&](const GemvPlan& g) { return weight_bytes(g.p.Npad, g.p.K) / 16; };  // uint4 per matrix
  auto walloc = [&](const GemvPlan& g) { return dalloc<uint4>(wchunks(g), "weights"); };
  // k_full: the input width of the whole (unsharded) matrix -- FP8 scales span it
  // (grouped expert blocks pass their slice of one [E_local][Npad] scale array)
  auto init = [&](uint4* w, GemvPlan& g, const std::vector<WSeg>& segs, int k_full, float* sc_slice = nullptr) {
    cuda_check(cudaMemcpyAsync(d_segs_, segs.data(), segs.size() * sizeof(WSeg), cudaMemcpyHostToDevice,
                               stream_), "segs");
    if (w4_) {  // e2m1 blocks of 32 inputs with their scales inline (gemv.cu FP4 tile image)
      cuda_check(launch_weight_init_hash_w4(reinterpret_cast<uint8_t*>(w), g.p.Npad, g.p.K, d_segs_,
                                            static_cast<int>(segs.size()), seed, stream_), "weight init");
    } else if (w8_) {
      float* sc = sc_slice;
      if (!sc) {
        float*& slot = wscale_[w];
        if (!slot) slot = dalloc<float>(static_cast<size_t>(g.p.Npad), "weight scales");
        sc = slot;
      }
      cuda_check(launch_weight_init_hash_w8(reinterpret_cast<uint8_t*>(w), sc, g.p.Npad, g.p.K, k_full, d_segs_,
                                            static_cast<int>(segs.size()), seed, stream_), "weight init");
      g.p.wscale = sc;
    } else {
      cuda_check(launch_weight_init_hash(w, g.p.Npad, g.p.K, d_segs_, static_cast<int>(segs.size()), seed,
                                         stream_, tc_ ? 1 : 0), "weight init");
    }
    cuda_check(cudaStreamSynchronize(stream_), "weight init sync");
  };
  // WSeg: {stream, rows_begin, rows_end, cols_total, col_offset, interleave, scale, k_offset, col_limit}
  const double sh = 1.0 / std::sqrt(static_cast<double>(H_));
  const double sf = 1.0 / std::sqrt(static_cast<double>(F_));
  const int Qall = static_cast<int>(Qh_ * D_), Kall = static_cast<int>(Kh_ * D_);
  for (int64_t l = 0; l < L_; ++l) {
    if (w_qkv_.size() <= static_cast<size_t>(l)) w_qkv_.push_back(walloc(plan_qkv_[l]));
    if (mla_) {  // W_q [H x Q*Hsz] (kWq) and the latent down-projection (kWk), both 1/sqrt(H)
      init(w_qkv_[l], plan_qkv_[l],
           {{hash_stream(kWq, l), 0, nq, nq, 0, 0, sh, 0, 0},
            {hash_stream(kWk, l), nq, nq + W_, W_, 0, 0, sh, 0, 0}}, Hh);
      // per-head absorptions: W_UK for every head, W_UV for the heads held here
      const long long uk = Qh_ * D_ * W_, uv = static_cast<long long>(uv_heads_) * DV_ * D_;
      if (w_uk_.size() <= static_cast<size_t>(l)) {
        w_uk_.push_back(dalloc<uint16_t>(static_cast<size_t>(uk), "w_uk"));
        w_uv_.push_back(dalloc<uint16_t>(static_cast<size_t>(uv), "w_uv"));
      }
      cuda_check(launch_plain_init_hash(w_uk_[l], uk, seed, hash_stream(kWuk, l), 0,
                                        16.0 / std::sqrt(static_cast<double>(D_)), stream_), "w_uk init");
      cuda_check(launch_plain_init_hash(w_uv_[l], uv, seed, hash_stream(kWuv, l),
                                        static_cast<long long>(uv_h0_) * DV_ * D_,
                                        1.0 / std::sqrt(static_cast<double>(DV_)), stream_), "w_uv init");
    } else if (qkv_hash) {
      init(w_qkv_[l], plan_qkv_[l],
           {{hash_stream(kWq, l), 0, nq, Qall, q0, 0, 1.0, 0, 0},
            {hash_stream(kWk, l), nq, nq + nk, Kall, k0, 0, 1.0, 0, 0},
            {hash_stream(kWv, l), nq + nk, nq + 2 * nk, Kall, k0, 0, 1.0, 0, 0}}, Hh);
    }
    plan_qkv_[l].p.w = w_qkv_[l];
    if (!attn_only_) {
      if (w_o_.size() <= static_cast<size_t>(l)) {
        w_o_.push_back(walloc(plan_o_[l]));
        if (F > 0) {
          w_gu_.push_back(walloc(plan_gu_[l]));
          w_down_.push_back(walloc(plan_down_[l]));
        }
      }
      // O-proj input rows: this rank's slice of its group's flattened heads
      // (MLA: the rows of the W_UV outputs of this rank's heads)
      const int ko = !dist ? 0 : (mla_ ? uv_h0_ * static_cast<int>(D_) : grp_ * q_per_slot_ * AD_ + r_ * slice_);
      init(w_o_[l], plan_o_[l], {{hash_stream(kWo, l), 0, Hh, Hh, 0, 0, sh, ko, 0}}, Hh);
      plan_o_[l].p.w = w_o_[l];
      plan_o_[l].p.bump_total = (one_src_merge_ || fused_combine_) ? d_total_ + l * B_ : nullptr;
      if (F > 0) {
        init(w_gu_[l], plan_gu_[l],
             {{hash_stream(kWgate, l), 0, plan_gu_[l].p.Npad, static_cast<int>(F_), f0, 1, sh, 0, f0 + F},
              {hash_stream(kWup, l), 0, plan_gu_[l].p.Npad, static_cast<int>(F_), f0, 2, sh, 0, f0 + F}}, Hh);
        init(w_down_[l], plan_down_[l], {{hash_stream(kWdown, l), 0, Hh, Hh, 0, 0, sf, f0, 0}},
             static_cast<int>(F_));
        plan_gu_[l].p.w = w_gu_[l];
        plan_down_[l].p.w = w_down_[l];
      }
    }
    if (moe_) {
      // router replicated; experts [e_begin, e_begin + E_local) of this EP group,
      // each sliced to this rank's tpf share of the expert FFN width
      GemvPlan& r = plan_router_[l];
      GemvPlan& gu = plan_egu_[l];
      GemvPlan& dn = plan_edown_[l];
      if (w_router_.size() <= static_cast<size_t>(l)) {
        w_router_.push_back(walloc(r));
        w_egu_.push_back(dalloc<uint4>(static_cast<size_t>(E_local_) * wchunks(gu), "expert gate/up"));
        w_edown_.push_back(dalloc<uint4>(static_cast<size_t>(E_local_) * wchunks(dn), "expert down"));
        if (w8_) {
          wscale_[w_egu_.back()] = dalloc<float>(static_cast<size_t>(E_local_) * gu.p.Npad, "expert scales");
          wscale_[w_edown_.back()] = dalloc<float>(static_cast<size_t>(E_local_) * dn.p.Npad, "expert scales");
        }
      }
      const int E = static_cast<int>(E_), Fe = Fe_local_, fe0 = tpf_rank_ * Fe_local_;
      const double se = 1.0 / std::sqrt(static_cast<double>(Fe_));
      init(w_router_[l], r, {{hash_stream(kWrouter, l), 0, E, E, 0, 0, sh, 0, 0}}, Hh);
      for (int el = 0; el < E_local_; ++el) {
        const int64_t e = e_begin_ + el;
        init(w_egu_[l] + static_cast<size_t>(el) * wchunks(gu), gu,
             {{expert_stream(kEgate, l, e), 0, gu.p.Npad, static_cast<int>(Fe_), fe0, 1, sh, 0, fe0 + Fe},
              {expert_stream(kEup, l, e), 0, gu.p.Npad, static_cast<int>(Fe_), fe0, 2, sh, 0, fe0 + Fe}}, Hh,
             w8_ ? wscale_[w_egu_[l]] + static_cast<size_t>(el) * gu.p.Npad : nullptr);
        init(w_edown_[l] + static_cast<size_t>(el) * wchunks(dn), dn,
             {{expert_stream(kEdown, l, e), 0, Hh, Hh, 0, 0, se, fe0, 0}}, static_cast<int>(Fe_),
             w8_ ? wscale_[w_edown_[l]] + static_cast<size_t>(el) * dn.p.Npad : nullptr);
      }
      r.p.w = w_router_[l];
      gu.p.w = w_egu_[l];
      dn.p.w = w_edown_[l];
      if (w8_) {  // every expert's scales (indexed by expert id - group_base in the epilogue)
        gu.p.wscale = wscale_[w_egu_[l]];
        dn.p.wscale = wscale_[w_edown_[l]];
      }
    }
  }
  if (!attn_only_) {
    if (!w_lm_) w_lm_ = walloc(plan_lm_);
    init(w_lm_, plan_lm_, {{hash_stream(kLm, 0), 0, vrows, static_cast<int>(V_), v0, 0, sh, 0, 0}}, Hh);
    plan_lm_.p.w = w_lm_;
    if (!emb_) emb_ = dalloc<uint16_t>(static_cast<size_t>(V_) * H_, "embedding");
    cuda_check(launch_emb_init_hash(emb_, static_cast<int>(V_), Hh, seed, hash_stream(kEmb, 0), stream_),
               "emb init");
    cuda_check(cudaStreamSynchronize(stream_), "emb init sync");
  }
  // wire the remaining pointers of every plan
  const int hblk = round_up(Hh, 128) / 128;
  for (int64_t l = 0; l < L_; ++l) {
    GemvParams& q = plan_qkv_[l].p;
    q.ypart = d_ypart_;
    q.counters = d_counters_;
    q.q_out = d_q_;
    q.q_img = d_qimg_;
    q.kv = kv_[l];
    q.total = d_total_ + l * B_;
    q.xf = d_xf_resid_;  // harness: the host x prepared into the same buffer
    q.ss_part = d_ss_;
    q.n_ss = hblk;  // per-128-column-block partials from the embedding / residual writers
    if (!attn_only_) {
      GemvParams& o = plan_o_[l].p;
      o.ypart = d_ypart_;
      o.counters = d_counters_;
      o.xf = d_xf_attn_;
      o.out = dist ? d_parth_ : d_x_;
      o.out_stride = static_cast<int>(H_);
      o.ss_out = dist ? nullptr : d_ss_;
      o.xf_out = d_xf_resid_;
      if (fused_combine_) {
        o.merge = dist ? 1 : 2;
        if (const char* e = std::getenv("HX_FUSED_COMBINE_DEBUG")) o.merge |= std::atoi(e);  // 4: no wait, 8: no merge (timing only)
        o.merge_ctr = d_plan_ctr_ + 2 * (7 * L_ + 2) + l;
        o.m_kvp = kvp_;
        o.m_head_dim = AD_;
        o.m_recv = d_recv_;
        o.m_chunk = xchunk_;
        o.m_slice = slice_;
        o.m_rank = r_;
        o.m_frag_o = d_frag_o_;
        o.m_frag_lse = d_frag_lse_;
        o.m_q_per_slot = q_per_slot_;
        o.m_dp = ADP_;
      }
      // the FFN's last GEMV writes the residual (local) or the TP partial (dist)
      float* ffn_out = dist ? d_parth_ : d_x_;
      float* ffn_ss = dist ? nullptr : d_ss_;
      if (F_ > 0) {
        GemvParams& gu = plan_gu_[l].p;
        gu.ypart = d_ypart_;
        gu.counters = d_counters_;
        gu.xf = d_xf_resid_;
        gu.ss_part = d_ss_;
        gu.n_ss = hblk;
        gu.xf_out = d_xf_m_;
        GemvParams& dn = plan_down_[l].p;
        dn.ypart = d_ypart_;
        dn.counters = d_counters_;
        dn.xf = d_xf_m_;
        dn.out = ffn_out;
        dn.out_stride = static_cast<int>(H_);
        dn.ss_out = ffn_ss;
        dn.xf_out = d_xf_resid_;
        dn.addend = moe_ ? d_moe_y_ : nullptr;  // shared expert + routed experts
      }
      if (moe_) {
        GemvParams& r = plan_router_[l].p;
        r.ypart = d_ypart_;
        r.counters = d_counters_;
        r.xf = d_xf_resid_;
        r.ss_part = d_ss_;
        r.n_ss = hblk;
        r.out = d_rlog_;
        GemvParams& gu = plan_egu_[l].p;
        gu.ypart = d_ypart_;
        gu.counters = d_counters_;
        gu.xf = d_xf_resid_;
        gu.ss_part = d_ss_;
        gu.n_ss = hblk;
        gu.xf_out = d_xf_em_;
        gu.group_count = d_gcount_;
        gu.group_ids = d_gids_;
        GemvParams& dn = plan_edown_[l].p;
        dn.ypart = d_ypart_;
        dn.counters = d_counters_;
        dn.xf = d_xf_em_;
        dn.group_count = d_gcount_;
        dn.group_ids = d_gids_;
        dn.route_w = d_route_w_;
        dn.out_stride = static_cast<int>(H_);
        if (F_ > 0) {
          dn.out = d_moe_y_;
        } else {
          dn.out = ffn_out;
          dn.ss_out = ffn_ss;
          dn.xf_out = d_xf_resid_;
        }
      }
    }
  }
  if (!attn_only_) {
    GemvParams& lm = plan_lm_.p;
    lm.ypart = d_ypart_;
    lm.counters = d_counters_;
    lm.xf = d_xf_resid_;
    lm.ss_part = d_ss_;
    lm.n_ss = hblk;
    lm.best = d_best_;
    lm.out = nullptr;
    lm.out_stride = V_local_;
  }
  weights_ready_ = true;
  drop_graphs();
}

void Engine::drop_graphs() {
  for (auto& g : graphs_cache_) cudaGraphExecDestroy(g.exec);
  graphs_cache_.clear();
}

void Engine::mark(int kind) {
  if (!prof_) return;
  cudaEvent_t ev;
  cuda_check(cudaEventCreate(&ev), "event");
  cuda_check(cudaEventRecord(ev, stream_), "event record");
  prof_->push_back({kind, ev});
}

void Engine::init_weights_hash(uint64_t seed) { build_weights_common(seed, true); }

void Engine::init_weights_mt19937(uint64_t seed) {
  if (mla_) throw std::invalid_argument("MLA weights come from the counter hash (the reference has no MLA draws)");
  build_weights_common(seed, false);
  const int64_t nq = Qh_ * D_, nk = Kh_ * D_;
  for (int64_t l = 0; l < L_; ++l) {
    // DecodeHarness ctor draw order: W_q, W_k, W_v (attention.hpp:438-442)
    std::mt19937_64 rng(seed + static_cast<uint64_t>(l));
    std::vector<double> wq(static_cast<size_t>(H_ * nq)), wk(static_cast<size_t>(H_ * nk)),
        wv(static_cast<size_t>(H_ * nk));
    for (double& v : wq) v = unit_draw(rng);
    for (double& v : wk) v = unit_draw(rng);
    for (double& v : wv) v = unit_draw(rng);
    upload_qkv_host(l, wq, wk, wv);
    if (f64_) {  // [H][q cols | k cols | v cols] in double, the reference's values exactly
      const size_t ncols = static_cast<size_t>(nq + 2 * nk);
      std::vector<double> w(static_cast<size_t>(H_) * ncols);
      for (int64_t k = 0; k < H_; ++k) {
        std::memcpy(&w[k * ncols], &wq[k * nq], nq * sizeof(double));
        std::memcpy(&w[k * ncols + nq], &wk[k * nk], nk * sizeof(double));
        std::memcpy(&w[k * ncols + nq + nk], &wv[k * nk], nk * sizeof(double));
      }
      cuda_check(cudaMemcpyAsync(w64_[l], w.data(), w.size() * sizeof(double), cudaMemcpyHostToDevice, stream_),
                 "f64 weights");
      cuda_check(cudaStreamSynchronize(stream_), "f64 weights sync");
    }
  }
}

void Engine::upload_qkv_host(int64_t layer, const std::vector<double>& wq, const std::vector<double>& wk,
                             const std::vector<double>& wv) {
  // wq [H x Q*Hsz], wk/wv [H x K*Hsz] row-major (reference orientation); this
  // device keeps all columns (local pool) or its TPA group's heads.
  const bool dist = dist_mode_ != HX_POOL_LOCAL;
  if (w8_ || w4_) throw std::invalid_argument("FP8 / FP4 weights are hash-initialised (hx_init_weights_hash)");
  const GemvPlan& g = plan_qkv_[layer];
  const int K = g.p.K, kst = K / 16;
  const int Qall = static_cast<int>(Qh_ * D_), Kall = static_cast<int>(Kh_ * D_);
  const int nq = g.p.nq, nk = g.p.nk;
  const int q0 = dist ? grp_ * nq : 0, k0 = dist ? grp_ * nk : 0;
  std::vector<uint16_t> img(static_cast<size_t>(g.p.Npad) * K, 0);
  auto woff = [&](int n, int k, int kst_) { return tc_ ? wtc_offset_host(n, k, kst_) : wfrag_offset_host(n, k, kst_); };
  for (int k = 0; k < K; ++k) {
    for (int n = 0; n < nq; ++n)
      img[woff(n, k, kst) / 2] = bf16_bits_from_double(wq[static_cast<size_t>(k) * Qall + q0 + n]);
    for (int n = 0; n < nk; ++n) {
      img[woff(nq + n, k, kst) / 2] =
          bf16_bits_from_double(wk[static_cast<size_t>(k) * Kall + k0 + n]);
      img[woff(nq + nk + n, k, kst) / 2] =
          bf16_bits_from_double(wv[static_cast<size_t>(k) * Kall + k0 + n]);
    }
  }
  // on the engine stream (a legacy-stream copy from pageable memory may still be
  // in flight when later kernels on the non-blocking engine stream run)
  cuda_check(cudaMemcpyAsync(w_qkv_[layer], img.data(), img.size() * 2, cudaMemcpyHostToDevice, stream_),
             "qkv upload");
  cuda_check(cudaStreamSynchronize(stream_), "qkv upload sync");
}

// ---------------------------------------------------------------------------
void Engine::check_layer(int64_t layer) const {
  if (layer < 0 || layer >= L_) throw std::invalid_argument("layer out of range");
}

void Engine::grow_random(int64_t layer, int64_t request, int64_t n, std::mt19937_64& rng) {
  check_layer(layer);
  if (mla_) throw std::invalid_argument("MLA caches are grown with the counter hash (fill_kv_hash)");
  if (request < 0 || request >= B_) throw std::invalid_argument("request out of range");
  const int64_t per = Kh_ * D_;
  const int64_t block = 4096;
  if (f64_) {  // the reference's doubles, unrounded
    std::vector<double> k, v;
    for (int64_t done = 0; done < n; done += block) {
      const int64_t m = std::min(block, n - done);
      k.resize(static_cast<size_t>(m * per));
      v.resize(static_cast<size_t>(m * per));
      for (int64_t i = 0; i < m; ++i) {  // attention.hpp:454-455 under g++: V drawn before K
        for (int64_t j = 0; j < per; ++j) v[static_cast<size_t>(i * per + j)] = unit_draw(rng);
        for (int64_t j = 0; j < per; ++j) k[static_cast<size_t>(i * per + j)] = unit_draw(rng);
      }
      append_kv_f64(layer, request, m, k.data(), v.data());
    }
    return;
  }
  std::vector<float> k, v;
  for (int64_t done = 0; done < n; done += block) {
    const int64_t m = std::min(block, n - done);
    k.resize(static_cast<size_t>(m * per));
    v.resize(static_cast<size_t>(m * per));
    for (int64_t i = 0; i < m; ++i) {
      // attention.hpp:454-455 under g++: V drawn before K (right-to-left args)
      std::vector<double> vv(static_cast<size_t>(per)), kk(static_cast<size_t>(per));
      for (double& x : vv) x = unit_draw(rng);
      for (double& x : kk) x = unit_draw(rng);
      if (kv4_) {  // e2m1 blocks of 32 dims per (token, head), rounded from the doubles; the stored
                   // values are exact floats, and append_kv's re-rounding keeps them (fp8.cuh)
        for (int64_t j0 = 0; j0 < per; j0 += 32)
          for (int w = 0; w < 2; ++w) {
            const double* src = (w ? kk : vv).data() + j0;
            float* dst = (w ? k : v).data() + i * per + j0;
            double am = 0.0;
            for (int j = 0; j < 32; ++j) am = std::max(am, std::fabs(src[j]));
            const int ex = e2m1_block_exp(am);
            for (int j = 0; j < 32; ++j) dst[j] = e2m1_to_float(e2m1_from_double(src[j], ex), ex);
          }
        continue;
      }
      for (int64_t j = 0; j < per; ++j) {
        // exact: route the double through its stored value (bf16, or e4m3 -- both exact in float)
        const double dv = vv[static_cast<size_t>(j)], dk = kk[static_cast<size_t>(j)];
        v[static_cast<size_t>(i * per + j)] =
            kv8_ ? e4m3_to_float(e4m3_from_double(dv)) : float_from_bf16_bits(bf16_bits_from_double(dv));
        k[static_cast<size_t>(i * per + j)] =
            kv8_ ? e4m3_to_float(e4m3_from_double(dk)) : float_from_bf16_bits(bf16_bits_from_double(dk));
      }
    }
    append_kv(layer, request, m, k.data(), v.data());
  }
}

void Engine::append_kv(int64_t layer, int64_t request, int64_t n, const float* k, const float* v) {
  check_layer(layer);
  if (f64_) {
    const size_t cnt = static_cast<size_t>(std::max<int64_t>(n, 0) * Kh_ * D_);
    std::vector<double> kd(k, k + cnt), vd(v, v + cnt);
    append_kv_f64(layer, request, n, kd.data(), vd.data());
    return;
  }
  if (mla_) throw std::invalid_argument("append_kv takes GQA K/V rows; MLA caches hold latents");
  if (request < 0 || request >= B_) throw std::invalid_argument("request out of range");
  if (n < 0) throw std::invalid_argument("token count must be >= 0");
  if (h_total_[static_cast<size_t>(layer * B_ + request)] + n > cap_)
    throw std::invalid_argument("KV capacity exceeded");
  if (n == 0) return;
  const size_t cnt = static_cast<size_t>(n * Kh_ * D_);
  if (kv4_) {  // host e2m1 block rounding (fp8.cuh) of each 32-dim block of a token's row
    const size_t nblk = cnt / 32;
    std::vector<uint8_t> ck(cnt), cv(cnt);
    std::vector<int8_t> ek(nblk), ev(nblk);
    for (size_t blk = 0; blk < nblk; ++blk)
      for (int w = 0; w < 2; ++w) {
        const float* src = (w ? v : k) + blk * 32;
        double am = 0.0;
        for (int j = 0; j < 32; ++j) am = std::max(am, std::fabs(static_cast<double>(src[j])));
        const int ex = e2m1_block_exp(am);
        (w ? ev : ek)[blk] = static_cast<int8_t>(ex);
        for (int j = 0; j < 32; ++j) (w ? cv : ck)[blk * 32 + j] = e2m1_from_double(src[j], ex);
      }
    uint8_t* dbuf = nullptr;
    cuda_check(cudaMalloc(&dbuf, 2 * cnt + 2 * nblk), "append staging");
    cuda_check(cudaMemcpyAsync(dbuf, ck.data(), cnt, cudaMemcpyHostToDevice, stream_), "append h2d");
    cuda_check(cudaMemcpyAsync(dbuf + cnt, cv.data(), cnt, cudaMemcpyHostToDevice, stream_), "append h2d");
    cuda_check(cudaMemcpyAsync(dbuf + 2 * cnt, ek.data(), nblk, cudaMemcpyHostToDevice, stream_), "append h2d");
    cuda_check(cudaMemcpyAsync(dbuf + 2 * cnt + nblk, ev.data(), nblk, cudaMemcpyHostToDevice, stream_), "append h2d");
    cuda_check(launch_kv4_append_rows(kv_[layer], dbuf, dbuf + cnt, reinterpret_cast<int8_t*>(dbuf + 2 * cnt),
                                      reinterpret_cast<int8_t*>(dbuf + 2 * cnt + nblk), static_cast<int>(n),
                                      static_cast<int>(request), d_total_ + layer * B_, B_, static_cast<int>(Kh_),
                                      kvh_per_slot_, kvp_, chunk_, static_cast<int>(D_), DP_, page_cap_, slot_base_,
                                      n_slots_, stream_),
               "fp4 append kernel");
    cuda_check(cudaStreamSynchronize(stream_), "append sync");
    cudaFree(dbuf);
    h_total_[static_cast<size_t>(layer * B_ + request)] += n;
    return;
  }
  const size_t esz = kv8_ ? 1 : 2;  // stored element bytes
  std::vector<uint8_t> kb(cnt * esz), vb(cnt * esz);
  for (size_t i = 0; i < cnt; ++i) {
    if (kv8_) {  // e4m3 RNE of the float value (fp8.cuh)
      kb[i] = e4m3_from_double(static_cast<double>(k[i]));
      vb[i] = e4m3_from_double(static_cast<double>(v[i]));
    } else {
      const uint16_t kh = bf16_bits_from_float(k[i]), vh = bf16_bits_from_float(v[i]);
      std::memcpy(&kb[2 * i], &kh, 2);
      std::memcpy(&vb[2 * i], &vh, 2);
    }
  }
  uint8_t *dk = nullptr, *dv = nullptr;
  cuda_check(cudaMalloc(&dk, cnt * esz), "append staging");
  cuda_check(cudaMalloc(&dv, cnt * esz), "append staging");
  cuda_check(cudaMemcpyAsync(dk, kb.data(), cnt * esz, cudaMemcpyHostToDevice, stream_), "append h2d");
  cuda_check(cudaMemcpyAsync(dv, vb.data(), cnt * esz, cudaMemcpyHostToDevice, stream_), "append h2d");
  cuda_check(launch_kv_append_rows(kv_[layer], dk, dv, static_cast<int>(n), static_cast<int>(request),
                                   d_total_ + layer * B_, B_, static_cast<int>(Kh_), kvh_per_slot_, kvp_,
                                   chunk_, static_cast<int>(D_), DP_, page_cap_, slot_base_, n_slots_, kv8_fmt(),
                                   stream_),
             "append kernel");
  cuda_check(cudaStreamSynchronize(stream_), "append sync");
  cudaFree(dk);
  cudaFree(dv);
  h_total_[static_cast<size_t>(layer * B_ + request)] += n;
}

void Engine::fill_kv_hash(int64_t n, uint64_t seed) {
  if (f64_) throw std::invalid_argument("the exact fp64 harness grows with grow_random / append");
  for (int64_t l = 0; l < L_; ++l)
    for (int b = 0; b < B_; ++b)
      if (h_total_[static_cast<size_t>(l * B_ + b)] + n > cap_) throw std::invalid_argument("KV capacity exceeded");
  for (int64_t l = 0; l < L_ && mla_; ++l) {
    cuda_check(launch_kv_fill_hash_mla(kv_[l], d_total_ + l * B_, B_, kvp_, chunk_, page_cap_, slot_base_, n_slots_,
                                       n, seed, hash_stream(kCacheK, l), stream_, kv8_),
               "kv fill");
    for (int b = 0; b < B_; ++b) h_total_[static_cast<size_t>(l * B_ + b)] += n;
  }
  for (int64_t l = 0; l < L_ && !mla_ && kv4_; ++l) {
    cuda_check(launch_kv4_fill_hash(kv_[l], d_total_ + l * B_, B_, static_cast<int>(Kh_), kvh_per_slot_, kvp_,
                                    chunk_, static_cast<int>(D_), DP_, page_cap_, slot_base_, n_slots_, n, seed,
                                    hash_stream(kCacheK, l), hash_stream(kCacheV, l), stream_),
               "kv fill");
    for (int b = 0; b < B_; ++b) h_total_[static_cast<size_t>(l * B_ + b)] += n;
  }
  for (int64_t l = 0; l < L_ && !mla_ && !kv4_; ++l) {
    cuda_check(launch_kv_fill_hash(kv_[l], d_total_ + l * B_, B_, static_cast<int>(Kh_), kvh_per_slot_, kvp_,
                                   chunk_, static_cast<int>(D_), DP_, page_cap_, slot_base_, n_slots_, n, seed,
                                   hash_stream(kCacheK, l), hash_stream(kCacheV, l), kv8_fmt(), stream_),
               "kv fill");
    for (int b = 0; b < B_; ++b) h_total_[static_cast<size_t>(l * B_ + b)] += n;
  }
  cuda_check(cudaStreamSynchronize(stream_), "kv fill sync");
}

int64_t Engine::total_tokens(int64_t layer, int64_t request) const {
  check_layer(layer);
  if (request < 0 || request >= B_) throw std::invalid_argument("request out of range");
  return h_total_[static_cast<size_t>(layer * B_ + request)];
}

int64_t Engine::effective_tokens(int64_t layer, int64_t request, int64_t rank) const {
  if (rank < 0 || rank >= kvp_) throw std::invalid_argument("rank out of range");
  return rr_count(total_tokens(layer, request), static_cast<int>(rank), chunk_, kvp_);
}

int64_t Engine::max_min_gap(int64_t layer, int64_t request) const {
  int64_t lo = INT64_MAX, hi = 0;
  for (int r = 0; r < kvp_; ++r) {
    const int64_t c = effective_tokens(layer, request, r);
    lo = std::min(lo, c);
    hi = std::max(hi, c);
  }
  return hi - lo;
}

int Engine::slot_local_of(int rank, int group) const { return group * kvp_ + rank - slot_base_; }

void Engine::read_kv(int64_t layer, int64_t request, int64_t rank, int64_t head, float* k, float* v) {
  check_layer(layer);
  if (mla_) {  // latent rows: k = [n x W], v = [n x DV] (the value part of the same rows)
    if (head != 0) throw std::invalid_argument("kv head out of range");
    const int64_t n = effective_tokens(layer, request, rank);
    const int sl = slot_local_of(static_cast<int>(rank), 0);
    if (sl < 0 || sl >= n_slots_) throw std::invalid_argument("rank not resident on this device");
    const int pages = static_cast<int>((n + kMlaPageRows - 1) / kMlaPageRows);
    std::vector<uint8_t> buf(static_cast<size_t>(pages) * page_bytes_);
    const size_t base = (static_cast<size_t>(sl) * B_ + request) * page_cap_ * page_bytes_;
    cuda_check(cudaStreamSynchronize(stream_), "read_kv sync");
    if (pages)
      cuda_check(cudaMemcpy(buf.data(), kv_[layer] + base, buf.size(), cudaMemcpyDeviceToHost), "read_kv");
    for (int64_t t = 0; t < n; ++t) {
      const uint8_t* page = buf.data() + static_cast<size_t>(t / kMlaPageRows) * page_bytes_;
      for (int d = 0; d < W_; ++d) {
        float x;
        if (kv8_) {
          x = e4m3_to_float(page[mla_kv_offset8(static_cast<int>(t % kMlaPageRows), d)]);
        } else {
          uint16_t kb;
          std::memcpy(&kb, page + mla_kv_offset(static_cast<int>(t % kMlaPageRows), d), 2);
          x = float_from_bf16_bits(kb);
        }
        k[t * W_ + d] = x;
        if (d < DV_) v[t * DV_ + d] = x;
      }
    }
    return;
  }
  if (f64_) {
    const int64_t n = effective_tokens(layer, request, rank);
    std::vector<double> kd(static_cast<size_t>(n * D_)), vd(static_cast<size_t>(n * D_));
    read_kv_f64(layer, request, rank, head, kd.data(), vd.data());
    for (size_t i = 0; i < kd.size(); ++i) {
      k[i] = static_cast<float>(kd[i]);
      v[i] = static_cast<float>(vd[i]);
    }
    return;
  }
  if (head < 0 || head >= Kh_) throw std::invalid_argument("kv head out of range");
  const int64_t n = effective_tokens(layer, request, rank);
  const int grp = static_cast<int>(head / kvh_per_slot_), kvh = static_cast<int>(head % kvh_per_slot_);
  const int sl = slot_local_of(static_cast<int>(rank), grp);
  if (sl < 0 || sl >= n_slots_) throw std::invalid_argument("rank not resident on this device");
  const int pages = static_cast<int>((n + 15) / 16);
  std::vector<uint8_t> buf(static_cast<size_t>(pages) * page_bytes_);
  const size_t base = ((static_cast<size_t>(sl) * B_ + request) * kvh_per_slot_ + kvh) * page_cap_ * page_bytes_;
  cuda_check(cudaStreamSynchronize(stream_), "read_kv sync");
  if (pages)
    cuda_check(cudaMemcpy(buf.data(), kv_[layer] + base, buf.size(), cudaMemcpyDeviceToHost), "read_kv");
  for (int64_t t = 0; t < n && kv4_; ++t) {
    const uint8_t* page = buf.data() + static_cast<size_t>(t / 16) * page_bytes_;
    for (int d = 0; d < D_; ++d)
      for (int w = 0; w < 2; ++w) {
        bool high = false;
        const uint32_t off = kv4_offset(DP_, static_cast<int>(t % 16), d, w != 0, &high);
        const uint8_t code = static_cast<uint8_t>((page[off] >> (high ? 4 : 0)) & 15);
        const int ex = kv4_scale_exp(page[kv4_scale_offset(DP_, static_cast<int>(t % 16), d, w != 0)], w != 0);
        (w ? v : k)[t * D_ + d] = e2m1_to_float(code, ex);
      }
  }
  for (int64_t t = 0; t < n && !kv4_; ++t) {
    const uint8_t* page = buf.data() + static_cast<size_t>(t / 16) * page_bytes_;
    for (int d = 0; d < D_; ++d) {
      const uint8_t* pk = page + kv_offset(DP_, static_cast<int>(t % 16), d, false, kv8_fmt());
      const uint8_t* pv = page + kv_offset(DP_, static_cast<int>(t % 16), d, true, kv8_fmt());
      if (kv8_) {
        k[t * D_ + d] = e4m3_to_float(*pk);
        v[t * D_ + d] = e4m3_to_float(*pv);
      } else {
        uint16_t kb, vb;
        std::memcpy(&kb, pk, 2);
        std::memcpy(&vb, pv, 2);
        k[t * D_ + d] = float_from_bf16_bits(kb);
        v[t * D_ + d] = float_from_bf16_bits(vb);
      }
    }
  }
}

// ---------------------------------------------------------------------------
void Engine::require_context(int64_t layer) const {
  for (int b = 0; b < B_; ++b)
    if (h_total_[static_cast<size_t>(layer * B_ + b)] == 0)
      throw std::invalid_argument("decode needs a nonempty context");
  for (int b = 0; b < B_; ++b)
    if (h_total_[static_cast<size_t>(layer * B_ + b)] + 1 > cap_) throw std::invalid_argument("KV capacity exceeded");
}

void Engine::record_transcript(int64_t layers) {
  // attention.hpp:466-468 (broadcast) and :492-502 (all-to-all), per request.
  const int64_t pool = static_cast<int64_t>(tpa_) * kvp_;
  const int64_t group_width = static_cast<int64_t>(q_per_slot_) * D_;
  const int64_t slice = group_width / kvp_;
  // bounded for long serving runs: the first kMaxTranscript records are kept
  // (hx_clear_transcript starts a new window)
  constexpr size_t kMaxTranscript = size_t{1} << 20;
  const size_t per_step = static_cast<size_t>(layers) * B_ * (pool - 1 + (mla_ ? 0 : tpa_ * kvp_ * (kvp_ - 1)));
  if (transcript_.size() + per_step > kMaxTranscript) return;
  for (int64_t l = 0; l < layers; ++l)
    for (int b = 0; b < B_; ++b) {
      for (int64_t r = 1; r < pool; ++r) transcript_.push_back({0, 0, r, H_, 0});
      if (mla_) continue;  // the message records are DecodeHarness (GQA) semantics
      for (int g = 0; g < tpa_; ++g)
        for (int r = 0; r < kvp_; ++r)
          for (int p = 0; p < kvp_; ++p) {
            if (p == r) continue;
            const int64_t first = p * slice / D_, last = ((p + 1) * slice - 1) / D_;
            transcript_.push_back({1, static_cast<int64_t>(g) * kvp_ + r, static_cast<int64_t>(g) * kvp_ + p,
                                   slice, last - first + 1});
          }
    }
}

AttnParams Engine::attn_params(int64_t layer, int b_begin, int b_count) {
  attn_layer_ = layer;
  AttnParams a{};
  a.kv = kv_[layer];
  a.q = d_q_;
  a.total = d_total_ + layer * B_;
  a.part_o = d_part_o_;
  a.part_lse2 = d_part_lse_;
  a.work_counter = d_work_;
  a.done_counter = d_work_ + 1;
  a.dp = DP_;
  a.batch = B_;
  a.q_heads = dist_mode_ == HX_POOL_LOCAL ? static_cast<int>(Qh_) : q_per_slot_;
  a.q_grp_base = dist_mode_ == HX_POOL_LOCAL ? 0 : grp_;
  a.group = G_;
  a.q_chunks = q_chunks_;
  a.qrows = q_rows_;
  a.kv8 = kv8_ ? 1 : 0;
  a.kv4 = kv4_ ? 1 : 0;
  if (one_src_merge_) {
    a.xf_out = d_xf_attn_;
    a.xf16 = xf16_();
    a.hd = static_cast<int>(D_);
  }
  a.kvh_per_slot = kvh_per_slot_;
  a.q_per_slot = q_per_slot_;
  a.kvp = kvp_;
  a.chunk = chunk_;
  a.page_cap = page_cap_;
  a.slot_base = slot_base_;
  a.n_local_slots = n_slots_;
  a.b_begin = b_begin;
  a.stream_batch = b_count;
  a.n_streams = n_slots_ * b_count * kvh_per_slot_ * q_chunks_;
  a.splits = live_splits(layer, b_count != B_);
  a.n_items = a.n_streams * a.splits;  // HOP-B (one request): splits_req_ balanced page ranges
  a.qscale = static_cast<float>(1.4426950408889634 / std::sqrt(static_cast<double>(mla_ ? W_ : D_)));
  a.stream_major = std::getenv("HX_STREAM_MAJOR") && std::getenv("HX_STREAM_MAJOR")[0] == '1';  // A/B
  a.hd = static_cast<int>(D_);
  a.pushed = d_pushed_;
  if (fused_ && hopb_ && device_exchange()) {
    // HOP-B: request-ordered work, each stream reduced (and pushed) as it
    // completes, overlapping the attention of the streams after it -- by the
    // co-resident stream reducer (2, the attention CTAs never pause their KV
    // stream) or, with HX_HOPB_INKERNEL=1, by the attention CTA that finished
    // the stream's last split (1)
    a.fused = hopb_inkernel_ ? 1 : (std::getenv("HX_HOPB_DEBUG_NOCOUNT") ? 3 : 2);
    // work in groups of hopb_group_ requests (split-major inside a group): the
    // groups' exchanges overlap the attention of the groups after them, while
    // each group keeps the batched launch's split-major KV order
    a.stream_major = hopb_inkernel_ ? 1 : std::max(1, a.n_streams / b_count * hopb_group_);
    a.stream_done = d_stream_done_;
    a.frag_o = d_frag_o_;
    a.frag_lse = d_frag_lse_;
    a.pushed = d_pushed_;
    a.hd = static_cast<int>(D_);
  }
  if (local_stream_reduce_ && dist_mode_ == HX_POOL_LOCAL && !mla_ && !(attn_tc_ && attn_tc_supported(a))) {
    // local pools: the same co-resident stream reducer replaces the split-reduce
    // kernel -- streams are merged while the attention of later streams runs,
    // instead of one reduce launch after the whole attention kernel
    a.fused = 2;
    a.stream_major = std::max(1, a.n_streams / b_count * hopb_group_);
    a.stream_done = d_stream_done_;
    a.frag_o = d_frag_o_;
    a.frag_lse = d_frag_lse_;
  }
  if (mla_) {
    a.qimg = d_qimg_;
    a.dp = DV_;
  }
  return a;
}

// 2-3: flash-decode partials over every local rank's shard (attend BEFORE
// append), then per-rank fragments (split merge); the token totals are bumped
// by the merge kernel, after which the appended token counts.
void Engine::launch_attention_kernels(const AttnParams& a) {
  if (mla_) {
    cuda_check(launch_mla_decode(a, std::min(attn_grid_, a.n_items), stream_, mla_tm_[attn_layer_].s,
                                 mla_tm_[attn_layer_].v),
               "mla attention");
    mark(2);
    cuda_check(launch_mla_split_reduce(a, d_frag_o_, d_frag_lse_, stream_), "mla split reduce");
  } else {
    if (kv8tc_ && !attn_tc_supported(a))  // tensor-core FP8 pages: only the tcgen05 kernel reads them
      throw std::runtime_error("attention: FP8 tensor-core pages need the tcgen05 kernel (unsupported launch)");
    if (attn_tc_ && attn_tc_supported(a))
      cuda_check(launch_attn_tc(a, std::min(attn_grid_, (a.n_items + 1) / 2), stream_), "attention (tcgen05)");
    else
      cuda_check(launch_attn_decode(a, std::min(attn_grid_, a.n_items), stream_), "attention");
    mark(2);
    if (!a.fused) cuda_check(launch_attn_split_reduce(a, d_frag_o_, d_frag_lse_, stream_), "split reduce");
    if (a.fused >= 2) cuda_check(launch_attn_stream_reduce(a, stream_), "hop-b stream reduce");
  }
}

void Engine::enqueue_attention(int64_t layer) {
  // 1. QKV projection (input fragments already in d_xf_resid_) with fused
  //    round-robin append of this token's K/V
  const GemvPlan& q = plan_qkv_[layer];
  cuda_check(launch_gemv(q.p, q.xmode, E_QKV, num_sms_, stream_), "qkv gemv");
  if (mla_)  // W_UK absorption: q heads -> the 576-wide latent query image
    cuda_check(launch_mla_absorb_q(d_q_, w_uk_[layer], B_, static_cast<int>(Qh_), static_cast<int>(D_), DP_,
                                   d_qimg_, stream_, kv8_),
               "mla absorb q");
  mark(1);
  if (dist_mode_ != HX_POOL_LOCAL) {
    enqueue_exchange_and_attention_dist(layer);
    return;
  }
  // 2. flash-decode partials over every local rank's shard (attend BEFORE append)
  const AttnParams a = attn_params(layer, 0, B_);
  launch_attention_kernels(a);
  mark(3);
}

// One rank of the pool: attention over its own KV shard, pack the fragment
// into per-peer slices, all-to-all inside the KVP group (attention.hpp:492-502).
// HOP-B (overlap.hpp:37-69): request b's exchange runs on the comm stream while
// request b+1's attention runs on the compute stream.
void Engine::enqueue_exchange_and_attention_dist(int64_t layer) {
  if (device_exchange()) {
    // Device-initiated exchange: the split reduce stores each rank's slices
    // straight into the peers' receive buffers (NVLink P2P / CUDA IPC) and the
    // last CTA raises this rank's flag in every peer -- no pack kernel, no
    // collective. HOP-B on (overlap.hpp:37-69, at stream granularity): ONE
    // request-ordered attention launch whose CTAs reduce and push each stream
    // as it completes, while the later requests are still streaming.
    AttnParams a = attn_params(layer, 0, B_);
    const bool skip = skip_comm_ & 1;  // measurement: every slice stays on this rank
    a.push = 1;
    a.peer_recv = skip ? d_self_recv_ : d_peer_recv_;
    a.peer_flag = skip ? d_self_flag_ : d_peer_flag_;
    a.xchunk = xchunk_;
    a.xslice = slice_;
    a.xrank = r_;
    launch_attention_kernels(a);
    mark(3);
    if (loopback_ && !skip) {
      // in-process pool: every rank's pushes land before any rank's flag wait
      // runs. A kernel spinning on a flag that another thread's not-yet-launched
      // kernel raises can deadlock one shared context (lazy module loading
      // synchronises it); across processes (NCCL pools) the wait spins on the device.
      cuda_check(cudaStreamSynchronize(stream_), "loopback exchange sync");
      transport_->host_barrier();
    }
    cuda_check(launch_wait_flags(skip ? d_flags_ + r_ : d_flags_, skip ? 1 : kvp_, stream_), "exchange wait");
    mark(9);
    return;
  }
  const size_t stride = static_cast<size_t>(B_) * xchunk_;
  const int rounds = hopb_ ? B_ : 1;
  const int per = hopb_ ? 1 : B_;
  // HOP-B: each request's exchange (or its measurement stand-in, the local copy)
  // runs on the comm stream behind an event; the loopback transport
  // synchronises on the host, so it stays on the compute stream
  const bool side_stream = hopb_ && (dist_mode_ == HX_POOL_NCCL || (skip_comm_ & 1));
  for (int i = 0; i < rounds; ++i) {
    const int b0 = i * per;
    const AttnParams a = attn_params(layer, b0, per);
    launch_attention_kernels(a);
    cuda_check(launch_pack_exchange(d_frag_o_, d_frag_lse_, b0, per, B_, q_per_slot_, AD_, ADP_,
                                    kvp_, slice_, xchunk_, d_send_, stream_),
               "pack");
    mark(3);
    float* send = d_send_ + static_cast<size_t>(b0) * xchunk_;
    float* recv = d_recv_ + static_cast<size_t>(b0) * xchunk_;
    const size_t count = static_cast<size_t>(per) * xchunk_;
    cudaStream_t cs = stream_;
    if (side_stream) {
      cuda_check(cudaEventRecord(hop_events_[static_cast<size_t>(i)], stream_), "hopb event");
      cuda_check(cudaStreamWaitEvent(comm_stream_, hop_events_[static_cast<size_t>(i)], 0), "hopb wait");
      cs = comm_stream_;
    }
    if (skip_comm_ & 1) {  // measurement: keep only this rank's own block, no wire traffic
      cuda_check(cudaMemcpyAsync(recv + static_cast<size_t>(r_) * stride, send + static_cast<size_t>(r_) * stride,
                                 count * sizeof(float), cudaMemcpyDeviceToDevice, cs),
                 "skip-comm copy");
    } else {
      transport_->all_to_all(send, recv, count, stride, cs);
    }
  }
  if (side_stream) {
    cuda_check(cudaEventRecord(hop_events_.back(), comm_stream_), "hopb join");
    cuda_check(cudaStreamWaitEvent(stream_, hop_events_.back(), 0), "hopb join wait");
  }
  mark(9);
}

// Map the KVP group's receive buffers and flags (device-initiated exchange):
// once, collectively, before the first distributed step (outside capture).
void Engine::ensure_peers() {
  if (peers_mapped_ || dist_mode_ == HX_POOL_LOCAL) return;
  std::vector<void*> recv, flags;
  try {
    transport_->map_peers(d_recv_, d_flags_, recv, flags);
  } catch (const std::exception& ex) {
    // no peer mapping on this system (e.g. CUDA IPC unavailable): exchange through the collective
    std::fprintf(stderr, "helix-b200: device exchange unavailable (%s); using the collective all-to-all\n",
                 ex.what());
    nccl_a2a_ = true;
    return;
  }
  std::vector<float*> pr(static_cast<size_t>(kvp_));
  std::vector<unsigned*> pf(static_cast<size_t>(kvp_));
  for (int p = 0; p < kvp_; ++p) {
    pr[static_cast<size_t>(p)] = static_cast<float*>(recv[static_cast<size_t>(p)]);
    pf[static_cast<size_t>(p)] = static_cast<unsigned*>(flags[static_cast<size_t>(p)]) + r_;  // my word in peer p
  }
  cuda_check(cudaMemcpyAsync(d_peer_recv_, pr.data(), pr.size() * sizeof(float*), cudaMemcpyHostToDevice, stream_),
             "peer table");
  cuda_check(cudaMemcpyAsync(d_peer_flag_, pf.data(), pf.size() * sizeof(unsigned*), cudaMemcpyHostToDevice, stream_),
             "peer table");
  cuda_check(cudaStreamSynchronize(stream_), "peer table");
  // in-process pools: nobody launches a flag wait before every rank is past its uploads
  transport_->host_barrier();
  peers_mapped_ = true;
}

void Engine::harness_step(int64_t layer, const float* x_host, int64_t x_len, float* out, float* lse) {
  check_layer(layer);
  if (f64_) {
    std::vector<double> xd(x_host, x_host + std::max<int64_t>(x_len, 0));
    std::vector<double> od(static_cast<size_t>(B_ * Qh_ * D_)), ld(static_cast<size_t>(B_ * Qh_));
    harness_step_f64(layer, xd.data(), x_len, od.data(), ld.data());
    for (size_t i = 0; i < od.size(); ++i) out[i] = static_cast<float>(od[i]);
    if (lse)
      for (size_t i = 0; i < ld.size(); ++i) lse[i] = static_cast<float>(ld[i]);
    return;
  }
  if (x_len != static_cast<int64_t>(B_) * H_) throw std::invalid_argument("hidden state has wrong width");
  if (!weights_ready_) throw StateError("weights are not initialised");
  require_context(layer);
  cuda_check(cudaMemcpyAsync(d_x_, x_host, static_cast<size_t>(x_len) * 4, cudaMemcpyHostToDevice, stream_),
             "x h2d");
  harness_step_device(layer, d_x_, d_out_);
  if (lse)
    cuda_check(cudaMemcpyAsync(lse, d_out_lse_, static_cast<size_t>(B_) * Qh_ * 4, cudaMemcpyDeviceToHost, stream_),
               "lse d2h");
  cuda_check(cudaMemcpyAsync(out, d_out_, static_cast<size_t>(B_) * Qh_ * D_ * 4, cudaMemcpyDeviceToHost, stream_),
             "out d2h");
  cuda_check(cudaStreamSynchronize(stream_), "harness sync");
}

void Engine::harness_step_device(int64_t layer, const float* x_dev, float* out_dev) {
  check_layer(layer);
  if (f64_) throw StateError("the exact fp64 harness takes host doubles (hx_harness_step_f64)");
  if (mla_) throw StateError("the attention-only harness is DecodeHarness (GQA); MLA runs through decode_step");
  if (dist_mode_ != HX_POOL_LOCAL)
    throw StateError("the attention-only harness runs on a local pool; distributed pools use decode_step");
  if (!weights_ready_) throw StateError("weights are not initialised");
  require_context(layer);
  cuda_check(launch_xprep_plain(x_dev, B_, static_cast<int>(H_), static_cast<int>(H_), d_xf_resid_, stream_,
                                xf16_()),
             "xprep");
  enqueue_attention(layer);
  cuda_check(launch_merge_out(d_frag_o_, d_frag_lse_, B_, static_cast<int>(Qh_), q_per_slot_, kvp_,
                              static_cast<int>(D_), DP_, out_dev, d_out_lse_, d_total_ + layer * B_, stream_),
             "merge");
  mark(8);
  for (int b = 0; b < B_; ++b) h_total_[static_cast<size_t>(layer * B_ + b)] += 1;
  record_transcript(1);
}

void Engine::enqueue_decode(const int32_t* tokens_dev, int32_t* next_dev) {
  cuda_check(launch_embed(emb_, tokens_dev, B_, static_cast<int>(H_), d_x_, d_ss_, d_xf_resid_, stream_, xf16_()),
             "embed");
  mark(0);
  if (capture_hidden_)
    cuda_check(cudaMemcpyAsync(d_hidden_, d_x_, static_cast<size_t>(B_) * H_ * 4, cudaMemcpyDeviceToDevice, stream_),
               "hidden");
  const bool dist = dist_mode_ != HX_POOL_LOCAL;
  for (int64_t l = 0; l < L_; ++l) {
    enqueue_attention(l);
    if (!dist) {
      // LSE-rescale combine of the KVP fragments -> O-proj activations (attention.hpp:118-175)
      // (a fused split+KVP merge kernel measured 0.2 ms/step slower than this pair)
      if (!one_src_merge_ && !fused_combine_)
        cuda_check(launch_xprep_merge_local(d_frag_o_, d_frag_lse_, B_, q_per_slot_, kvp_, AD_, ADP_,
                                            static_cast<int>(Qh_) * AD_, d_xf_attn_, d_total_ + l * B_, stream_,
                                            mla_ ? d_att_ : nullptr, xf16_()),
                   "merge");
      if (mla_)
        cuda_check(launch_mla_uv(d_att_, w_uv_[l], B_, uv_heads_, static_cast<int>(D_), d_xf_attn_, stream_, xf16_()),
                   "mla uv");
      cuda_check(launch_gemv(plan_o_[l].p, 0, E_RESID, num_sms_, stream_), "o-proj");
      mark(4);
      enqueue_ffn(l);
    } else {
      // merge of the exchanged slices, then TP O-proj over this rank's slice and
      // AllReduce over the pool (latency.cpp:85-94)
      if (!fused_combine_)
        cuda_check(launch_xprep_merge_recv(d_recv_, B_, kvp_, xchunk_, slice_, r_, AD_, d_xf_attn_,
                                           d_total_ + l * B_, stream_, mla_ ? d_att_ : nullptr, xf16_()),
                   "merge");
      if (mla_)
        cuda_check(launch_mla_uv(d_att_, w_uv_[l], B_, uv_heads_, static_cast<int>(D_), d_xf_attn_, stream_, xf16_()),
                   "mla uv");
      cuda_check(launch_gemv(plan_o_[l].p, 0, E_STORE, num_sms_, stream_), "o-proj");
      mark(4);
      if (!(skip_comm_ & 2)) transport_->all_reduce_sum(d_parth_, static_cast<size_t>(B_) * H_, stream_);
      cuda_check(launch_residual_add(d_x_, d_parth_, B_, static_cast<int>(H_), d_ss_, d_xf_resid_, stream_,
                                     xf16_()),
                 "residual");
      mark(9);
      // TP FFN over F/N features (or EP x TPF experts), AllReduce (latency.cpp:110-144)
      enqueue_ffn(l);
      if (!(skip_comm_ & 2)) transport_->all_reduce_sum(d_parth_, static_cast<size_t>(B_) * H_, stream_);
      cuda_check(launch_residual_add(d_x_, d_parth_, B_, static_cast<int>(H_), d_ss_, d_xf_resid_, stream_,
                                     xf16_()),
                 "residual");
      mark(9);
    }
    if (capture_hidden_)
      cuda_check(cudaMemcpyAsync(d_hidden_ + (l + 1) * B_ * H_, d_x_, static_cast<size_t>(B_) * H_ * 4,
                                 cudaMemcpyDeviceToDevice, stream_),
                 "hidden");
  }
  GemvParams lm = plan_lm_.p;
  lm.out = store_logits_ ? d_logits_ : nullptr;
  cuda_check(launch_gemv(lm, 1, E_LOGITS, num_sms_, stream_), "lm head");
  if (dist && !(skip_comm_ & 2)) transport_->all_reduce_max_u64(d_best_, static_cast<size_t>(B_), stream_);  // vocab-sharded argmax
  cuda_check(launch_argmax_finish(d_best_, B_, next_dev, d_best_, stream_), "argmax");
  mark(7);
}

// FFN of one layer: input = rmsnorm(x) via d_xf_resid_ + d_ss_; output into the
// residual (local pool) or the TP partial d_parth_ (distributed pool).
//   dense: gate/up (SwiGLU epilogue) -> down
//   MoE (latency.cpp:110-137): router GEMV -> top-k routing kernel -> grouped
//   expert gate/up over the active experts only -> grouped expert down whose
//   epilogue combines the experts with the routing weights in ascending expert
//   order -> [shared expert gate/up -> down, adding the routed output]
void Engine::enqueue_ffn(int64_t l) {
  const bool dist = dist_mode_ != HX_POOL_LOCAL;
  const int em_last = dist ? E_STORE : E_RESID;
  if (moe_) {
    cuda_check(launch_gemv(plan_router_[l].p, 1, E_STORE, num_sms_, stream_), "router");
    cuda_check(launch_moe_route(d_rlog_, B_, static_cast<int>(E_), static_cast<int>(topk_), e_begin_,
                                e_begin_ + E_local_, d_route_w_, d_gids_, d_gcount_, stream_),
               "route");
    cuda_check(launch_gemv(plan_egu_[l].p, 1, E_SWIGLU, num_sms_, stream_), "expert gate/up");
    mark(5);
    const bool shared = F_ > 0;
    cuda_check(launch_gemv(plan_edown_[l].p, 0, shared ? E_STORE : em_last, num_sms_, stream_), "expert down");
    if (shared) {
      cuda_check(launch_gemv(plan_gu_[l].p, 1, E_SWIGLU, num_sms_, stream_), "shared gate/up");
      cuda_check(launch_gemv(plan_down_[l].p, 0, em_last, num_sms_, stream_), "shared down");
    }
    mark(6);
    return;
  }
  cuda_check(launch_gemv(plan_gu_[l].p, 1, E_SWIGLU, num_sms_, stream_), "gate/up");
  mark(5);
  cuda_check(launch_gemv(plan_down_[l].p, 0, em_last, num_sms_, stream_), "down");
  mark(6);
}

void Engine::decode_step_device(const int32_t* tokens_dev, int32_t* next_dev) {
  if (attn_only_) throw StateError("decode_step needs a full model (attention_only = 0)");
  if (!weights_ready_) throw StateError("weights are not initialised");
  for (int64_t l = 0; l < L_; ++l) require_context(l);
  if (device_exchange() && !(skip_comm_ & 1)) ensure_peers();  // skip: the self tables (alloc) suffice
  if (graphs_ && !(loopback_ && skip_comm_ != 3) && !prof_) {
    cudaGraphExec_t exec = nullptr;
    // the attention plan is baked into the graph: key it by every layer's live splits
    std::vector<int> plan(static_cast<size_t>(L_));
    for (int64_t l = 0; l < L_; ++l) plan[static_cast<size_t>(l)] = live_splits(l, false);
    for (auto& g : graphs_cache_)
      if (g.tokens == tokens_dev && g.next == next_dev && g.hidden == capture_hidden_ && g.logits == store_logits_ &&
          g.plan == plan)
        exec = g.exec;
    if (!exec) {
      cudaGraph_t g;
      cuda_check(cudaStreamBeginCapture(stream_, cudaStreamCaptureModeThreadLocal), "capture begin");
      enqueue_decode(tokens_dev, next_dev);
      cuda_check(cudaStreamEndCapture(stream_, &g), "capture end");
      cuda_check(cudaGraphInstantiate(&exec, g, 0), "graph instantiate");
      cuda_check(cudaGraphUpload(exec, stream_), "graph upload");  // device-side setup once, not per launch
      cudaGraphDestroy(g);
      graphs_cache_.push_back({tokens_dev, next_dev, capture_hidden_, store_logits_, exec, plan});
    }
    cuda_check(cudaGraphLaunch(exec, stream_), "graph launch");
  } else {
    enqueue_decode(tokens_dev, next_dev);
  }
  for (int64_t l = 0; l < L_; ++l)
    for (int b = 0; b < B_; ++b) h_total_[static_cast<size_t>(l * B_ + b)] += 1;
  record_transcript(L_);
}

void Engine::decode_step(const int32_t* tokens, int32_t* next, float* logits, float* hidden) {
  if (attn_only_) throw StateError("decode_step needs a full model (attention_only = 0)");
  for (int b = 0; b < B_; ++b)
    if (tokens[b] < 0 || tokens[b] >= V_) throw std::invalid_argument("token id out of range");
  capture_hidden_ = hidden != nullptr;
  store_logits_ = logits != nullptr;
  cuda_check(cudaMemcpyAsync(d_tokens_, tokens, static_cast<size_t>(B_) * 4, cudaMemcpyHostToDevice, stream_),
             "tokens h2d");
  decode_step_device(d_tokens_, d_next_);
  cuda_check(cudaMemcpyAsync(next, d_next_, static_cast<size_t>(B_) * 4, cudaMemcpyDeviceToHost, stream_),
             "next d2h");
  if (logits)
    cuda_check(cudaMemcpyAsync(logits, d_logits_, static_cast<size_t>(B_) * V_local_ * 4, cudaMemcpyDeviceToHost,
                               stream_),
               "logits d2h");
  if (hidden)
    cuda_check(cudaMemcpyAsync(hidden, d_hidden_, static_cast<size_t>(L_ + 1) * B_ * H_ * 4,
                               cudaMemcpyDeviceToHost, stream_),
               "hidden d2h");
  cuda_check(cudaStreamSynchronize(stream_), "decode sync");
}

void Engine::set_flag(int flag, int value) {
  if (flag == HX_FLAG_SKIP_COMM) {
    skip_comm_ = value;
    drop_graphs();
  } else if (flag == HX_FLAG_HOPB) {
    hopb_ = value != 0;
    drop_graphs();
  } else if (flag == HX_FLAG_COLLECTIVE_A2A) {
    nccl_a2a_ = value != 0;
    drop_graphs();
  } else {
    throw std::invalid_argument("unknown engine flag");
  }
}

int64_t Engine::moe_active_experts() {
  if (!moe_) return 0;
  int n = 0;
  cuda_check(cudaStreamSynchronize(stream_), "sync");
  cuda_check(cudaMemcpy(&n, d_gcount_, sizeof(int), cudaMemcpyDeviceToHost), "expert count");
  return n;
}

void Engine::synchronize() { cuda_check(cudaStreamSynchronize(stream_), "synchronize"); }

void Engine::profile_step(int64_t reps, double* ms) {
  if (!weights_ready_) throw StateError("weights are not initialised");
  for (int k = 0; k < 10; ++k) ms[k] = 0.0;
  std::vector<std::pair<int, cudaEvent_t>> evs;
  for (int64_t r = 0; r < reps; ++r) {
    evs.clear();
    prof_ = &evs;
    mark(-1);
    try {
      if (attn_only_) {
        for (int64_t l = 0; l < L_; ++l) harness_step_device(l, d_x_, d_out_);
      } else {
        decode_step_device(d_tokens_, d_next_);
      }
    } catch (...) {
      prof_ = nullptr;
      throw;
    }
    prof_ = nullptr;
    cuda_check(cudaStreamSynchronize(stream_), "profile sync");
    for (size_t i = 1; i < evs.size(); ++i) {
      float t = 0.f;
      cuda_check(cudaEventElapsedTime(&t, evs[i - 1].second, evs[i].second), "elapsed");
      if (evs[i].first >= 0 && evs[i].first < 10) ms[evs[i].first] += t / static_cast<double>(reps);
    }
    for (auto& e : evs) cudaEventDestroy(e.second);
  }
}

// ---------------------------------------------------------------------------
// Exact fp64 harness (HX_KV_F64; exact64.cu)
F64HarnessParams Engine::f64_params(int64_t layer) const {
  F64HarnessParams p{};
  p.k = k64_[layer];
  p.v = v64_[layer];
  p.qkv = d_qkv64_;
  p.total = d_total_ + layer * B_;
  p.qkv_stride = static_cast<int>((Qh_ + 2 * Kh_) * D_);
  p.batch = B_;
  p.tpa = tpa_;
  p.kvp = kvp_;
  p.chunk = chunk_;
  p.kvh_per_slot = kvh_per_slot_;
  p.q_per_slot = q_per_slot_;
  p.group = G_;
  p.w = static_cast<int>(D_);
  p.rows_cap = rows_cap64_;
  p.scale = 1.0 / std::sqrt(static_cast<double>(D_));
  return p;
}

// x [B][H] -> d_qkv64_ [B][(Q+2K)*Hsz] (x^T W_q | x^T W_k | x^T W_v, attention.hpp:479-484, 531-539)
void Engine::qkv_f64(int64_t layer, const double* x, int64_t x_len) {
  check_layer(layer);
  if (!f64_) throw StateError("the fp64 entry points need an exact harness (kv_dtype HX_KV_F64)");
  if (x_len != static_cast<int64_t>(B_) * H_) throw std::invalid_argument("hidden state has wrong width");
  if (!weights_ready_) throw StateError("weights are not initialised");
  cuda_check(cudaMemcpyAsync(d_x64_, x, static_cast<size_t>(x_len) * sizeof(double), cudaMemcpyHostToDevice,
                             stream_),
             "x h2d");
  cuda_check(launch_gemv_f64(d_x64_, B_, w64_[layer], static_cast<int>(H_), static_cast<int>((Qh_ + 2 * Kh_) * D_),
                             d_qkv64_, stream_),
             "f64 qkv");
}

void Engine::harness_step_f64(int64_t layer, const double* x, int64_t x_len, double* out, double* lse) {
  check_layer(layer);
  if (x_len != static_cast<int64_t>(B_) * H_) throw std::invalid_argument("hidden state has wrong width");
  require_context(layer);
  qkv_f64(layer, x, x_len);
  const F64HarnessParams p = f64_params(layer);
  cuda_check(launch_attn_f64_harness(p, 0, d_frag64_o_, d_frag64_lse_, stream_), "f64 shard attention");
  cuda_check(launch_merge_f64_harness(p, d_frag64_o_, d_frag64_lse_, d_out64_, d_lse64_, stream_), "f64 merge");
  const size_t ncols = static_cast<size_t>(p.qkv_stride);
  for (int b = 0; b < B_; ++b) {  // attend-then-append (attention.hpp:504-508)
    const double* kp = d_qkv64_ + b * ncols + Qh_ * D_;
    cuda_check(launch_append_f64(p, kp, kp + Kh_ * D_, ncols, b, 1, static_cast<int>(Kh_), stream_), "f64 append");
  }
  cuda_check(cudaMemcpyAsync(out, d_out64_, static_cast<size_t>(B_) * Qh_ * D_ * sizeof(double),
                             cudaMemcpyDeviceToHost, stream_),
             "out d2h");
  if (lse)
    cuda_check(cudaMemcpyAsync(lse, d_lse64_, static_cast<size_t>(B_) * Qh_ * sizeof(double), cudaMemcpyDeviceToHost,
                               stream_),
               "lse d2h");
  cuda_check(cudaStreamSynchronize(stream_), "f64 step sync");
  for (int b = 0; b < B_; ++b) h_total_[static_cast<size_t>(layer * B_ + b)] += 1;
  record_transcript(1);
}

void Engine::harness_reference_f64(int64_t layer, const double* x, int64_t x_len, double* out) {
  check_layer(layer);
  for (int b = 0; b < B_; ++b)  // reference_attention (attention.hpp:45)
    if (h_total_[static_cast<size_t>(layer * B_ + b)] == 0)
      throw std::invalid_argument("attention needs >= 1 context token");
  qkv_f64(layer, x, x_len);
  const F64HarnessParams p = f64_params(layer);
  // one softmax per query head over its KV head's whole global context ([tpa][B][q_per_slot] = [B][Q] for tpa 1)
  cuda_check(launch_attn_f64_harness(p, 1, d_frag64_o_, d_frag64_lse_, stream_), "f64 reference attention");
  std::vector<double> frag(static_cast<size_t>(tpa_) * B_ * q_per_slot_ * D_);
  cuda_check(cudaMemcpyAsync(frag.data(), d_frag64_o_, frag.size() * sizeof(double), cudaMemcpyDeviceToHost, stream_),
             "reference d2h");
  cuda_check(cudaStreamSynchronize(stream_), "f64 reference sync");
  for (int g = 0; g < tpa_; ++g)
    for (int b = 0; b < B_; ++b)
      std::memcpy(out + (static_cast<size_t>(b) * Qh_ + static_cast<size_t>(g) * q_per_slot_) * D_,
                  frag.data() + (static_cast<size_t>(g) * B_ + b) * q_per_slot_ * D_,
                  static_cast<size_t>(q_per_slot_) * D_ * sizeof(double));
}

void Engine::append_projected_f64(int64_t layer, const double* x, int64_t x_len) {
  for (int b = 0; b < B_; ++b)
    if (h_total_[static_cast<size_t>(layer * B_ + b)] + 1 > cap_) throw std::invalid_argument("KV capacity exceeded");
  qkv_f64(layer, x, x_len);
  const F64HarnessParams p = f64_params(layer);
  const size_t ncols = static_cast<size_t>(p.qkv_stride);
  for (int b = 0; b < B_; ++b) {
    const double* kp = d_qkv64_ + b * ncols + Qh_ * D_;
    cuda_check(launch_append_f64(p, kp, kp + Kh_ * D_, ncols, b, 1, static_cast<int>(Kh_), stream_), "f64 append");
  }
  cuda_check(cudaStreamSynchronize(stream_), "f64 append sync");
  for (int b = 0; b < B_; ++b) h_total_[static_cast<size_t>(layer * B_ + b)] += 1;
}

void Engine::append_kv_f64(int64_t layer, int64_t request, int64_t n, const double* k, const double* v) {
  check_layer(layer);
  if (!f64_) throw StateError("the fp64 entry points need an exact harness (kv_dtype HX_KV_F64)");
  if (request < 0 || request >= B_) throw std::invalid_argument("request out of range");
  if (n < 0) throw std::invalid_argument("token count must be >= 0");
  if (h_total_[static_cast<size_t>(layer * B_ + request)] + n > cap_)
    throw std::invalid_argument("KV capacity exceeded");
  if (n == 0) return;
  const size_t cnt = static_cast<size_t>(n * Kh_ * D_);
  double *dk = nullptr, *dv = nullptr;
  cuda_check(cudaMalloc(&dk, cnt * sizeof(double)), "append staging");
  cuda_check(cudaMalloc(&dv, cnt * sizeof(double)), "append staging");
  cuda_check(cudaMemcpyAsync(dk, k, cnt * sizeof(double), cudaMemcpyHostToDevice, stream_), "append h2d");
  cuda_check(cudaMemcpyAsync(dv, v, cnt * sizeof(double), cudaMemcpyHostToDevice, stream_), "append h2d");
  cuda_check(launch_append_f64(f64_params(layer), dk, dv, static_cast<size_t>(Kh_ * D_), static_cast<int>(request), n,
                               static_cast<int>(Kh_), stream_),
             "f64 append");
  cuda_check(cudaStreamSynchronize(stream_), "append sync");
  cudaFree(dk);
  cudaFree(dv);
  h_total_[static_cast<size_t>(layer * B_ + request)] += n;
}

void Engine::read_kv_f64(int64_t layer, int64_t request, int64_t rank, int64_t head, double* k, double* v) {
  check_layer(layer);
  if (!f64_) throw StateError("the fp64 entry points need an exact harness (kv_dtype HX_KV_F64)");
  if (head < 0 || head >= Kh_) throw std::invalid_argument("kv head out of range");
  const int64_t n = effective_tokens(layer, request, rank);
  const int grp = static_cast<int>(head / kvh_per_slot_), kvh = static_cast<int>(head % kvh_per_slot_);
  if (n == 0) return;
  double *dk = nullptr, *dv = nullptr;
  const size_t cnt = static_cast<size_t>(n * D_);
  cuda_check(cudaMalloc(&dk, cnt * sizeof(double)), "read staging");
  cuda_check(cudaMalloc(&dv, cnt * sizeof(double)), "read staging");
  cuda_check(launch_read_f64(f64_params(layer), grp * kvp_ + static_cast<int>(rank), static_cast<int>(request), kvh,
                             n, dk, dv, stream_),
             "f64 read");
  cuda_check(cudaMemcpyAsync(k, dk, cnt * sizeof(double), cudaMemcpyDeviceToHost, stream_), "read d2h");
  cuda_check(cudaMemcpyAsync(v, dv, cnt * sizeof(double), cudaMemcpyDeviceToHost, stream_), "read d2h");
  cuda_check(cudaStreamSynchronize(stream_), "read sync");
  cudaFree(dk);
  cudaFree(dv);
}

void Engine::info(hx_engine_info* o) const {
  std::memset(o, 0, sizeof(*o));
  o->kv_bytes_per_layer = static_cast<int64_t>(n_slots_) * B_ * kvh_per_slot_ * page_cap_ * page_bytes_;
  int64_t wb = static_cast<int64_t>(weight_bytes(plan_qkv_[0].p.Npad, plan_qkv_[0].p.K));
  if (mla_) wb += (Qh_ * D_ * W_ + static_cast<int64_t>(uv_heads_) * DV_ * D_) * 2;  // W_UK + W_UV
  auto bytes = [this](const GemvPlan& g) { return static_cast<int64_t>(weight_bytes(g.p.Npad, g.p.K)); };
  if (!attn_only_) {
    wb += bytes(plan_o_[0]);
    if (F_ > 0) wb += bytes(plan_gu_[0]) + bytes(plan_down_[0]);
    if (moe_)  // all experts held here (only the routed ones are read per step)
      wb += bytes(plan_router_[0]) + static_cast<int64_t>(E_local_) * (bytes(plan_egu_[0]) + bytes(plan_edown_[0]));
  }
  o->weight_bytes_per_layer = wb;
  o->head_bytes = attn_only_ ? 0 : bytes(plan_lm_) + V_ * H_ * 2;
  o->attn_streams = n_streams_;
  o->attn_splits = live_splits(0, false);  // the plan the next batched launch of layer 0 uses
  o->attn_items = static_cast<int64_t>(n_streams_) * o->attn_splits;
  o->attn_grid = attn_grid_;
  o->kernels_per_step = launches_per_step();
  o->page_cap = page_cap_;
  o->head_dim_padded = DP_;
  o->kv_dtype = kv4_ ? HX_KV_FP4_E2M1 : (f64_ ? HX_KV_F64 : (kv8_ ? HX_KV_FP8_E4M3 : HX_KV_BF16));
  o->w_dtype = w4_ ? HX_W_FP4_E2M1 : (w8_ ? HX_W_FP8_E4M3 : HX_W_BF16);
  o->comm_ranks = transport_ ? transport_->world() : 1;
  o->nccl_version = transport_ ? transport_->nccl_version() : 0;
  o->exchange = dist_mode_ == HX_POOL_LOCAL ? HX_EXCHANGE_NONE
                : !device_exchange()       ? HX_EXCHANGE_COLLECTIVE
                : (hopb_ && fused_)        ? HX_EXCHANGE_DEVICE_HOPB
                                           : HX_EXCHANGE_DEVICE;
}

}  // namespace hx

// ---------------------------------------------------------------------------
// Free functions (fp64, current device): the reference's primitives on
// caller-supplied operands (attention.hpp:43-78, 118-137).
namespace hx {
namespace {
struct DevBuf {
  void* p = nullptr;
  explicit DevBuf(size_t bytes) { cuda_check(cudaMalloc(&p, std::max<size_t>(bytes, 16)), "primitive buffer"); }
  ~DevBuf() { cudaFree(p); }
  double* d() const { return static_cast<double*>(p); }
};
void require_blackwell() {
  int dev = 0;
  cuda_check(cudaGetDevice(&dev), "cudaGetDevice");
  cudaDeviceProp prop{};
  cuda_check(cudaGetDeviceProperties(&prop, dev), "cudaGetDeviceProperties");
  if (prop.major < 10) throw CudaError("device is not sm_100 class (Blackwell); this build targets sm_100a only");
}
}  // namespace

void attention_f64(const double* q, int64_t nq, const double* keys, const double* values, int64_t tokens,
                   int64_t width, double* out, double* lse) {
  if (nq < 1 || tokens < 0 || width < 1) throw std::invalid_argument("attention operand sizes must be >= 1");
  if (width > kF64MaxWidth) throw std::invalid_argument("attention width > 512 is not supported");
  require_blackwell();
  const size_t qn = static_cast<size_t>(nq * width), kn = static_cast<size_t>(tokens * width);
  DevBuf dq(qn * 8), dk(kn * 8), dv(kn * 8), dout(qn * 8), dl(static_cast<size_t>(nq) * 8);
  cuda_check(cudaMemcpy(dq.d(), q, qn * 8, cudaMemcpyHostToDevice), "q h2d");
  if (kn) {
    cuda_check(cudaMemcpy(dk.d(), keys, kn * 8, cudaMemcpyHostToDevice), "keys h2d");
    cuda_check(cudaMemcpy(dv.d(), values, kn * 8, cudaMemcpyHostToDevice), "values h2d");
  }
  cuda_check(launch_attn_f64_plain(dq.d(), static_cast<int>(nq), dk.d(), dv.d(), tokens, static_cast<int>(width),
                                   dout.d(), dl.d(), nullptr),
             "f64 attention");
  cuda_check(cudaMemcpy(out, dout.d(), qn * 8, cudaMemcpyDeviceToHost), "out d2h");
  if (lse) cuda_check(cudaMemcpy(lse, dl.d(), static_cast<size_t>(nq) * 8, cudaMemcpyDeviceToHost), "lse d2h");
}

void merge_f64(int64_t nf, int64_t width, const double* outs, const double* lses, double* out, double* lse) {
  if (nf < 1) throw std::invalid_argument("merge needs >= 1 fragment");
  if (width < 0) throw std::invalid_argument("fragment widths differ");
  bool any = false;
  for (int64_t i = 0; i < nf; ++i) any |= lses[i] != -INFINITY;
  if (!any) throw std::invalid_argument("all fragments empty: nothing to merge");
  require_blackwell();
  const size_t on = static_cast<size_t>(nf * width);
  DevBuf dout(on * 8), dl(static_cast<size_t>(nf) * 8), dres(static_cast<size_t>(width) * 8), dlse(8);
  if (on) cuda_check(cudaMemcpy(dout.d(), outs, on * 8, cudaMemcpyHostToDevice), "outs h2d");
  cuda_check(cudaMemcpy(dl.d(), lses, static_cast<size_t>(nf) * 8, cudaMemcpyHostToDevice), "lses h2d");
  cuda_check(launch_merge_f64_plain(dout.d(), dl.d(), static_cast<int>(nf), static_cast<int>(width), dres.d(),
                                    dlse.d(), nullptr),
             "f64 merge");
  if (width) cuda_check(cudaMemcpy(out, dres.d(), static_cast<size_t>(width) * 8, cudaMemcpyDeviceToHost), "out d2h");
  if (lse) cuda_check(cudaMemcpy(lse, dlse.d(), 8, cudaMemcpyDeviceToHost), "lse d2h");
}
}  // namespace hx
