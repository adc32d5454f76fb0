// Host runtime of the B200 Helix decode step (C++, behind the C ABI).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <map>
#include <random>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/helix_b200.h"
#include "kernels.h"

namespace hx {

struct CudaError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct NcclError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct StateError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

void cuda_check(cudaError_t e, const char* what);

// Fragment-exchange layout (attention.hpp:492-502): per destination KVP rank p,
// out[4p..] = {first element, slice, first head, heads touched}; returns the
// padded chunk (floats per peer and request: slice + lse slots).
int64_t exchange_layout(int64_t q_per_group, int64_t head_size, int64_t kvp, int64_t* out);

struct Message {
  int64_t kind, src, dst, payload, lse;
};

// Free-function numerics in fp64 on the current device (exact64.cu kernels):
// partial_head_attention / merge_head_fragments on caller-supplied host operands.
void attention_f64(const double* q, int64_t nq, const double* keys, const double* values, int64_t tokens,
                   int64_t width, double* out, double* lse);
void merge_f64(int64_t nf, int64_t width, const double* outs, const double* lses, double* out, double* lse);

struct GemvPlan {
  GemvParams p{};
  int xmode = 0, emode = 0;  // xmode: 1 = RMSNorm consumer (scale y by the row's rsqrt(mean x^2))
};

class Transport;
class LoopbackHub;

class Engine {
 public:
  Engine(const hx_model_config& m, const hx_parallel_config& par, const hx_runtime_config& rt);
  ~Engine();

  void init_weights_mt19937(uint64_t seed);
  void init_weights_hash(uint64_t seed);
  void grow_random(int64_t layer, int64_t request, int64_t n, std::mt19937_64& rng);
  void append_kv(int64_t layer, int64_t request, int64_t n, const float* k, const float* v);
  void fill_kv_hash(int64_t n, uint64_t seed);
  int64_t total_tokens(int64_t layer, int64_t request) const;
  int64_t effective_tokens(int64_t layer, int64_t request, int64_t rank) const;
  int64_t max_min_gap(int64_t layer, int64_t request) const;
  void read_kv(int64_t layer, int64_t request, int64_t rank, int64_t head, float* k, float* v);

  void harness_step(int64_t layer, const float* x_host, int64_t x_len, float* out, float* lse);
  // Exact fp64 harness (kv_dtype HX_KV_F64, exact64.cu): DecodeHarness<double>
  // step / reference / append_projected and caller rows in double.
  void harness_step_f64(int64_t layer, const double* x, int64_t x_len, double* out, double* lse);
  void harness_reference_f64(int64_t layer, const double* x, int64_t x_len, double* out);
  void append_projected_f64(int64_t layer, const double* x, int64_t x_len);
  void append_kv_f64(int64_t layer, int64_t request, int64_t n, const double* k, const double* v);
  void read_kv_f64(int64_t layer, int64_t request, int64_t rank, int64_t head, double* k, double* v);
  bool exact_f64() const { return f64_; }
  void harness_step_device(int64_t layer, const float* x_dev, float* out_dev);
  void decode_step(const int32_t* tokens, int32_t* next, float* logits, float* hidden);
  void decode_step_device(const int32_t* tokens_dev, int32_t* next_dev);
  void synchronize();
  // Eager decode (or harness) steps with CUDA events after every launch on the
  // engine stream; ms[kind] += average milliseconds per step (see hx_profile_step).
  void profile_step(int64_t reps, double* ms);
  cudaStream_t stream() const { return stream_; }
  void info(hx_engine_info* out) const;
  void set_flag(int flag, int value);
  int64_t moe_active_experts();

  const std::vector<Message>& transcript() const { return transcript_; }
  void clear_transcript() { transcript_.clear(); }

  std::string last_error;

 private:
  void validate_reference_dims() const;
  void alloc();
  void plan_gemvs();
  void build_weights_common(uint64_t seed, bool qkv_hash);
  void upload_qkv_host(int64_t layer, const std::vector<double>& wq, const std::vector<double>& wk,
                       const std::vector<double>& wv);
  void enqueue_attention(int64_t layer);
  void enqueue_decode(const int32_t* tokens_dev, int32_t* next_dev);
  void record_transcript(int64_t layers);
  void require_context(int64_t layer) const;
  void check_layer(int64_t layer) const;
  int slot_local_of(int rank, int group) const;

  // ---- configuration
  int64_t H_, Qh_, Kh_, D_, F_, L_, V_;
  bool attn_only_;
  int tpa_, kvp_, chunk_;
  bool distributed_;
  int rank_;
  int B_;
  int64_t cap_;
  int device_;
  bool hopb_, graphs_;
  bool loopback_ = false;
  bool kv8_ = false;  // FP8 e4m3 GQA pages (hx_runtime_config.kv_dtype)
  bool kv4_ = false;  // FP4 e2m1 block-scaled GQA pages
  bool tc_ = false;   // batch > 16: tcgen05 GEMVs (weights / x-fragments in their operand images)
  bool w8_ = false;   // FP8 e4m3 GEMV weights (hx_runtime_config.w_dtype), per-output pow2 scales
  // local pool with KVP = 1 (one fragment per query head): the split reduce
  // writes the O-projection's x-fragments itself, the O-proj epilogue bumps
  // the token totals, and the merge kernel is not launched
  bool one_src_merge_ = false;
  bool fused_combine_ = false;   // LSE combine fused into the O-projection GEMV (HX_FUSED_COMBINE=0: merge kernel)
  // exact fp64 harness (HX_KV_F64): fp64 shards, weights and projections (exact64.cu)
  bool f64_ = false;
  int64_t rows_cap64_ = 0;
  std::vector<double*> k64_, v64_, w64_;  // per layer: K/V shards, [H][(Q+2K)*Hsz] weights
  double *d_x64_ = nullptr, *d_qkv64_ = nullptr, *d_frag64_o_ = nullptr, *d_frag64_lse_ = nullptr;
  double *d_out64_ = nullptr, *d_lse64_ = nullptr;
  F64HarnessParams f64_params(int64_t layer) const;
  void qkv_f64(int64_t layer, const double* x, int64_t x_len);
  bool w4_ = false;   // FP4 e2m1 GEMV weights: MX blocks of 32 inputs, pow2 scales inline (gemv.cu)
  int xf16_() const { return (w8_ || w4_) ? 1 : 0; }  // x-fragments as f16 terms (xfrag.cuh)
  // GEMV weight image bytes of an [Npad x K] matrix: bf16 2 B, e4m3 1 B, e2m1 17/32 B per
  // element (per 128 rows x 32 inputs: 2 KB of codes + 128 exponent bytes)
  size_t weight_bytes(int Npad, int K) const {
    const size_t n = static_cast<size_t>(Npad) * static_cast<size_t>(K);
    return w4_ ? n / 32 * 17 : (w8_ ? n : 2 * n);
  }
  std::map<const void*, float*> wscale_;     // FP8 weight block -> its [Npad] scales
  int DP_, G_, q_rows_, q_chunks_, kvh_per_slot_, q_per_slot_, n_slots_, slot_base_;
  int page_cap_;
  size_t page_bytes_;
  int num_sms_;
  // attention plan
  int n_streams_, splits_, n_items_, attn_grid_;
  int splits_req_ = 1;  // splits per stream for per-request (HOP-B) launches
  int ips_ = 8, min_pages_ = 32;  // split planner knobs (HX_ATTN_SPLIT)
  bool split_env_ = false;
  int plan_splits(int streams, int pages) const;
  bool attn_tc_ = false;
  bool kv8tc_ = false;  // FP8 pages in the tensor-core layout (kv_layout.cuh kv8tc_offset)
  int kv8_fmt() const { return kv8_ ? (kv8tc_ ? 2 : 1) : 0; }
  bool hopb_inkernel_ = false;
  bool local_stream_reduce_ = false;  // local pools: stream reducer instead of the split-reduce kernel (HX_LOCAL_STREAM_REDUCE=1; measured slower: DESIGN)
  int hopb_group_ = 1;  // HOP-B: requests per work group (HX_HOPB_GROUP; 1 = stream-major)  // HOP-B reduce inside the attention kernel (HX_HOPB_INKERNEL=1) vs the stream reducer  // quantised pages on the tcgen05 kernel (attention_tc.cu)
  int live_splits(int64_t layer, bool per_request) const;

  // ---- device state
  cudaStream_t stream_ = nullptr;
  std::vector<uint8_t*> kv_;   // per layer page pool
  int* d_total_ = nullptr;     // [L][B]
  std::vector<int64_t> h_total_;
  float* d_q_ = nullptr;
  float* d_part_o_ = nullptr;
  float* d_part_lse_ = nullptr;
  int* d_work_ = nullptr;      // [2] work counter, done counter
  float* d_frag_o_ = nullptr;
  float* d_frag_lse_ = nullptr;
  std::vector<uint4*> w_qkv_, w_o_, w_gu_, w_down_;
  uint4* w_lm_ = nullptr;
  uint16_t* emb_ = nullptr;
  float* d_ypart_ = nullptr;
  int* d_counters_ = nullptr;
  float* d_x_ = nullptr;       // residual stream / harness x [B][H]
  float* d_ss_ = nullptr;      // [max blocks][B]
  float* d_m_ = nullptr;       // [B][F]
  float* d_logits_ = nullptr;  // [B][V]
  unsigned long long* d_best_ = nullptr;
  int* d_tokens_ = nullptr;
  int* d_next_ = nullptr;
  float* d_out_ = nullptr;     // harness out [B][Q][Hsz]
  float* d_out_lse_ = nullptr;
  float* d_hidden_ = nullptr;  // [(L+1)][B][H]
  uint8_t* d_xf_resid_ = nullptr;  // x-fragments of the residual stream (QKV / gate-up / LM head input)
  uint8_t* d_xf_attn_ = nullptr;   // x-fragments of the merged attention output (O-proj input)
  uint8_t* d_xf_m_ = nullptr;      // x-fragments of silu(gate)*up (down-proj input)
  int* d_plan_ctr_ = nullptr;      // per-GEMV persistent tile queues
  WSeg* d_segs_ = nullptr;
  bool weights_ready_ = false;
  bool capture_hidden_ = false;
  bool store_logits_ = false;

  std::vector<GemvPlan> plan_qkv_, plan_o_, plan_gu_, plan_down_;
  GemvPlan plan_lm_;
  size_t ypart_elems_ = 0;
  int max_counters_ = 0;
  int64_t launches_per_step() const;

  struct GraphEntry {
    const int32_t* tokens;
    int32_t* next;
    bool hidden, logits;
    cudaGraphExec_t exec;
    std::vector<int> plan;  // live attention splits per layer baked into the graph
  };
  std::vector<GraphEntry> graphs_cache_;
  void drop_graphs();
  void mark(int kind);
  std::vector<std::pair<int, cudaEvent_t>>* prof_ = nullptr;

  std::vector<Message> transcript_;

  // ---- distributed pool (one rank of tpa*kvp; comm.h)
  int dist_mode_ = 0;          // HX_POOL_LOCAL / NCCL / LOOPBACK
  int skip_comm_ = 0;          // HX_FLAG_SKIP_COMM bitmask: 1 all-to-all, 2 all-reduces (measurement only)
  int grp_ = 0, r_ = 0, N_ = 1;
  int slice_ = 0, xchunk_ = 0; // exchanged elements per (peer, request) and padded chunk (+ lse slots)
  int F_local_ = 0, V_local_ = 0;
  Transport* transport_ = nullptr;
  float* d_send_ = nullptr;
  float* d_recv_ = nullptr;
  float* d_parth_ = nullptr;   // [B][H] partial products before the TP AllReduce
  cudaStream_t comm_stream_ = nullptr;
  // fused split reduce (GQA) and the device-initiated exchange (HOP-B on)
  bool fused_ = true;            // HX_FUSED_REDUCE=0: HOP-B keeps the split-reduce kernel (A/B)
  bool nccl_a2a_ = false;        // HX_A2A_NCCL=1: pack + NCCL grouped send/recv instead of the device exchange
  int* d_stream_done_ = nullptr;
  int* d_pushed_ = nullptr;
  unsigned* d_flags_ = nullptr;  // [kvp] raised by the peer that pushed to this rank
  float** d_peer_recv_ = nullptr;       // [kvp] group receive buffers (peer pointers)
  unsigned** d_peer_flag_ = nullptr;    // [kvp] this rank's flag word in each peer
  float** d_self_recv_ = nullptr;       // HX_FLAG_SKIP_COMM stand-ins: everything to this rank
  unsigned** d_self_flag_ = nullptr;
  bool peers_mapped_ = false;
  void ensure_peers();
  // GQA pools exchange device-initiated: the split reduce (or, under HOP-B, the
  // attention kernel itself) stores the slices into the peers' receive buffers
  bool device_exchange() const { return !mla_ && !nccl_a2a_ && dist_mode_ != HX_POOL_LOCAL; }
  std::vector<cudaEvent_t> hop_events_;
  void enqueue_exchange_and_attention_dist(int64_t layer);
  void init_dist_weights(uint64_t seed, bool qkv_hash);
  AttnParams attn_params(int64_t layer, int b_begin, int b_count);
  void launch_attention_kernels(const AttnParams& a);

  // ---- MoE FFN (router -> top-k -> grouped expert GEMVs over the active list)
  // ---- MLA attention (latent KV, tcgen05 kernel in mla.cu)
  bool mla_ = false;
  int W_ = 0, DV_ = 0;           // latent width (576) and value width (512)
  int AD_ = 0, ADP_ = 0;         // attention output width per head and its padded stride
  // MLA weight absorption (layer_oracle.hpp): W_UK [Q][Hsz][576] per layer (all heads),
  // W_UV [uv_heads][512][Hsz] per layer (the heads whose O-projection rows are held here)
  std::vector<uint16_t*> w_uk_, w_uv_;
  float* d_att_ = nullptr;       // MLA merged latent attention output [B][Q*512 or slice]
  int uv_heads_ = 0, uv_h0_ = 0;
  int K_o_ = 0;                  // O-projection input width on this device
  uint8_t* d_qimg_ = nullptr;    // [B] bf16 absorbed-query images
  struct alignas(64) MlaTmaps {  // CUtensorMap x 2 per layer over the latent pool
    unsigned char s[128], v[128];
  };
  std::vector<MlaTmaps> mla_tm_;
  int64_t attn_layer_ = 0;       // layer whose attention is being enqueued
  bool moe_ = false;
  int64_t E_ = 0, topk_ = 0, Fe_ = 0;
  int ep_ = 1, tpf_ = 1, ep_rank_ = 0, tpf_rank_ = 0, E_local_ = 0, e_begin_ = 0, Fe_local_ = 0;
  int n_groups_max_ = 0;
  std::vector<GemvPlan> plan_router_, plan_egu_, plan_edown_;
  std::vector<uint4*> w_router_, w_egu_, w_edown_;
  float* d_rlog_ = nullptr;     // [B][E] router logits
  float* d_route_w_ = nullptr;  // [B][E] routing weights (dense, zeros off the top-k)
  int* d_gids_ = nullptr;       // active local experts (ascending global ids)
  int* d_gcount_ = nullptr;
  uint8_t* d_xf_em_ = nullptr;  // [active slot] x-fragments of silu(gate)*up per expert
  float* d_moe_y_ = nullptr;    // [B][H] routed-expert output (when a shared expert follows)
  void enqueue_ffn(int64_t layer);
};

}  // namespace hx
