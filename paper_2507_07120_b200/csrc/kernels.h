// Kernel parameter blocks and launchers (internal to libhelix_b200.so).
#pragma once

#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

#include <mutex>

namespace hx {

#ifdef __CUDACC__
#define HX_HD __host__ __device__
#else
#define HX_HD
#endif
// Batch groups of 8 in the x-fragment image (xfrag.cuh): the GEMV instantiates
// 1, 2, 4 or 8 groups, so writers, readers and allocations use the padded count.
HX_HD inline int xf_nb8(int batch) { return batch <= 8 ? 1 : (batch <= 16 ? 2 : (batch <= 32 ? 4 : 8)); }

// Largest KVP width the fragment merges handle (merge.cuh): validate_config's
// max_gpus (types.hpp:63).
constexpr int kMaxKvp = 64;


// Dynamic shared memory opt-in (cudaFuncAttributeMaxDynamicSharedMemorySize)
// lives in each device's context: remembered per (kernel, device) with the
// largest size set so far, under a lock (loopback pools launch from several
// host threads; engines may sit on different devices of one process).
template <auto Kernel>
cudaError_t smem_optin(size_t bytes) {
  static std::mutex mu;
  static size_t done[64] = {};
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  const int slot = dev >= 0 && dev < 64 ? dev : 63;
  std::lock_guard<std::mutex> lk(mu);
  if (bytes <= done[slot] && dev < 64) return cudaSuccess;
  e = cudaFuncSetAttribute(Kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(bytes));
  if (e == cudaSuccess) done[slot] = bytes;
  return e;
}

// Programmatic dependent launch for the decode-step kernels (set by the engine).
void set_pdl(bool on);
bool pdl_enabled();

template <typename... KArgs, typename... Args>
cudaError_t launch_k(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t stream,
                     Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
}

// ---------------------------------------------------------------- attention
struct AttnParams {
  const uint8_t* kv;       // page pool for this layer: [slot_local][B][kvh_per_slot][page_cap] pages
  const float* q;          // [B][q_heads][DP] fp32 (padded rows)
  const int* total;        // [B] tokens appended to this layer's cache so far
  float* part_o;           // [n_items][qrows][DP]
  float* part_lse2;        // [n_items][qrows]  (log2 domain)
  int* work_counter;       // persistent-kernel work queue (self-resetting)
  int* done_counter;
  int dp, batch, q_heads, group, q_chunks, kvh_per_slot, q_per_slot;
  int kvp, chunk, page_cap, slot_base, n_local_slots;
  int n_streams, splits, n_items;
  float qscale;            // log2(e) / sqrt(head_size)
  int q_grp_base;          // first TPA group whose query heads are in `q` (0: all groups)
  int b_begin;             // requests [b_begin, b_begin + stream_batch) in this launch
  int stream_batch;        // (HOP-B launches one request at a time)
  const uint8_t* qimg;     // MLA: [B] absorbed-query images (kv_layout.cuh mla_q_offset)
  int qrows;               // GQA: query rows per stream (8, or 16 when the group exceeds 8)
  // one-source pools (local, KVP = 1): the split reduce also writes the merged
  // output's x-fragments (the merge of one fragment is the identity) -- no merge kernel
  uint8_t* xf_out;
  int xf16, hd;
  int kv8;                 // GQA: FP8 (e4m3) pages (kv_layout.cuh), f16 MMAs
  int kv4;                 // GQA: FP4 (e2m1 blocks of 32, power-of-two scales) pages, f16 MMAs
  // Fused split reduce (GQA): the CTA that completes a stream's last non-empty
  // split merges the stream's partials (split order) into frag_o / frag_lse
  // [slot_local][b][q][DP] (natural-log lse) -- no split-reduce launch (1); or
  // the attention kernel only counts the stream's finished splits and the
  // co-resident stream reducer merges and pushes (2).
  int fused;
  int stream_major;        // work order (attention.cu attn_item): 0 split-major, G > 0 groups of G streams
  int* stream_done;        // [n_streams] completed splits per stream (self-resetting)
  float* frag_o;
  float* frag_lse;
  // Device-initiated fragment exchange (HOP-B, distributed GQA pools): each
  // reduced stream is stored straight into the KVP peers' receive buffers
  // [src rank][batch][xchunk] (slice + lse slots, attention.hpp:492-502); once
  // every stream of the launch is out, the last CTA raises this rank's flag in
  // every peer (system-scope release). Exchange of request b overlaps the
  // attention of the requests after it.
  int push;
  float* const* peer_recv; // [kvp] receive buffers of this rank's KVP group (own included)
  unsigned* const* peer_flag; // [kvp] this rank's flag word in each peer
  int* pushed;             // streams pushed in this launch (self-resetting)
  int xchunk, xslice, xrank;
};
cudaError_t launch_attn_decode(const AttnParams& p, int grid, cudaStream_t stream);
// HOP-B stream reducer (fused == 2): reduce + push each stream as its splits land,
// next to the running attention kernel (attention.cu).
cudaError_t launch_attn_stream_reduce(const AttnParams& p, cudaStream_t stream);
// Quantised (FP8 / FP4) pages at DP = 128, <= 16 query rows, no fused reduce:
// the tcgen05 kernel (attention_tc.cu). grid = CTAs; items are statically
// assigned (item = CTA + n * grid).
bool attn_tc_supported(const AttnParams& p);
cudaError_t launch_attn_tc(const AttnParams& p, int grid, cudaStream_t stream);
// FP4 (e2m1 block) KV pages (kv_layout.cuh kv4_*): device hash fill, and the
// scatter of host-quantized rows (codes per element, exponents per 32-dim block).
cudaError_t launch_kv4_fill_hash(uint8_t* kv, int* total, int batch, int kv_heads, int kvh_per_slot, int kvp,
                                 int chunk, int head_dim, int dp, int page_cap, int slot_base, int n_local_slots,
                                 long long n, uint64_t seed, uint64_t stream_k, uint64_t stream_v,
                                 cudaStream_t stream);
cudaError_t launch_kv4_append_rows(uint8_t* kv, const uint8_t* codes_k, const uint8_t* codes_v, const int8_t* exp_k,
                                   const int8_t* exp_v, int n, int b, int* total, int batch, int kv_heads,
                                   int kvh_per_slot, int kvp, int chunk, int head_dim, int dp, int page_cap,
                                   int slot_base, int n_local_slots, cudaStream_t stream);
// Spin (one CTA) until every flag is raised, then lower it: the receive side
// of the device-initiated exchange (flags written by the peers' attention kernels).
cudaError_t launch_wait_flags(unsigned* flags, int n, cudaStream_t stream);
// MLA (tcgen05): items = (split, stream, value half); part_o [n_items][128][256],
// part_lse2 [n_items][128]; the split reduce writes frag_o [slot][b][q][512].
// tm_s / tm_v: CUtensorMap (128 B each) over the layer's latent pool viewed as
// [rows of 2 KB] x [256 x u64], boxes of 8 rows (16 KB chunk) / 16 rows (32 KB block);
// FP8 latents (p.kv8 = 1, kv_layout.cuh mla_kv_offset8): 12-row (24 KB) S chunks,
// 8-row (16 KB) V blocks, the e4m3 query image (mla_q_offset8) and kind::f8f6f4.
cudaError_t launch_mla_decode(const AttnParams& p, int grid, cudaStream_t stream, const void* tm_s, const void* tm_v);
// Encode the two tensor maps for a latent pool of `bytes` bytes (multiple of 2 KB).
cudaError_t make_mla_tensor_maps(const void* pool, size_t bytes, void* tm_s, void* tm_v, bool f8 = false);
cudaError_t launch_mla_split_reduce(const AttnParams& p, float* frag_o, float* frag_lse, cudaStream_t stream);
// MLA weight absorption (layer_oracle.hpp): q image = bf16(n_h . Wuk_h) from the
// QKV epilogue's n [B][Q][dp] and wuk [Q][hs][576]; v = o_h . Wuv_h from the merged
// latent output att [B][n_heads*512] and wuv [n_heads][512][hs] -> x-fragments of
// v [B][n_heads*hs] for the O-projection.
// f8: the e4m3 image with per-head power-of-two scales (kv_layout.cuh mla_q_offset8).
cudaError_t launch_mla_absorb_q(const float* n, const uint16_t* wuk, int batch, int q_heads, int hs, int dp,
                                uint8_t* qimg, cudaStream_t stream, bool f8 = false);
cudaError_t launch_mla_uv(const float* att, const uint16_t* wuv, int batch, int n_heads, int hs, uint8_t* xf,
                          cudaStream_t stream, int xf16 = 0);
cudaError_t launch_kv_fill_hash_mla(uint8_t* kv, int* total, int batch, int kvp, int chunk, int page_cap,
                                    int slot_base, int n_local_slots, long long n, uint64_t seed, uint64_t stream_k,
                                    cudaStream_t stream, bool f8 = false);
cudaError_t launch_attn_split_reduce(const AttnParams& p, float* frag_o, float* frag_lse,
                                     cudaStream_t stream);
cudaError_t launch_bump_totals(int* total, int n, cudaStream_t stream);
size_t attn_decode_smem_bytes(int dp);

// ---------------------------------------------------------------- GEMV
enum EMode : int { E_STORE = 0, E_QKV = 1, E_RESID = 2, E_SWIGLU = 3, E_LOGITS = 4 };

struct GemvParams {
  const uint4* w;        // bf16 weights, CTA-tile-major fragments [Npad/128][K/16][8][32 lanes][16 B]
                         // (tc: [Npad/128][K/16][16 row groups][2 k-halves][8 rows][16 B], gemv_tc.cu)
  int tc;                // batch > 16: tcgen05 GEMV (weights and x-fragments in its operand layouts)
  const uint8_t* xf;     // input activation fragments for K (xfrag.cuh)
  int N, Npad, K;
  int ksplit, kr_steps;  // k-chunks per 128-row block and k-steps per chunk
  int n_tiles;           // (Npad/128) * ksplit
  int* work_counter;     // [2] persistent tile queue (self-resetting), one pair per plan
  int batch;
  // RMSNorm statistics of the input (norm consumers scale y by rsqrt(mean(x^2) + eps))
  const float* ss_part;  // [n_ss][B]
  int n_ss;
  float eps;
  // split-K plumbing
  float* ypart;          // [ksplit][B][Npad]
  int* counters;         // [Npad/128], self-resetting
  // epilogue
  float* out;            // E_STORE / E_RESID (in-place residual) / E_LOGITS (optional)
  int out_stride;
  float* ss_out;         // [Npad/128][B] partial sums of squares of the written rows (E_RESID, E_STORE)
  uint8_t* xf_out;       // E_RESID: fragments of the new residual; E_SWIGLU: fragments of m
  // E_QKV
  float* q_out;          // [B][q_heads][DP]
  uint8_t* kv;           // page pool of this layer
  const int* total;      // [B]
  float* kv_dbg;         // optional [B][2][kv_heads][head_dim] fp32 copy of appended K/V
  int nq, nk, kv_heads, kvh_per_slot, rr_chunk, page_cap, slot_base, n_local_slots;
  int kv_head_base;      // global index of the first KV head in this projection
  int append;            // write K/V into the cache
  int kv8;               // GQA cache pages: 0 bf16, 1 FP8 e4m3 fragment-major, 2 FP8 tensor-core layout (kv_layout.cuh)
  int kv4;               // GQA cache pages are FP4 e2m1 blocks (fp8.cuh, kv_layout.cuh)
  uint8_t* q_img;        // MLA (mla = 1): q -> bf16 query images, latent -> MLA pages
  int mla;
  int kvp, head_dim, dp;
  // E_LOGITS
  unsigned long long* best;  // [B] packed (orderable logit, ~index)
  int n_offset;              // global index of row 0 (vocabulary shard offset)
  // Grouped GEMV (MoE experts): tiles run over the device-side active-expert list
  const int* group_count;    // active groups (nullptr: one ungrouped GEMV)
  const int* group_ids;      // [group] -> global expert id (ascending)
  int group_base;            // first expert id held here (weight block = id - group_base)
  int n_groups_max, tiles_per_group;
  long long w_group_stride;      // bytes between experts' weight blocks
  long long xf_group_stride;     // bytes between groups' input fragments (0: shared input)
  long long part_group_stride;   // floats between groups' split-K partials
  long long xf_out_group_stride; // bytes between groups' output fragments (E_SWIGLU)
  const float* route_w;      // [B][n_experts] routing weights: the epilogue combines groups
  int n_experts;
  const float* addend;       // optional [B][out_stride] added by E_RESID / E_STORE
  int* bump_total;           // optional [B]: token totals bumped by the epilogue (merge kernel skipped)
  int prefetch_stages;       // weight stages streamed before griddepcontrol.wait (<= ring depth)
  // FP8 weights (w8 = 1; B <= 16): w holds e4m3 bytes in the same tile order
  // ([Npad/128][K/16][8][32 lanes][8 B]), wscale the per-output power-of-two scales.
  // FP4 weights (w8 = 2; B <= 16): per (128-row block, pair of k-steps = 32 inputs)
  // 2 x [8 n-tiles][32 lanes][4 B] e2m1 codes (nibbles in the bf16 chunk's element
  // order) then 128 exponent bytes (e + 15, one per row), 2176 B; no wscale.
  int w8;
  const float* wscale;       // [Npad]
  int xf16;                  // xf_out written as two f16 terms (the next GEMV has FP8 weights)
  // Fused LSE combine (the O-projection, north star item 2; attention.hpp:118-175):
  // before its first x copy the GEMV's consumer warps merge the KVP fragments
  // into this GEMV's own input fragments (xf, in the xf16 image the weights
  // need), every CTA a slice, then raise merge_ctr; the producer streams weights
  // meanwhile and issues the x copies once all CTAs have merged. 0: off,
  // 1: received slices (distributed pools: merge_recv layout), 2: local fragments.
  // Needs the whole grid resident (launch_gemv refuses otherwise) and p.tc == 0;
  // the token-total bump of the skipped merge kernel moves to bump_total.
  int merge;
  const float* m_recv;        // merge 1: [kvp][B][xchunk] (slice values + lse slots)
  int m_chunk, m_slice, m_rank;
  const float* m_frag_o;      // merge 2: [slots][B][q_per_slot][dp]
  const float* m_frag_lse;    // merge 2: [slots][B][q_per_slot]
  int m_q_per_slot, m_dp;
  int m_kvp, m_head_dim;
  int* merge_ctr;             // arrivals (self-resetting)
};
cudaError_t launch_gemv(const GemvParams& p, int norm, int emode, int grid, cudaStream_t stream);
// tcgen05 inner product for p.tc plans (gemv_tc.cu); the epilogue kernel is shared.
cudaError_t launch_gemv_tc(const GemvParams& p, int nb8, int xs, int grid, cudaStream_t stream);
size_t gemv_smem_bytes(const GemvParams& p);

// x-fragment producers (xfrag.cuh layout; nb8 = ceil(batch / 8))
// xf16: write the fragments as two f16 terms (consumer GEMV has FP8 weights, xfrag.cuh)
cudaError_t launch_xprep_plain(const float* x, int batch, int K, int x_stride, uint8_t* xf, cudaStream_t s,
                               int xf16 = 0);
// Merged attention output (canonical LSE merge over KVP fragments, attention.hpp:90-137):
//  local pool: frag_o [slot][B][q_per_slot][DP], frag_lse [slot][B][q_per_slot]; K = hidden
//  exchanged:  recv [kvp src][B][chunk] (slice + lse slots); K = slice of rank exch_rank
// Both also bump the layer's per-request token totals (bump_total may be null):
// the attention has read them, so the token appended by the QKV epilogue now counts.
// plain != null: write the merged output as fp32 [B][K] there instead of x-fragments.
cudaError_t launch_xprep_merge_local(const float* frag_o, const float* frag_lse, int batch, int q_per_slot,
                                     int kvp, int head_dim, int dp, int K, uint8_t* xf, int* bump_total,
                                     cudaStream_t s, float* plain = nullptr, int xf16 = 0);
cudaError_t launch_xprep_merge_recv(const float* recv, int batch, int kvp, int chunk, int slice, int exch_rank,
                                    int head_dim, uint8_t* xf, int* bump_total, cudaStream_t s,
                                    float* plain = nullptr, int xf16 = 0);

// ---------------------------------------------------------------- misc
cudaError_t launch_merge_out(const float* frag_o, const float* frag_lse, int batch, int q_heads,
                             int q_per_slot, int kvp, int head_dim, int dp, float* out,
                             float* out_lse, int* bump_total, cudaStream_t stream);
cudaError_t launch_embed(const uint16_t* emb, const int* tokens, int batch, int hidden,
                         float* x, float* ss_part, uint8_t* xf, cudaStream_t stream, int xf16 = 0);
cudaError_t launch_argmax_finish(const unsigned long long* best, int batch, int* tokens_out,
                                 unsigned long long* best_reset, cudaStream_t stream);
// Scatter n tokens (bf16 K/V rows [n][kv_heads][head_dim]) of request b at global
// positions total[b] .. total[b]+n-1 into the round-robin page pool, then bump total.
cudaError_t launch_kv_append_rows(uint8_t* kv, const void* k_rows, const void* v_rows,
                                  int n, int b, int* total, int batch, int kv_heads,
                                  int kvh_per_slot, int kvp, int chunk, int head_dim, int dp,
                                  int page_cap, int slot_base, int n_local_slots, int fp8,
                                  cudaStream_t stream);
// Device-side synthetic fill: tokens [t0, t0+n) of every request from the hash RNG.
cudaError_t launch_kv_fill_hash(uint8_t* kv, int* total, int batch, int kv_heads,
                                int kvh_per_slot, int kvp, int chunk, int head_dim, int dp,
                                int page_cap, int slot_base, int n_local_slots, long long n,
                                uint64_t seed, uint64_t stream_k, uint64_t stream_v, int fp8,
                                cudaStream_t stream);
// Weight init from the hash RNG straight into the fragment-major layout.
// Segment list maps combined rows to (hash stream, column count, column offset).
struct WSeg {
  uint64_t stream;
  int rows_begin, rows_end;  // rows of the combined matrix covered
  int cols_total;            // columns of the source (reference-orientation) matrix
  int col_offset;            // source column of rows_begin (interleaved: of feature 0)
  int interleave;            // 0: contiguous; 1: SwiGLU gate rows; 2: SwiGLU up rows
  double scale;
  int k_offset;              // source row of k = 0 (tensor-parallel input shard)
  int col_limit;             // interleaved: first source column past this shard
};
cudaError_t launch_weight_init_hash(uint4* w, int Npad, int K, const WSeg* segs, int nseg,
                                    uint64_t seed, cudaStream_t stream, int tc = 0);
// FP8 weights: per-output power-of-two scales over the full input range k_full, then the e4m3 image.
cudaError_t launch_weight_init_hash_w8(uint8_t* w, float* scale, int Npad, int K, int k_full, const WSeg* segs,
                                       int nseg, uint64_t seed, cudaStream_t stream);
// FP4 weights: e2m1 blocks of 32 inputs per output row with a power-of-two
// scale (oracle quantize_fp4_cols), image per (128-row block, 32-input pair of
// k-steps): 2 x 1 KB fragment-major codes + 128 exponent bytes (gemv.cu).
cudaError_t launch_weight_init_hash_w4(uint8_t* w, int Npad, int K, const WSeg* segs, int nseg, uint64_t seed,
                                       cudaStream_t stream);
cudaError_t launch_emb_init_hash(uint16_t* emb, int vocab, int hidden, uint64_t seed,
                                 uint64_t stream_id, cudaStream_t stream);
// Plain row-major bf16: w[i] = bf16(hash_unit(seed, stream_id, idx0 + i) * scale), i < n.
cudaError_t launch_plain_init_hash(uint16_t* w, long long n, uint64_t seed, uint64_t stream_id, long long idx0,
                                   double scale, cudaStream_t stream);
cudaError_t launch_fill_zero(void* p, size_t bytes, cudaStream_t stream);
// Distributed Helix exchange: pack this rank's fragment into per-destination
// slices [kvp][batch][chunk] (chunk = slice + lse slots) for requests
// [b_begin, b_begin + b_count).
cudaError_t launch_pack_exchange(const float* frag_o, const float* frag_lse, int b_begin, int b_count, int batch,
                                 int q_per_slot, int head_dim, int dp, int kvp, int slice, int chunk, float* send,
                                 cudaStream_t s);
// MoE routing (one block): per request, top-k of router logits [B][E] (ties:
// lower index), softmax over the selected -> dense weights route_w [B][E];
// ascending list of selected experts within [e_begin, e_end) -> group_ids, count.
cudaError_t launch_moe_route(const float* logits, int batch, int n_experts, int top_k, int e_begin, int e_end,
                             float* route_w, int* group_ids, int* group_count, cudaStream_t s);
// Residual add of an all-reduced partial product + RMSNorm statistics.
cudaError_t launch_residual_add(float* x, const float* part, int batch, int hidden, float* ss_part,
                                uint8_t* xf, cudaStream_t s, int xf16 = 0);

// ---------------------------------------------------------------- exact fp64 harness (exact64.cu)
// DecodeHarness<double> numerics on the GPU for the drop-in C++ API: fp64 KV
// shards [slot][request][kv head][rows_cap][w] (row-major), fp64 weights,
// projections and merges. Widths up to kF64MaxWidth.
constexpr int kF64MaxWidth = 512;
struct F64HarnessParams {
  double* k;            // K shards
  double* v;            // V shards
  const double* qkv;    // [batch][qkv_stride] projections: query heads at column head*w
  int* total;           // [batch] tokens appended so far (this layer)
  int qkv_stride, batch, tpa, kvp, chunk, kvh_per_slot, q_per_slot, group, w;
  long long rows_cap;   // rows per (slot, request, kv head)
  double scale;         // 1/sqrt(w) (logit_scale, attention.hpp:35-38)
};
cudaError_t launch_attn_f64_plain(const double* q, int nq, const double* K, const double* V, long long n, int w,
                                  double* out, double* lse, cudaStream_t s);
cudaError_t launch_merge_f64_plain(const double* outs, const double* lses, int nf, int w, double* out, double* lse,
                                   cudaStream_t s);
cudaError_t launch_gemv_f64(const double* x, int B, const double* W, int K, int N, double* y, cudaStream_t s);
// mono = 0: per-rank fragments [tpa*kvp][batch][q_per_slot]; 1: one softmax over the group, [tpa][batch][q_per_slot]
cudaError_t launch_attn_f64_harness(const F64HarnessParams& p, int mono, double* frag_o, double* frag_lse,
                                    cudaStream_t s);
cudaError_t launch_merge_f64_harness(const F64HarnessParams& p, const double* frag_o, const double* frag_lse,
                                     double* out, double* lse, cudaStream_t s);
// append n token rows (ksrc/vsrc + t*src_stride: [kv_heads][w]) to request b, then total[b] += n
cudaError_t launch_append_f64(const F64HarnessParams& p, const double* ksrc, const double* vsrc, size_t src_stride,
                              int b, long long n, int kv_heads, cudaStream_t s);
cudaError_t launch_read_f64(const F64HarnessParams& p, int slot, int b, int kvh, long long n, double* k, double* v,
                            cudaStream_t s);

}  // namespace hx
