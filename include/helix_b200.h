/* helix_b200.h -- C-ABI boundary of the B200-native Helix decode step.
 *
 * Drop-in replacement for the reference's decode path
 * (/root/reference/proj/include/helixsim/attention.hpp, namespace
 * helixsim::exact). The reference is a header-only C++ template library with
 * no FFI; these entry points are what its C++ API lowers to, one per
 * reference operation (the C++ mirror in include/helixsim/exact_b200.hpp
 * re-exposes them under the reference's names):
 *
 *   DecodeHarness ctor          attention.hpp:428-443  -> hx_engine_create + hx_init_weights_mt19937
 *   DecodeHarness::grow_random  attention.hpp:452-456  -> hx_grow_random
 *   DecodeHarness::step         attention.hpp:460-510  -> hx_harness_step
 *   DecodeHarness::append_projected :531-539           -> fused into hx_harness_step / hx_decode_step
 *   DecodeHarness::transcript   attention.hpp:401-411  -> hx_transcript
 *   ShardedKVCache::{effective_tokens,total_tokens,max_min_gap} :286-299
 *                                                      -> hx_effective_tokens / hx_total_tokens / hx_max_min_gap
 *   ShardedKVCache::context     attention.hpp:303-309  -> hx_read_kv
 *   (analytical decode layer, latency.cpp:45-146)      -> hx_decode_step (full layer: O-proj, FFN, LM head)
 *
 * Conventions: plain pointers and sizes only; host buffers are caller-owned
 * and copied; no exceptions cross the ABI. Every call returns HX_OK or an
 * error code; the message (the reference's std::invalid_argument text where
 * the reference throws) is available from hx_last_error().
 * There is no CPU fallback: a missing/failed CUDA device is HX_ERR_CUDA.
 */
#ifndef HELIX_B200_H_
#define HELIX_B200_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HX_OK 0
#define HX_ERR_INVALID 1 /* reference std::invalid_argument */
#define HX_ERR_CUDA 2
#define HX_ERR_NCCL 3
#define HX_ERR_STATE 4

typedef struct hx_engine hx_engine;
typedef struct hx_rng hx_rng;

typedef struct hx_model_config {
  int64_t hidden;       /* H = query_heads * head_size (types.hpp:31) */
  int64_t query_heads;  /* Q */
  int64_t kv_heads;     /* K */
  int64_t head_size;    /* Hsz */
  int64_t ffn;          /* F (dense SwiGLU width) */
  int64_t layers;
  int64_t vocab;
  int32_t attention_only; /* 1: DecodeHarness semantics only (no norm/O/FFN/LM head) */
  int32_t reserved;
  /* MoE FFN (types.hpp:19-25): n_experts > 0 replaces the dense FFN by top_k-of-n_experts
   * routed SwiGLU experts of width expert_ffn plus a shared expert of width `ffn` (0: none). */
  int64_t n_experts;
  int64_t top_k;
  int64_t expert_ffn;
  /* MLA attention (types.hpp:37-49): kv_latent > 0 gives one latent KV head of width
   * 2*kv_latent (must be 576 = 512 value dims + 64 rope dims), kv_heads = 1, tpa = 1,
   * query_heads <= 128, absorbed projections (oracle/layer_oracle.hpp). */
  int64_t kv_latent;
} hx_model_config;

typedef struct hx_loopback hx_loopback;

typedef struct hx_parallel_config {
  int64_t tpa;          /* attention tensor parallelism (types.hpp:97) */
  int64_t kvp;          /* KV parallelism across the sequence (types.hpp:98) */
  int64_t chunk_size;   /* round-robin chunk (attention.hpp:237, default 16) */
  int32_t distributed;  /* HX_POOL_LOCAL: whole tpa*kvp pool on this device;
                           HX_POOL_NCCL: this process is one rank (one GPU) of the pool;
                           HX_POOL_LOOPBACK: one rank per host thread on one device (tests) */
  int32_t rank;         /* global rank id g*kvp + r (attention.hpp:555) when distributed */
  const void* nccl_unique_id; /* 128 bytes (ncclUniqueId) for HX_POOL_NCCL */
  hx_loopback* loopback;      /* shared group for HX_POOL_LOOPBACK */
  int64_t ep;           /* MoE expert parallelism (types.hpp:100); tpf = tpa*kvp/ep. 0 or 1: ep = 1 */
} hx_parallel_config;

#define HX_POOL_LOCAL 0
#define HX_POOL_NCCL 1
#define HX_POOL_LOOPBACK 2

typedef struct hx_runtime_config {
  int64_t batch;            /* concurrent requests (one DecodeHarness each) */
  int64_t capacity_tokens;  /* max global context per request */
  int32_t device;
  int32_t hopb;             /* HOP-B batch-wise comm/compute overlap (overlap.hpp:37-69) */
  int32_t use_graphs;       /* capture the decode step in a CUDA graph */
  int32_t kv_dtype;         /* KV page storage: HX_KV_BF16, or HX_KV_FP8_E4M3 (e4m3 RNE, saturating
                               at +-448, unit scale -- SURVEY 8f rank 2; GQA K/V pages, or MLA
                               latents on kind::f8f6f4 with an e4m3 query image and e4m3 P) */
  int32_t w_dtype;          /* GEMV weight storage: HX_W_BF16, HX_W_FP8_E4M3 (batch <= 16, hash init;
                               e4m3 with a power-of-two scale per output feature, applied in the
                               GEMV epilogue -- SURVEY 8f rank 2) or HX_W_FP4_E2M1 (batch <= 16,
                               hash init; e2m1 in MX-style blocks of 32 inputs per output feature
                               with a power-of-two scale -- the paper's FP4) */
  int32_t reserved;
} hx_runtime_config;

#define HX_KV_BF16 0
#define HX_KV_FP8_E4M3 1
#define HX_KV_F64 2 /* exact harness: fp64 shards, weights, projections and merges (DecodeHarness<double>) */
#define HX_KV_FP4_E2M1 3 /* GQA: e2m1 codes, one power-of-two scale per 32 dims of a token's K or V row
                            (MX-style blocks; head_size 32/64/128) -- the paper's FP4 */
#define HX_W_BF16 0
#define HX_W_FP8_E4M3 1
#define HX_W_FP4_E2M1 2

typedef struct hx_engine_info {
  int64_t kv_bytes_per_layer;      /* resident KV pool bytes on this device, per layer */
  int64_t weight_bytes_per_layer;  /* QKV + O + FFN weight bytes on this device, per layer */
  int64_t head_bytes;              /* embedding + LM head bytes */
  int64_t attn_streams, attn_splits, attn_items, attn_grid;
  int64_t kernels_per_step;        /* kernel launches of one hx_decode_step (or harness step) */
  int64_t page_cap;
  int64_t head_dim_padded;
  int64_t kv_dtype;                /* HX_KV_BF16 / HX_KV_FP8_E4M3 */
  int64_t w_dtype;                 /* HX_W_BF16 / HX_W_FP8_E4M3 / HX_W_FP4_E2M1 */
  int64_t comm_ranks;              /* ranks of the pool's world communicator (1: local pool) */
  int64_t nccl_version;            /* ncclGetVersion of the linked NCCL (0: no NCCL pool) */
  int64_t exchange;                /* KVP fragment exchange: HX_EXCHANGE_* (distributed pools) */
} hx_engine_info;

#define HX_EXCHANGE_NONE 0      /* local pool: the merge reads every rank's fragment */
#define HX_EXCHANGE_COLLECTIVE 1 /* pack + grouped send/recv all-to-all (NCCL, or loopback copies) */
#define HX_EXCHANGE_DEVICE 2    /* split reduce stores into the peers' receive buffers, flag-signalled */
#define HX_EXCHANGE_DEVICE_HOPB 3 /* attention kernel reduces + pushes each stream as it completes */

const char* hx_version(void);
const char* hx_last_error(const hx_engine* e); /* e may be NULL: last create/global error */

int hx_engine_create(const hx_model_config* model, const hx_parallel_config* par,
                     const hx_runtime_config* rt, hx_engine** out);
void hx_engine_destroy(hx_engine* e);
int hx_engine_get_info(const hx_engine* e, hx_engine_info* info);

/* --- weights --- */
/* W_q/W_k/W_v of layer l drawn exactly as DecodeHarness(seed + l) draws them
 * (attention.hpp:438-442, mt19937_64, row-major U[-1,1)), stored bf16;
 * extension weights from the counter hash (oracle/layer_oracle.hpp). */
int hx_init_weights_mt19937(hx_engine* e, uint64_t seed);
/* All weights from the counter hash (device-side, fast; bench shapes). */
int hx_init_weights_hash(hx_engine* e, uint64_t seed);

/* --- KV cache growth (reference grow_random: per token V then K) --- */
int hx_rng_create(uint64_t seed, hx_rng** out);
void hx_rng_destroy(hx_rng* r);
double hx_rng_unit_draw(hx_rng* r); /* attention.hpp:549-552 */
int hx_grow_random(hx_engine* e, int64_t layer, int64_t request, int64_t n, hx_rng* rng);
/* Append n tokens of host K/V rows [n][kv_heads][head_size] (fp32, stored bf16). */
int hx_append_kv(hx_engine* e, int64_t layer, int64_t request, int64_t n, const float* k,
                 const float* v);
/* Device-side synthetic growth of every (layer, request) cache by n tokens
 * (hash RNG, same values as ModelOracle::grow_hash). */
int hx_fill_kv_hash(hx_engine* e, int64_t n, uint64_t seed);

int64_t hx_total_tokens(const hx_engine* e, int64_t layer, int64_t request);
int64_t hx_effective_tokens(const hx_engine* e, int64_t layer, int64_t request, int64_t rank);
int64_t hx_max_min_gap(const hx_engine* e, int64_t layer, int64_t request);
/* Rows of (rank, kv head) in append order, trimmed (ShardedKVCache::context). */
int hx_read_kv(hx_engine* e, int64_t layer, int64_t request, int64_t rank, int64_t head,
               float* keys, float* values);

/* --- the decode step --- */
/* DecodeHarness::step for every request of the batch on one layer's cache:
 * x [batch][hidden] -> out [batch][query_heads][head_size] (+ lse [batch][query_heads],
 * natural log), then append each request's projected K/V (attend-then-append). */
int hx_harness_step(hx_engine* e, int64_t layer, const float* x, int64_t x_len, float* out,
                    float* lse);
/* Full decode step of the layer stack for the batch: tokens [batch] -> next
 * greedy tokens [batch]; optional logits [batch][vocab] and residual-stream
 * hidden states [layers+1][batch][hidden]. */
int hx_decode_step(hx_engine* e, const int32_t* tokens, int32_t* next_tokens, float* logits,
                   float* hidden);
/* Device-resident variant (no host copies): tokens/next are device pointers. */
int hx_decode_step_device(hx_engine* e, const int32_t* tokens_dev, int32_t* next_dev);
/* Device-resident harness step (x/out device pointers, [batch][hidden] / [batch][Q][Hsz]). */
int hx_harness_step_device(hx_engine* e, int64_t layer, const float* x_dev, float* out_dev);
int hx_synchronize(hx_engine* e);

/* --- exact harness (kv_dtype HX_KV_F64): DecodeHarness<double> in fp64 on the GPU ---
 * The reference's own precision for callers holding its tolerances (1e-10 / 1e-12);
 * attention-only local pools. x [batch][hidden]; out [batch][query_heads][head_size]. */
int hx_harness_step_f64(hx_engine* e, int64_t layer, const double* x, int64_t x_len, double* out,
                        double* lse);                                   /* step, attention.hpp:460-510 */
int hx_harness_reference_f64(hx_engine* e, int64_t layer, const double* x, int64_t x_len,
                             double* out);                              /* reference, :514-529 */
int hx_append_projected_f64(hx_engine* e, int64_t layer, const double* x, int64_t x_len); /* :531-539 */
/* append_round_robin of caller rows [n][kv_heads][head_size] (attention.hpp:262-282) */
int hx_append_kv_f64(hx_engine* e, int64_t layer, int64_t request, int64_t n, const double* k,
                     const double* v);
int hx_read_kv_f64(hx_engine* e, int64_t layer, int64_t request, int64_t rank, int64_t head, double* k,
                   double* v);                                          /* context, :303-309 */

/* --- free functions on caller-supplied operands (fp64, current CUDA device) --- */
/* partial_head_attention (attention.hpp:65-78) for n_queries queries [n_queries][width] over
 * one K/V [tokens][width] (row-major): out [n_queries][width], lse [n_queries] (natural log;
 * tokens == 0 gives the identity (0, -inf)). shard_attention (:375-396) is one call per KV
 * head; reference_attention (:43-53) is the same call over the whole context. width <= 512. */
int hx_attention_f64(const double* q, int64_t n_queries, const double* keys, const double* values,
                     int64_t tokens, int64_t width, double* out, double* lse);
/* merge_head_fragments (attention.hpp:118-137): canonical order (descending lse, ties by the
 * first differing coefficient), outs [n][width], lses [n] -> out [width], lse. */
int hx_merge_f64(int64_t n_fragments, int64_t width, const double* outs, const double* lses, double* out,
                 double* lse);
/* Profiling: `reps` eager steps (decode step, or one harness step per layer in
 * attention-only mode) with CUDA events after every launch on the engine
 * stream; ms[kind] = average milliseconds per step for kind
 * 0 embed, 1 qkv+append, 2 attention, 3 split-reduce, 4 o-proj (+merge),
 * 5 gate/up, 6 down, 7 lm-head+argmax, 8 merge (harness), 9 exchange /
 * all-reduce / residual (distributed pools). Advances the caches like real steps. */
#define HX_PROF_KINDS 10
int hx_profile_step(hx_engine* e, int64_t reps, double* ms);
/* The engine's CUDA stream (cudaStream_t) for event timing by the caller. */
void* hx_stream(hx_engine* e);

/* --- transcript: reference Message records (attention.hpp:401-411) ---
 * Bounded: the first 2^20 records are kept (hx_clear_transcript opens a new window). */
int64_t hx_transcript_size(const hx_engine* e);
/* out [n][5] = kind (0 broadcast, 1 all-to-all), src, dst, payload_scalars, lse_scalars */
int hx_transcript(const hx_engine* e, int64_t* out);
int hx_clear_transcript(hx_engine* e);

/* --- distributed plumbing --- */
/* Rank 0 creates the NCCL id and shares it (e.g. torch.distributed broadcast). */
int hx_nccl_get_unique_id(void* out128);
/* Fragment-exchange layout of one TPA group (attention.hpp:492-502), host only:
 * for each destination KVP rank p, out[4p..4p+3] = first flattened element,
 * element count (= slice), first head touched, heads touched; returns the
 * padded per-(peer, request) chunk in floats (slice + lse slots), or < 0. */
int64_t hx_exchange_layout(int64_t q_per_group, int64_t head_size, int64_t kvp, int64_t* out);
/* Runtime switches. HX_FLAG_HOPB: HOP-B on/off. HX_FLAG_SKIP_COMM (measurement
 * only, results are then wrong): bitmask 1 = replace the all-to-all by a local
 * copy, 2 = skip the all-reduces -- exposed-communication measurement. */
#define HX_FLAG_SKIP_COMM 1
#define HX_FLAG_HOPB 2
#define HX_FLAG_COLLECTIVE_A2A 3 /* 1: exchange through the collective transport instead of device stores */
int hx_engine_set_flag(hx_engine* e, int32_t flag, int32_t value);
/* MoE: experts held by this device that the last step's router selected in the
 * last layer (the grouped GEMVs streamed exactly these weight blocks); 0 for
 * dense models. Synchronises the engine stream. */
int64_t hx_moe_active_experts(hx_engine* e);
/* In-process group of n ranks on one device (one host thread per rank). */
int hx_loopback_create(int32_t n_ranks, hx_loopback** out);
void hx_loopback_destroy(hx_loopback* lb);

#ifdef __cplusplus
}
#endif

#endif /* HELIX_B200_H_ */
