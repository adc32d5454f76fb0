"""ctypes view of the CPU oracle (oracle/_build/libhelix_oracle.so).

TEST INFRASTRUCTURE ONLY: the oracle is the checker, never the product.
Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg use it.
"""
import ctypes as C
import os
import subprocess

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB_PATH = os.path.join(ROOT, "oracle", "_build", "libhelix_oracle.so")

_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            subprocess.check_call(["make", "-s", "-C", os.path.join(ROOT, "oracle")])
        L = C.CDLL(LIB_PATH)
        i64, u64, dp, ip, vp = C.c_int64, C.c_uint64, C.POINTER(C.c_double), C.POINTER(C.c_int64), C.c_void_p
        sig = {
            "oracle_last_error": (C.c_char_p, []),
            "oracle_rng_create": (vp, [u64]),
            "oracle_rng_free": (None, [vp]),
            "oracle_rng_unit_draw": (C.c_double, [vp]),
            "oracle_rng_next": (u64, [vp]),
            "oracle_round_bf16": (C.c_double, [C.c_double]),
            "oracle_round_e4m3": (C.c_double, [C.c_double]),
            "oracle_quantize_q_e4m3_pow2": (C.c_int, [C.POINTER(C.c_double), C.c_longlong]),
            "oracle_harness_set_kv_fp8": (None, [vp, C.c_int]),
            "oracle_model_set_kv_fp8": (None, [vp, C.c_int]),
            "oracle_harness_set_kv_fp4": (None, [vp, C.c_int]),
            "oracle_model_set_kv_fp4": (None, [vp, C.c_int]),
            "oracle_round_e2m1_block": (None, [dp, i64]),
            "oracle_harness_create": (C.c_int, [i64, i64, i64, i64, i64, i64, u64, C.c_int, C.POINTER(vp)]),
            "oracle_harness_free": (None, [vp]),
            "oracle_harness_grow_random": (C.c_int, [vp, i64, vp]),
            "oracle_harness_step": (C.c_int, [vp, dp, i64, dp, dp]),
            "oracle_harness_reference": (C.c_int, [vp, dp, i64, dp]),
            "oracle_harness_step_append": (C.c_int, [vp, dp, i64, dp, dp, dp, dp]),
            "oracle_harness_append_projected": (C.c_int, [vp, dp, i64]),
            "oracle_harness_project": (C.c_int, [vp, dp, i64, dp, dp, dp]),
            "oracle_harness_weights": (C.c_int, [vp, C.c_int, dp]),
            "oracle_harness_total_tokens": (i64, [vp]),
            "oracle_harness_effective_tokens": (i64, [vp, i64]),
            "oracle_harness_max_min_gap": (i64, [vp]),
            "oracle_harness_cache_rows": (C.c_int, [vp, i64, i64, C.c_int, dp]),
            "oracle_harness_token_order": (C.c_int, [vp, ip, ip]),
            "oracle_harness_transcript_size": (i64, [vp]),
            "oracle_harness_transcript": (C.c_int, [vp, ip]),
            "oracle_partial_head_attention": (C.c_int, [dp, dp, dp, i64, i64, dp, dp]),
            "oracle_reference_attention": (C.c_int, [dp, dp, dp, i64, i64, dp]),
            "oracle_merge_head_fragments": (C.c_int, [i64, i64, dp, dp, dp, dp]),
            "oracle_model_create": (C.c_int, [i64] * 11 + [u64, C.c_int, C.c_int, C.POINTER(vp)]),
            "oracle_model_create_moe": (C.c_int, [i64] * 14 + [u64, C.c_int, C.c_int, C.POINTER(vp)]),
            "oracle_model_create_ex": (C.c_int, [i64] * 15 + [u64, C.c_int, C.c_int, C.POINTER(vp)]),
            "oracle_model_create_w8": (C.c_int, [i64] * 11 + [u64, C.POINTER(vp)]),
            "oracle_model_create_wq": (C.c_int, [i64] * 15 + [u64, C.c_int, C.POINTER(vp)]),
            "oracle_model_create_ex_w8": (C.c_int, [i64] * 15 + [u64, C.POINTER(vp)]),
            "oracle_model_routes": (C.c_int, [vp, ip]),
            "oracle_model_route_gaps": (C.c_int, [vp, dp]),
            "oracle_model_free": (None, [vp]),
            "oracle_model_grow_random": (C.c_int, [vp, i64, i64, i64, vp]),
            "oracle_model_grow_hash": (C.c_int, [vp, i64, i64, i64]),
            "oracle_model_step": (C.c_int, [vp, ip, i64, dp, dp, ip]),
            "oracle_model_weight": (C.c_int, [vp, C.c_int, i64, dp]),
            "oracle_hash_unit": (C.c_double, [u64, u64, u64]),
        }
        for name, (res, args) in sig.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def _dp(a):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def _ip(a):
    return a.ctypes.data_as(C.POINTER(C.c_int64))


def check(rc):
    if rc == 1:
        raise ValueError(lib().oracle_last_error().decode())
    if rc != 0:
        raise RuntimeError(lib().oracle_last_error().decode())


class Rng:
    """std::mt19937_64 with the reference's unit_draw (attention.hpp:549-552)."""

    def __init__(self, seed):
        self.h = lib().oracle_rng_create(seed)

    def unit_draw(self):
        return lib().oracle_rng_unit_draw(self.h)

    def draws(self, n):
        return np.array([self.unit_draw() for _ in range(n)])

    def __del__(self):
        try:
            lib().oracle_rng_free(self.h)
        except Exception:
            pass


def round_e4m3(a):
    f = np.vectorize(lib().oracle_round_e4m3)
    return f(np.asarray(a, dtype=np.float64))


def quantize_q_e4m3_pow2(q):
    """FP8-latent MLA query quantisation (layer_oracle.cpp quantize_q_e4m3_pow2): returns (values, e)."""
    a = np.ascontiguousarray(np.asarray(q, dtype=np.float64)).copy()
    e = lib().oracle_quantize_q_e4m3_pow2(a.ctypes.data_as(C.POINTER(C.c_double)), a.size)
    return a, e


def round_bf16(a):
    f = np.vectorize(lib().oracle_round_bf16)
    return f(np.asarray(a, dtype=np.float64))


class Harness:
    """Oracle DecodeHarness<double> (attention.hpp:419-563)."""

    def __init__(self, q, k, hsz, tpa, kvp, chunk, seed, bf16=False, kv_fp8=False, kv_fp4=False):
        self.q, self.k, self.hsz, self.tpa, self.kvp = q, k, hsz, tpa, kvp
        h = C.c_void_p()
        check(lib().oracle_harness_create(q, k, hsz, tpa, kvp, chunk, seed, int(bf16), C.byref(h)))
        if kv_fp8:
            lib().oracle_harness_set_kv_fp8(h, 1)
        if kv_fp4:
            lib().oracle_harness_set_kv_fp4(h, 1)
        self.h = h

    @property
    def hidden(self):
        return self.q * self.hsz

    def grow_random(self, n, rng):
        check(lib().oracle_harness_grow_random(self.h, n, rng.h))

    def step(self, x):
        x = np.ascontiguousarray(x, dtype=np.float64)
        out = np.zeros((self.q, self.hsz))
        lse = np.zeros(self.q)
        check(lib().oracle_harness_step(self.h, _dp(x), x.size, _dp(out), _dp(lse)))
        return out, lse

    def step_append(self, x, k, v):
        """step(x) but append the given rows [kv_heads x w] (e.g. what the GPU stored)."""
        x = np.ascontiguousarray(x, dtype=np.float64)
        k = np.ascontiguousarray(k, dtype=np.float64)
        v = np.ascontiguousarray(v, dtype=np.float64)
        out = np.zeros((self.q, self.hsz))
        lse = np.zeros(self.q)
        check(lib().oracle_harness_step_append(self.h, _dp(x), x.size, _dp(out), _dp(lse), _dp(k), _dp(v)))
        return out, lse

    def reference(self, x):
        x = np.ascontiguousarray(x, dtype=np.float64)
        out = np.zeros((self.q, self.hsz))
        check(lib().oracle_harness_reference(self.h, _dp(x), x.size, _dp(out)))
        return out

    def append_projected(self, x):
        x = np.ascontiguousarray(x, dtype=np.float64)
        check(lib().oracle_harness_append_projected(self.h, _dp(x), x.size))

    def project(self, x):
        x = np.ascontiguousarray(x, dtype=np.float64)
        q = np.zeros(self.q * self.hsz)
        k = np.zeros((self.k, self.hsz))
        v = np.zeros((self.k, self.hsz))
        check(lib().oracle_harness_project(self.h, _dp(x), x.size, _dp(q), _dp(k), _dp(v)))
        return q, k, v

    def weights(self, which):
        cols = self.q * self.hsz if which == 0 else self.k * self.hsz
        out = np.zeros((self.hidden, cols))
        check(lib().oracle_harness_weights(self.h, which, _dp(out)))
        return out

    def total_tokens(self):
        return lib().oracle_harness_total_tokens(self.h)

    def effective_tokens(self, r):
        return lib().oracle_harness_effective_tokens(self.h, r)

    def max_min_gap(self):
        return lib().oracle_harness_max_min_gap(self.h)

    def cache_rows(self, rank, head, which):
        n = self.effective_tokens(rank)
        out = np.zeros((n, self.hsz))
        check(lib().oracle_harness_cache_rows(self.h, rank, head, which, _dp(out)))
        return out

    def token_order(self):
        n = self.total_tokens()
        r = np.zeros(n, dtype=np.int64)
        w = np.zeros(n, dtype=np.int64)
        check(lib().oracle_harness_token_order(self.h, _ip(r), _ip(w)))
        return r, w

    def transcript(self):
        n = lib().oracle_harness_transcript_size(self.h)
        out = np.zeros((n, 5), dtype=np.int64)
        check(lib().oracle_harness_transcript(self.h, _ip(out)))
        return out

    def __del__(self):
        try:
            lib().oracle_harness_free(self.h)
        except Exception:
            pass


def partial_head_attention(q, keys, values):
    q = np.ascontiguousarray(q, dtype=np.float64)
    keys = np.ascontiguousarray(keys, dtype=np.float64).reshape(-1, q.size)
    values = np.ascontiguousarray(values, dtype=np.float64).reshape(-1, q.size)
    out = np.zeros(q.size)
    lse = np.zeros(1)
    check(lib().oracle_partial_head_attention(_dp(q), _dp(keys), _dp(values), keys.shape[0], q.size, _dp(out), _dp(lse)))
    return out, lse[0]


def reference_attention(q, keys, values):
    q = np.ascontiguousarray(q, dtype=np.float64)
    keys = np.ascontiguousarray(keys, dtype=np.float64).reshape(-1, q.size)
    values = np.ascontiguousarray(values, dtype=np.float64).reshape(-1, q.size)
    out = np.zeros(q.size)
    check(lib().oracle_reference_attention(_dp(q), _dp(keys), _dp(values), keys.shape[0], q.size, _dp(out)))
    return out


def merge_head_fragments(outs, lses):
    outs = np.ascontiguousarray(outs, dtype=np.float64)
    lses = np.ascontiguousarray(lses, dtype=np.float64)
    out = np.zeros(outs.shape[1])
    lse = np.zeros(1)
    check(lib().oracle_merge_head_fragments(outs.shape[0], outs.shape[1], _dp(outs), _dp(lses), _dp(out), _dp(lse)))
    return out, lse[0]


class Model:
    """Oracle decoder stack (layer_oracle.hpp)."""

    WEIGHTS = {"wq": 0, "wk": 1, "wv": 2, "wo": 3, "wgate": 4, "wup": 5, "wdown": 6, "emb": 7, "lm": 8}

    def __init__(self, hidden, q, k, hsz, ffn, layers, vocab, tpa=1, kvp=1, chunk=16, batch=1,
                 seed=0, qkv_hash=False, bf16=True, moe=None, kv_latent=0, kv_fp8=False, w_fp8=False,
                 kv_fp4=False, w_fp4=False):
        """moe = (n_experts, top_k, expert_ffn): every layer's FFN is routed MoE,
        `ffn` is then the shared expert width (0: none). kv_latent > 0: MLA
        attention with latent width 2*kv_latent (layer_oracle.hpp). w_fp8: e4m3
        GEMV weights with per-output power-of-two scales (dense, hash init)."""
        self.dims = dict(hidden=hidden, q=q, k=k, hsz=hsz, ffn=ffn, layers=layers, vocab=vocab)
        self.batch = batch
        self.moe = moe
        h = C.c_void_p()
        if w_fp4:
            assert qkv_hash
            m = moe or (0, 0, 0)
            check(lib().oracle_model_create_wq(hidden, q, k, hsz, ffn, layers, vocab, m[0], m[1], m[2], kv_latent,
                                               tpa, kvp, chunk, batch, seed, 2, C.byref(h)))
        elif w_fp8 and (moe or kv_latent):
            assert qkv_hash
            m = moe or (0, 0, 0)
            check(lib().oracle_model_create_ex_w8(hidden, q, k, hsz, ffn, layers, vocab, m[0], m[1], m[2], kv_latent,
                                                  tpa, kvp, chunk, batch, seed, C.byref(h)))
        elif w_fp8:
            assert qkv_hash
            check(lib().oracle_model_create_w8(hidden, q, k, hsz, ffn, layers, vocab, tpa, kvp, chunk, batch, seed,
                                               C.byref(h)))
        elif kv_latent:
            m = moe or (0, 0, 0)
            check(lib().oracle_model_create_ex(hidden, q, k, hsz, ffn, layers, vocab, m[0], m[1], m[2], kv_latent,
                                               tpa, kvp, chunk, batch, seed, int(qkv_hash), int(bf16), C.byref(h)))
        elif moe:
            check(lib().oracle_model_create_moe(hidden, q, k, hsz, ffn, layers, vocab, moe[0], moe[1], moe[2],
                                                tpa, kvp, chunk, batch, seed, int(qkv_hash), int(bf16),
                                                C.byref(h)))
        else:
            check(lib().oracle_model_create(hidden, q, k, hsz, ffn, layers, vocab, tpa, kvp, chunk, batch,
                                            seed, int(qkv_hash), int(bf16), C.byref(h)))
        if kv_fp8:
            lib().oracle_model_set_kv_fp8(h, 1)
        if kv_fp4:
            lib().oracle_model_set_kv_fp4(h, 1)
        self.h = h

    def routes(self):
        """Last step's selected experts [layers][B][top_k] (descending router logit)."""
        out = np.zeros((self.dims["layers"], self.batch, self.moe[1]), dtype=np.int64)
        check(lib().oracle_model_routes(self.h, _ip(out)))
        return out

    def route_gaps(self):
        """Last step's router margin r[k-th] - r[(k+1)-th], [layers][B]."""
        out = np.zeros((self.dims["layers"], self.batch))
        check(lib().oracle_model_route_gaps(self.h, _dp(out)))
        return out

    def grow_random(self, layer, request, n, rng):
        check(lib().oracle_model_grow_random(self.h, layer, request, n, rng.h))

    def grow_hash(self, layer, request, n):
        check(lib().oracle_model_grow_hash(self.h, layer, request, n))

    def step(self, tokens):
        d = self.dims
        t = np.ascontiguousarray(tokens, dtype=np.int64)
        logits = np.zeros((self.batch, d["vocab"]))
        hidden = np.zeros((d["layers"] + 1, self.batch, d["hidden"]))
        nxt = np.zeros(self.batch, dtype=np.int64)
        check(lib().oracle_model_step(self.h, _ip(t), t.size, _dp(logits), _dp(hidden), _ip(nxt)))
        return logits, hidden, nxt

    def weight(self, name, layer=0):
        d = self.dims
        H, F, V = d["hidden"], d["ffn"], d["vocab"]
        shapes = {"wq": (H, d["q"] * d["hsz"]), "wk": (H, d["k"] * d["hsz"]), "wv": (H, d["k"] * d["hsz"]),
                  "wo": (H, H), "wgate": (H, F), "wup": (H, F), "wdown": (F, H), "emb": (V, H), "lm": (H, V)}
        out = np.zeros(shapes[name])
        check(lib().oracle_model_weight(self.h, self.WEIGHTS[name], layer, _dp(out)))
        return out

    def __del__(self):
        try:
            lib().oracle_model_free(self.h)
        except Exception:
            pass


def round_e2m1_block(x):
    """The oracle's FP4 block rounding (helix_oracle.cpp round_e2m1_block) of one block."""
    a = np.ascontiguousarray(x, dtype=np.float64).copy()
    lib().oracle_round_e2m1_block(_dp(a), a.size)
    return a


def hash_unit(seed, stream, index):
    return lib().oracle_hash_unit(seed, stream, index)
