"""B200 mirror of the reference's exact-attention harness API.

Reference: /root/reference/proj/include/helixsim/attention.hpp, namespace
helixsim::exact. Same names, argument meaning and error behaviour
(std::invalid_argument -> ValueError with the reference's message), computed
by libhelix_b200.so on the GPU. One DecodeHarness here drives `batch`
requests (one reference harness each, identical seeded weights,
attention.hpp:438-442) through a single batched GPU step.
"""
import ctypes as C
from dataclasses import dataclass

import numpy as np

from ._lib import (KV_DTYPES, W_DTYPES, EngineInfo, ModelConfig, ParallelConfig, RuntimeConfig, check, lib)

_fp = C.POINTER(C.c_float)
_dp = C.POINTER(C.c_double)


def _f32(a):
    return np.ascontiguousarray(a, dtype=np.float32)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


# ---------------------------------------------------------------------------- free functions (fp64, GPU)
def partial_head_attention(q, keys, values):
    """partial_head_attention (attention.hpp:65-78) for one query [w] or a group
    [nq, w] over keys/values [tokens, w]: (partial_out, lse); empty -> (0, -inf)."""
    q, k, v = _f64(q), _f64(keys), _f64(values)
    single = q.ndim == 1
    q2 = q.reshape(1, -1) if single else q
    nq, w = q2.shape
    n = k.shape[0] if k.size else 0
    out, lse = np.zeros((nq, w)), np.zeros(nq)
    check(lib().hx_attention_f64(q2.ctypes.data_as(_dp), nq, k.ctypes.data_as(_dp), v.ctypes.data_as(_dp), n, w,
                                 out.ctypes.data_as(_dp), lse.ctypes.data_as(_dp)))
    return (out[0], float(lse[0])) if single else (out, lse)


def reference_attention(q, keys, values):
    """reference_attention (attention.hpp:43-53): throws on an empty context."""
    k = _f64(keys)
    if k.shape[0] == 0:
        raise ValueError("attention needs >= 1 context token")
    return partial_head_attention(q, keys, values)[0]


def merge_head_fragments(outs, lses):
    """merge_head_fragments (attention.hpp:118-137): outs [n, w], lses [n] -> (out, lse)."""
    o, l = _f64(outs), _f64(lses)
    n = l.size
    w = o.shape[1] if o.ndim == 2 else 0
    out, lse = np.zeros(w), np.zeros(1)
    check(lib().hx_merge_f64(n, w, o.ctypes.data_as(_dp), l.ctypes.data_as(_dp), out.ctypes.data_as(_dp),
                             lse.ctypes.data_as(_dp)))
    return out, float(lse[0])


class Rng:
    """std::mt19937_64 with the reference's unit_draw (attention.hpp:549-552)."""

    def __init__(self, seed):
        h = C.c_void_p()
        check(lib().hx_rng_create(seed, C.byref(h)))
        self._h = h

    def unit_draw(self):
        return lib().hx_rng_unit_draw(self._h)

    def random_matrix(self, rows, cols):
        """DecodeHarness::random_matrix (attention.hpp:541-546), row-major draws."""
        return np.array([[self.unit_draw() for _ in range(cols)] for _ in range(rows)])

    def __del__(self):
        try:
            lib().hx_rng_destroy(self._h)
        except Exception:
            pass


@dataclass
class Dims:
    """DecodeHarness::Dims (attention.hpp:421-426)."""
    query_heads: int
    kv_heads: int
    head_size: int

    def hidden(self):
        return self.query_heads * self.head_size


class MsgKind:
    Broadcast = 0
    AllToAll = 1


class _Engine:
    def __init__(self, model, tpa, kvp, chunk_size, batch, capacity, device=0, use_graphs=True, hopb=False,
                 pool=0, rank=0, nccl_id=None, loopback=None, ep=1, kv_dtype="bf16", w_dtype="bf16"):
        self.mc = model
        self._nccl_buf = C.create_string_buffer(bytes(nccl_id), 128) if nccl_id is not None else None
        self._loopback = loopback  # the group must outlive its engines
        self.pc = ParallelConfig(tpa=tpa, kvp=kvp, chunk_size=chunk_size, distributed=pool, rank=rank,
                                 nccl_unique_id=C.cast(self._nccl_buf, C.c_void_p) if nccl_id is not None else None,
                                 loopback=loopback._h if loopback is not None else None, ep=ep)
        if kv_dtype not in KV_DTYPES:
            raise ValueError(f"kv_dtype must be one of {sorted(KV_DTYPES)}")
        if w_dtype not in W_DTYPES:
            raise ValueError(f"w_dtype must be one of {sorted(W_DTYPES)}")
        self.rc = RuntimeConfig(batch=batch, capacity_tokens=capacity, device=device, hopb=int(hopb),
                                use_graphs=int(use_graphs), kv_dtype=KV_DTYPES[kv_dtype], w_dtype=W_DTYPES[w_dtype])
        h = C.c_void_p()
        check(lib().hx_engine_create(C.byref(self.mc), C.byref(self.pc), C.byref(self.rc), C.byref(h)))
        self._h = h
        self.batch = batch

    def _check(self, rc):
        check(rc, self._h)

    def info(self):
        i = EngineInfo()
        self._check(lib().hx_engine_get_info(self._h, C.byref(i)))
        return {f: getattr(i, f) for f, _ in EngineInfo._fields_}

    def transcript(self):
        n = lib().hx_transcript_size(self._h)
        out = np.zeros((n, 5), dtype=np.int64)
        if n:
            self._check(lib().hx_transcript(self._h, out.ctypes.data_as(C.POINTER(C.c_int64))))
        return out

    def close(self):
        if getattr(self, "_h", None):
            lib().hx_engine_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class DecodeHarness(_Engine):
    """DecodeHarness(dims, tpa, kvp, chunk_size, seed) (attention.hpp:428-443) on the GPU.

    W_q/W_k/W_v are the reference's own mt19937_64(seed) draws, stored bf16.
    """

    def __init__(self, dims, tpa, kvp, chunk_size, seed, batch=1, capacity=4096, device=0, kv_dtype="bf16"):
        if not isinstance(dims, Dims):
            dims = Dims(*dims)
        self.dims = dims
        mc = ModelConfig(hidden=dims.query_heads * dims.head_size, query_heads=dims.query_heads,
                         kv_heads=dims.kv_heads, head_size=dims.head_size, ffn=16, layers=1, vocab=1,
                         attention_only=1)
        super().__init__(mc, tpa, kvp, chunk_size, batch, capacity, device, use_graphs=False, kv_dtype=kv_dtype)
        self._tpa, self._kvp = tpa, kvp
        self.exact = kv_dtype == "f64"  # fp64 weights / shards / merges (DecodeHarness<double> precision)
        self._check(lib().hx_init_weights_mt19937(self._h, seed))

    def pool(self):
        return self._tpa * self._kvp

    def grow_random(self, n, rng, request=0):
        """attention.hpp:452-456 (per token: V drawn before K)."""
        self._check(lib().hx_grow_random(self._h, 0, request, n, rng._h))

    def append(self, keys, values, request=0):
        """Append host K/V rows [n][kv_heads][head_size] round-robin."""
        k, v = _f32(keys), _f32(values)
        n = k.shape[0]
        self._check(lib().hx_append_kv(self._h, 0, request, n, k.ctypes.data_as(_fp), v.ctypes.data_as(_fp)))

    def step(self, x, return_lse=False):
        """DecodeHarness::step (attention.hpp:460-510) for every request.

        x: [hidden] (batch 1) or [batch, hidden]; returns [Q, Hsz] or [batch, Q, Hsz]."""
        if self.exact:
            x = _f64(x)
            out = np.zeros((self.batch, self.dims.query_heads, self.dims.head_size))
            lse = np.zeros((self.batch, self.dims.query_heads))
            self._check(lib().hx_harness_step_f64(self._h, 0, x.ctypes.data_as(_dp), x.size,
                                                  out.ctypes.data_as(_dp), lse.ctypes.data_as(_dp)))
            if x.ndim == 1 and self.batch == 1:
                out, lse = out[0], lse[0]
            return (out, lse) if return_lse else out
        x = _f32(x)
        single = x.ndim == 1
        out = np.zeros((self.batch, self.dims.query_heads, self.dims.head_size), dtype=np.float32)
        lse = np.zeros((self.batch, self.dims.query_heads), dtype=np.float32)
        self._check(lib().hx_harness_step(self._h, 0, x.ctypes.data_as(_fp), x.size, out.ctypes.data_as(_fp),
                                          lse.ctypes.data_as(_fp)))
        if single and self.batch == 1:
            out, lse = out[0], lse[0]
        return (out, lse) if return_lse else out

    def reference(self, x):
        """DecodeHarness::reference (attention.hpp:514-529): monolithic attention over
        the global context, no append (exact harness)."""
        x = _f64(x)
        out = np.zeros((self.batch, self.dims.query_heads, self.dims.head_size))
        self._check(lib().hx_harness_reference_f64(self._h, 0, x.ctypes.data_as(_dp), x.size, out.ctypes.data_as(_dp)))
        return out[0] if x.ndim == 1 and self.batch == 1 else out

    def append_projected(self, x):
        """DecodeHarness::append_projected (attention.hpp:531-539) (exact harness)."""
        x = _f64(x)
        self._check(lib().hx_append_projected_f64(self._h, 0, x.ctypes.data_as(_dp), x.size))

    # ShardedKVCache views (attention.hpp:286-309)
    def total_tokens(self, request=0):
        return lib().hx_total_tokens(self._h, 0, request)

    def effective_tokens(self, rank, request=0):
        return lib().hx_effective_tokens(self._h, 0, request, rank)

    def max_min_gap(self, request=0):
        return lib().hx_max_min_gap(self._h, 0, request)

    def context(self, rank, head, request=0):
        n = self.effective_tokens(rank, request)
        if self.exact:
            k, v = np.zeros((n, self.dims.head_size)), np.zeros((n, self.dims.head_size))
            self._check(lib().hx_read_kv_f64(self._h, 0, request, rank, head, k.ctypes.data_as(_dp),
                                             v.ctypes.data_as(_dp)))
            return k, v
        k = np.zeros((n, self.dims.head_size), dtype=np.float32)
        v = np.zeros((n, self.dims.head_size), dtype=np.float32)
        self._check(lib().hx_read_kv(self._h, 0, request, rank, head, k.ctypes.data_as(_fp), v.ctypes.data_as(_fp)))
        return k, v
