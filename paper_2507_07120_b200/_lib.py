"""ctypes binding of libhelix_b200.so (include/helix_b200.h).

The CUDA library is the product: there is no CPU fallback. If the library is
missing the import fails loudly with the build command.
"""
import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
# HX_LIB_PATH: A/B measurement of another in-tree build (tools only)
LIB_PATH = os.environ.get("HX_LIB_PATH") or os.path.join(HERE, "libhelix_b200.so")

HX_OK, HX_ERR_INVALID, HX_ERR_CUDA, HX_ERR_NCCL, HX_ERR_STATE = 0, 1, 2, 3, 4

i64, u64, i32, dp, fp, vp = C.c_int64, C.c_uint64, C.c_int32, C.POINTER(C.c_double), C.POINTER(C.c_float), C.c_void_p


class ModelConfig(C.Structure):
    _fields_ = [("hidden", i64), ("query_heads", i64), ("kv_heads", i64), ("head_size", i64), ("ffn", i64),
                ("layers", i64), ("vocab", i64), ("attention_only", i32), ("reserved", i32),
                ("n_experts", i64), ("top_k", i64), ("expert_ffn", i64), ("kv_latent", i64)]


POOL_LOCAL, POOL_NCCL, POOL_LOOPBACK = 0, 1, 2


class ParallelConfig(C.Structure):
    _fields_ = [("tpa", i64), ("kvp", i64), ("chunk_size", i64), ("distributed", i32), ("rank", i32),
                ("nccl_unique_id", vp), ("loopback", vp), ("ep", i64)]


class RuntimeConfig(C.Structure):
    _fields_ = [("batch", i64), ("capacity_tokens", i64), ("device", i32), ("hopb", i32), ("use_graphs", i32),
                ("kv_dtype", i32), ("w_dtype", i32), ("reserved", i32)]


KV_DTYPES = {"bf16": 0, "fp8": 1, "fp8_e4m3": 1, "f64": 2, "fp4": 3, "fp4_e2m1": 3}
W_DTYPES = {"bf16": 0, "fp8": 1, "fp8_e4m3": 1, "fp4": 2, "fp4_e2m1": 2}


class EngineInfo(C.Structure):
    _fields_ = [("kv_bytes_per_layer", i64), ("weight_bytes_per_layer", i64), ("head_bytes", i64),
                ("attn_streams", i64), ("attn_splits", i64), ("attn_items", i64), ("attn_grid", i64),
                ("kernels_per_step", i64), ("page_cap", i64), ("head_dim_padded", i64), ("kv_dtype", i64),
                ("w_dtype", i64), ("comm_ranks", i64), ("nccl_version", i64),
                ("exchange", i64)]


EXPORTS = {
    "hx_version": (C.c_char_p, []),
    "hx_last_error": (C.c_char_p, [vp]),
    "hx_engine_create": (C.c_int, [C.POINTER(ModelConfig), C.POINTER(ParallelConfig), C.POINTER(RuntimeConfig),
                                   C.POINTER(vp)]),
    "hx_engine_destroy": (None, [vp]),
    "hx_engine_get_info": (C.c_int, [vp, C.POINTER(EngineInfo)]),
    "hx_init_weights_mt19937": (C.c_int, [vp, u64]),
    "hx_init_weights_hash": (C.c_int, [vp, u64]),
    "hx_rng_create": (C.c_int, [u64, C.POINTER(vp)]),
    "hx_rng_destroy": (None, [vp]),
    "hx_rng_unit_draw": (C.c_double, [vp]),
    "hx_grow_random": (C.c_int, [vp, i64, i64, i64, vp]),
    "hx_append_kv": (C.c_int, [vp, i64, i64, i64, fp, fp]),
    "hx_fill_kv_hash": (C.c_int, [vp, i64, u64]),
    "hx_total_tokens": (i64, [vp, i64, i64]),
    "hx_effective_tokens": (i64, [vp, i64, i64, i64]),
    "hx_max_min_gap": (i64, [vp, i64, i64]),
    "hx_read_kv": (C.c_int, [vp, i64, i64, i64, i64, fp, fp]),
    "hx_harness_step": (C.c_int, [vp, i64, fp, i64, fp, fp]),
    "hx_harness_step_device": (C.c_int, [vp, i64, vp, vp]),
    "hx_decode_step": (C.c_int, [vp, C.POINTER(C.c_int32), C.POINTER(C.c_int32), fp, fp]),
    "hx_decode_step_device": (C.c_int, [vp, vp, vp]),
    "hx_synchronize": (C.c_int, [vp]),
    "hx_profile_step": (C.c_int, [vp, i64, dp]),
    "hx_stream": (vp, [vp]),
    "hx_transcript_size": (i64, [vp]),
    "hx_transcript": (C.c_int, [vp, C.POINTER(C.c_int64)]),
    "hx_clear_transcript": (C.c_int, [vp]),
    "hx_nccl_get_unique_id": (C.c_int, [vp]),
    "hx_loopback_create": (C.c_int, [i32, C.POINTER(vp)]),
    "hx_exchange_layout": (i64, [i64, i64, i64, C.POINTER(i64)]),
    "hx_engine_set_flag": (C.c_int, [vp, i32, i32]),
    "hx_moe_active_experts": (i64, [vp]),
    "hx_loopback_destroy": (None, [vp]),
    "hx_harness_step_f64": (C.c_int, [vp, i64, dp, i64, dp, dp]),
    "hx_harness_reference_f64": (C.c_int, [vp, i64, dp, i64, dp]),
    "hx_append_projected_f64": (C.c_int, [vp, i64, dp, i64]),
    "hx_append_kv_f64": (C.c_int, [vp, i64, i64, i64, dp, dp]),
    "hx_read_kv_f64": (C.c_int, [vp, i64, i64, i64, i64, dp, dp]),
    "hx_attention_f64": (C.c_int, [dp, i64, dp, dp, i64, i64, dp, dp]),
    "hx_merge_f64": (C.c_int, [i64, i64, dp, dp, dp, dp]),
}

_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: build it with `python -m paper_2507_07120_b200.build` "
                "(the B200 path has no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in EXPORTS.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


class HelixError(RuntimeError):
    pass


class CudaError(HelixError):
    pass


def check(rc, engine=None):
    if rc == HX_OK:
        return
    msg = lib().hx_last_error(engine).decode()
    if rc == HX_ERR_INVALID:
        raise ValueError(msg)  # the reference throws std::invalid_argument here
    if rc == HX_ERR_CUDA:
        raise CudaError(msg)
    raise HelixError(msg)
