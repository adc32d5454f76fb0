"""Decoder stack on the GPU + the reference's model/preset surface.

ModelSpec mirrors helixsim::ModelSpec (types.hpp:27-52) with the same strict
JSON schema as model_from_json / to_json (presets.cpp:96-163: snake_case keys,
unknown keys rejected, the error names the key). HelixDecoder runs the full
decode step (embedding -> L x [RMSNorm, Helix attention, O-proj, RMSNorm,
SwiGLU FFN] -> RMSNorm -> LM head -> greedy token) defined in
oracle/layer_oracle.hpp, entirely in libhelix_b200.so.
"""
import ctypes as C
import json
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from ._lib import ModelConfig, check, lib
from .exact import _Engine, _f32

_ip = C.POINTER(C.c_int32)
_fp = C.POINTER(C.c_float)


class ConfigError(RuntimeError):
    """presets.hpp:16-18 -- configuration-file problem (distinct from validation)."""


@dataclass
class MoESpec:
    total_experts: int = 0
    active_experts_per_token: int = 0
    expert_ffn_dim: int = 0
    shared_expert_ffn_dim: int = 0


@dataclass
class ModelSpec:
    name: str = ""
    layers: int = 0
    hidden_dim: int = 0
    query_heads: int = 0
    kv_heads: int = 0
    head_size: int = 0
    ffn_dim: int = 0
    ffn_gate_factor: int = 3
    attention: str = "gqa"
    kv_latent_dim: int = 0
    moe: Optional[MoESpec] = None
    vocab: int = 128256  # not part of the reference schema (it has no LM head); builder extension

    def validate(self):
        """ModelSpec::validate (types.cpp:16-44)."""
        def req(c, m):
            if not c:
                raise ValueError(m)
        req(self.layers >= 1, "layers must be >= 1")
        req(self.hidden_dim >= 1, "hidden_dim must be >= 1")
        req(self.query_heads >= 1, "query_heads must be >= 1")
        req(self.kv_heads >= 1, "kv_heads must be >= 1")
        req(self.head_size >= 1, "head_size must be >= 1")
        req(self.ffn_dim >= 1, "ffn_dim must be >= 1")
        req(self.ffn_gate_factor >= 1, "ffn_gate_factor must be >= 1")
        req(self.hidden_dim == self.query_heads * self.head_size, "hidden_dim must equal query_heads * head_size")
        if self.attention == "gqa":
            req(self.query_heads % self.kv_heads == 0, "query_heads must be a multiple of kv_heads")
            req(self.kv_latent_dim == 0, "kv_latent_dim is only meaningful for MLA")
        else:
            req(self.kv_heads == 1, "MLA keeps a single latent KV head")
            req(self.kv_latent_dim >= 0, "kv_latent_dim must be >= 0")
        if self.moe:
            m = self.moe
            req(m.total_experts >= 1, "moe.total_experts must be >= 1")
            req(m.active_experts_per_token >= 1, "moe.active_experts_per_token must be >= 1")
            req(m.active_experts_per_token <= m.total_experts,
                "moe.active_experts_per_token must not exceed moe.total_experts")
            req(m.expert_ffn_dim >= 1, "moe.expert_ffn_dim must be >= 1")
            req(m.shared_expert_ffn_dim >= 0, "moe.shared_expert_ffn_dim must be >= 0")

    def to_json(self):
        j = {"name": self.name, "layers": self.layers, "hidden_dim": self.hidden_dim,
             "query_heads": self.query_heads, "kv_heads": self.kv_heads, "head_size": self.head_size,
             "ffn_dim": self.ffn_dim, "ffn_gate_factor": self.ffn_gate_factor, "attention": self.attention,
             "kv_latent_dim": self.kv_latent_dim}
        if self.moe:
            j["moe"] = dict(self.moe.__dict__)
        return j

    @staticmethod
    def from_json(j):
        """model_from_json (presets.cpp:126-163): strict schema."""
        where = "model config"
        if not isinstance(j, dict):
            raise ConfigError(f"{where}: expected a JSON object")
        allowed = {"name", "layers", "hidden_dim", "query_heads", "kv_heads", "head_size", "ffn_dim",
                   "ffn_gate_factor", "attention", "kv_latent_dim", "moe"}
        for k in j:
            if k not in allowed:
                raise ConfigError(f"{where}: unknown key '{k}'")

        def geti(key, default=None):
            if key not in j:
                if default is not None:
                    return default
                raise ConfigError(f"{where}: missing field '{key}'")
            v = j[key]
            if not isinstance(v, int) or isinstance(v, bool):
                raise ConfigError(f"{where}: field '{key}' must be an integer")
            return v
        if "name" not in j:
            raise ConfigError(f"{where}: missing field 'name'")
        if not isinstance(j["name"], str):
            raise ConfigError(f"{where}: field 'name' must be a string")
        att = j.get("attention", "gqa")
        if att not in ("gqa", "mla"):
            raise ConfigError(f"{where}: field 'attention' must be \"gqa\" or \"mla\"")
        m = ModelSpec(name=j["name"], layers=geti("layers"), hidden_dim=geti("hidden_dim"),
                      query_heads=geti("query_heads"), kv_heads=geti("kv_heads"), head_size=geti("head_size"),
                      ffn_dim=geti("ffn_dim"), ffn_gate_factor=geti("ffn_gate_factor", 3), attention=att,
                      kv_latent_dim=geti("kv_latent_dim", 0))
        if "moe" in j:
            mj = j["moe"]
            mw = "model config.moe"
            if not isinstance(mj, dict):
                raise ConfigError(f"{mw}: expected a JSON object")
            for k in mj:
                if k not in MoESpec.__dataclass_fields__:
                    raise ConfigError(f"{mw}: unknown key '{k}'")
            m.moe = MoESpec(**{k: int(mj[k]) for k in mj})
        return m


PRESETS = {
    # reference presets (presets.cpp:11-44, presets/*.json)
    "llama405b-like": ModelSpec("llama405b-like", 126, 16384, 128, 8, 128, 65536, 3, "gqa", 0),
    "deepseek-r1-like": ModelSpec("deepseek-r1-like", 61, 16384, 128, 1, 128, 18432, 3, "mla", 288,
                                  MoESpec(256, 8, 2048, 2048)),
    # builder presets (the reference ships no tiny preset)
    "tiny-gqa": ModelSpec("tiny-gqa", 2, 64, 8, 4, 8, 128, 3, "gqa", 0, vocab=256),
    "llama3-8b-like": ModelSpec("llama3-8b-like", 32, 4096, 32, 8, 128, 14336, 3, "gqa", 0, vocab=128256),
}


def load_model(name_or_path):
    """load_model (presets.cpp:246-252): preset name, else a JSON file path."""
    if name_or_path in PRESETS:
        m = PRESETS[name_or_path]
    else:
        try:
            with open(name_or_path) as f:
                j = json.load(f)
        except OSError as e:
            raise ConfigError(f"cannot open model config '{name_or_path}': {e}")
        except json.JSONDecodeError as e:
            raise ConfigError(f"malformed JSON in '{name_or_path}': {e}")
        m = ModelSpec.from_json(j)
    m.validate()
    return m


# --------------------------------------------------------------------------- hardware / parallelism
@dataclass
class HardwareSpec:
    """helixsim::HardwareSpec (types.hpp:56-67); JSON keys as hardware_to_json
    (presets.cpp:115-124). The b200-measured preset carries this pod's measured
    copy bandwidth and sustained bf16 throughput (MEASURED_PEAKS.json) at bf16."""
    name: str = ""
    mem_bw: float = 8.0e12
    compute_throughput: float = 5.0e15
    link_bw: float = 9.0e11
    link_latency: float = 1.0e-7
    max_gpus: int = 64
    bytes_per_param: float = 0.5
    dram_capacity: float = 192.0e9

    _KEYS = {"name": "name", "mem_bw_bytes_per_s": "mem_bw", "compute_flops": "compute_throughput",
             "link_bw_bytes_per_s": "link_bw", "link_latency_s": "link_latency", "max_gpus": "max_gpus",
             "bytes_per_param": "bytes_per_param", "dram_capacity_bytes": "dram_capacity"}

    def to_json(self):
        return {k: getattr(self, a) for k, a in self._KEYS.items()}

    @staticmethod
    def from_json(j):
        where = "hardware config"
        if not isinstance(j, dict):
            raise ConfigError(f"{where}: expected a JSON object")
        for k in j:
            if k not in HardwareSpec._KEYS:
                raise ConfigError(f"{where}: unknown key '{k}'")
        hw = HardwareSpec()
        for k, a in HardwareSpec._KEYS.items():
            if k not in j:
                raise ConfigError(f"{where}: missing field '{k}'")
            v = j[k]
            if a == "name":
                if not isinstance(v, str):
                    raise ConfigError(f"{where}: field '{k}' must be a string")
            elif a == "max_gpus":
                if isinstance(v, bool) or not isinstance(v, int):
                    raise ConfigError(f"{where}: field '{k}' must be an integer")
            elif isinstance(v, bool) or not isinstance(v, (int, float)):
                raise ConfigError(f"{where}: field '{k}' must be a number")
            setattr(hw, a, v)
        return hw


HARDWARE_PRESETS = {
    "gb200-like": HardwareSpec("gb200-like", 8e12, 5e15, 9e11, 1e-7, 64, 0.5, 192e9),  # presets.cpp:45-51
    # this pod's B200 at the precision this engine stores (bf16): MEASURED_PEAKS.json copy
    # bandwidth and sustained cuBLAS bf16; NVLink 5 at 900 GB/s per direction, 180 GB HBM3e
    "b200-measured": HardwareSpec("b200-measured", 6.5562e12, 1.393e15, 9e11, 1e-7, 8, 2.0, 180e9),
}


def load_hardware(name_or_path):
    """load_hardware (presets.cpp): preset name, else a JSON file path."""
    if name_or_path in HARDWARE_PRESETS:
        return HARDWARE_PRESETS[name_or_path]
    try:
        with open(name_or_path) as f:
            j = json.load(f)
    except OSError as e:
        raise ConfigError(f"cannot open hardware config '{name_or_path}': {e}")
    except json.JSONDecodeError as e:
        raise ConfigError(f"malformed JSON in '{name_or_path}': {e}")
    return HardwareSpec.from_json(j)


STRATEGIES = ("helix", "tp", "tp_pp", "ep_dp", "medha_kvp")  # strategy_name (types.cpp)


@dataclass
class ParallelismConfig:
    """helixsim::ParallelismConfig (types.hpp:84-102)."""
    strategy: str = "tp"
    tpa: int = 1
    kvp: int = 1
    tpf: int = 1
    ep: int = 1
    pp: int = 1

    def stage_pool(self):
        return self.tpf * self.ep if self.strategy == "ep_dp" else self.kvp * self.tpa

    def total_gpus(self):
        return self.stage_pool() * self.pp

    def __str__(self):
        return f"{self.strategy}(tpa={self.tpa},kvp={self.kvp},tpf={self.tpf},ep={self.ep},pp={self.pp})"

    def to_json(self):
        return {"strategy": self.strategy, "tpa": self.tpa, "kvp": self.kvp, "tpf": self.tpf, "ep": self.ep,
                "pp": self.pp}

    @staticmethod
    def from_json(j):
        where = "parallelism config"
        if not isinstance(j, dict):
            raise ConfigError(f"{where}: expected a JSON object")
        keys = ("strategy", "tpa", "kvp", "tpf", "ep", "pp")
        for k in j:
            if k not in keys:
                raise ConfigError(f"{where}: unknown key '{k}'")
        for k in keys:
            if k not in j:
                raise ConfigError(f"{where}: missing field '{k}'")
        if not isinstance(j["strategy"], str):
            raise ConfigError(f"{where}: field 'strategy' must be a string")
        if j["strategy"] not in STRATEGIES:
            raise ConfigError(f"{where}: field 'strategy' has unknown value '{j['strategy']}'")
        for k in keys[1:]:
            if isinstance(j[k], bool) or not isinstance(j[k], int):
                raise ConfigError(f"{where}: field '{k}' must be an integer")
        return ParallelismConfig(*(j[k] for k in keys))


@dataclass
class Validity:
    """types.hpp:105-110: validity is a value; `rule` names the first broken rule."""
    ok: bool = True
    rule: str = ""

    def __bool__(self):
        return self.ok


def validate_config(cfg, model, hw):
    """validate_config (types.cpp:86-141): the reference's rules, in its order and
    with its diagnostics (the first broken rule wins)."""
    def fail(rule):
        return Validity(False, rule)
    if min(cfg.tpa, cfg.kvp, cfg.tpf, cfg.ep, cfg.pp) < 1:
        return fail("all parallelism widths must be >= 1")
    if cfg.total_gpus() > hw.max_gpus:
        return fail("total GPUs exceed max_gpus")
    k_eff = 1 if model.attention == "mla" else model.kv_heads
    if cfg.strategy == "helix":
        if cfg.pp != 1:
            return fail("helix runs as a single pipeline stage")
        if cfg.tpa > k_eff:
            return fail("helix requires tpa <= effective KV heads")
        if cfg.kvp * cfg.tpa != cfg.tpf * cfg.ep:
            return fail("helix re-provisions one pool: kvp*tpa must equal tpf*ep")
    elif cfg.strategy in ("tp", "tp_pp"):
        if cfg.strategy == "tp" and cfg.pp != 1:
            return fail("tp has no pipeline stages")
        if cfg.kvp != 1:
            return fail("tp keeps the whole sequence per GPU (kvp=1)")
        if cfg.ep != 1:
            return fail("tp shards experts with tensor parallelism (ep=1)")
        if cfg.tpf != cfg.tpa:
            return fail("tp ties attention and FFN widths")
    elif cfg.strategy == "ep_dp":
        if cfg.tpa != 1 or cfg.kvp != 1:
            return fail("ep_dp replicates attention (tpa=1, kvp=1)")
    elif cfg.strategy == "medha_kvp":
        if cfg.tpf != cfg.tpa:
            return fail("medha_kvp keeps the FFN on the tpa group")
        if cfg.ep != 1:
            return fail("medha_kvp does not shard experts (ep=1)")
    if model.query_heads % cfg.tpa:
        return fail("tpa must divide query_heads")
    if cfg.strategy in ("helix", "medha_kvp") and model.hidden_dim % (cfg.kvp * cfg.tpa):
        return fail("kvp*tpa must divide hidden_dim")
    if model.moe is not None:
        m = model.moe
        if m.total_experts % cfg.ep:
            return fail("ep must divide total_experts")
        if m.expert_ffn_dim % cfg.tpf:
            return fail("tpf must divide expert_ffn_dim")
        if m.shared_expert_ffn_dim > 0 and m.shared_expert_ffn_dim % cfg.tpf:
            return fail("tpf must divide shared_expert_ffn_dim")
    else:
        if cfg.ep != 1:
            return fail("expert parallelism needs an MoE model")
        if model.ffn_dim % cfg.tpf:
            return fail("tpf must divide ffn_dim")
    return Validity()


class HelixDecoder(_Engine):
    """Full decode step of a decoder stack under Helix (tpa, kvp): GQA attention, or
    MLA (attention == "mla": one 2*kv_latent_dim-wide latent KV head, absorbed
    projections, tcgen05 attention kernel; oracle/layer_oracle.hpp).

    `layers`/`vocab` override the spec (layer slices, small vocab for tests).
    With `spec.moe` every layer's FFN is the routed MoE (top-k of total_experts,
    SwiGLU experts of expert_ffn_dim) plus a shared expert of
    shared_expert_ffn_dim (0: none); in a distributed pool the FFN runs on the
    re-provisioned ep x tpf grid (types.hpp:100), tpf = tpa*kvp/ep."""

    def __init__(self, spec, tpa=1, kvp=1, chunk_size=16, batch=8, capacity=4096, layers=None, vocab=None,
                 device=0, use_graphs=True, hopb=False, pool=0, rank=0, nccl_id=None, loopback=None, ep=1,
                 kv_dtype="bf16", w_dtype="bf16"):
        self.spec = spec
        self.layers = layers or spec.layers
        self.vocab = vocab or spec.vocab
        m = spec.moe
        mc = ModelConfig(hidden=spec.hidden_dim, query_heads=spec.query_heads, kv_heads=spec.kv_heads,
                         head_size=spec.head_size, ffn=m.shared_expert_ffn_dim if m else spec.ffn_dim,
                         layers=self.layers, vocab=self.vocab, attention_only=0,
                         n_experts=m.total_experts if m else 0, top_k=m.active_experts_per_token if m else 0,
                         expert_ffn=m.expert_ffn_dim if m else 0,
                         kv_latent=spec.kv_latent_dim if spec.attention == "mla" else 0)
        super().__init__(mc, tpa, kvp, chunk_size, batch, capacity, device, use_graphs=use_graphs, hopb=hopb,
                         pool=pool, rank=rank, nccl_id=nccl_id, loopback=loopback, ep=ep, kv_dtype=kv_dtype,
                         w_dtype=w_dtype)
        self.n_ranks = tpa * kvp if pool else 1
        self.rank = rank
        self.vocab_local = -(-self.vocab // self.n_ranks)

    @classmethod
    def from_config(cls, spec, cfg, hw=None, **kw):
        """Build from the reference's configuration objects: `cfg` must be a valid
        Helix layout (validate_config against `hw`, default b200-measured); the
        FFN runs on cfg.tpf x cfg.ep over the same pool (types.hpp:84-102)."""
        hw = hw or HARDWARE_PRESETS["b200-measured"]
        v = validate_config(cfg, spec, hw)
        if not v:
            raise ValueError(v.rule)
        if cfg.strategy != "helix":
            raise ValueError("the B200 decode engine runs the helix strategy")
        return cls(spec, tpa=cfg.tpa, kvp=cfg.kvp, ep=cfg.ep, **kw)

    def init_weights(self, seed, qkv="mt19937"):
        if qkv == "mt19937":
            self._check(lib().hx_init_weights_mt19937(self._h, seed))
        else:
            self._check(lib().hx_init_weights_hash(self._h, seed))

    def grow_random(self, layer, request, n, rng):
        self._check(lib().hx_grow_random(self._h, layer, request, n, rng._h))

    def fill_kv_hash(self, n, seed):
        self._check(lib().hx_fill_kv_hash(self._h, n, seed))

    def total_tokens(self, layer=0, request=0):
        return lib().hx_total_tokens(self._h, layer, request)

    def step(self, tokens, want_logits=False, want_hidden=False):
        t = np.ascontiguousarray(tokens, dtype=np.int32)
        if t.shape != (self.batch,):  # hx_decode_step reads exactly `batch` ids from the pointer
            raise ValueError(f"tokens must have shape ({self.batch},), got {t.shape}")
        nxt = np.zeros(self.batch, dtype=np.int32)
        logits = np.zeros((self.batch, self.vocab_local), dtype=np.float32) if want_logits else None
        hidden = np.zeros((self.layers + 1, self.batch, self.spec.hidden_dim), dtype=np.float32) \
            if want_hidden else None
        self._check(lib().hx_decode_step(self._h, t.ctypes.data_as(_ip), nxt.ctypes.data_as(_ip),
                                         logits.ctypes.data_as(_fp) if logits is not None else None,
                                         hidden.ctypes.data_as(_fp) if hidden is not None else None))
        return nxt, logits, hidden

    def step_device(self, tokens_ptr, next_ptr):
        self._check(lib().hx_decode_step_device(self._h, tokens_ptr, next_ptr))

    def synchronize(self):
        self._check(lib().hx_synchronize(self._h))

    def stream(self):
        return lib().hx_stream(self._h)


class Loopback:
    """In-process group of n ranks on one device (HX_POOL_LOOPBACK): one engine
    per host thread, collectives through device copies + a host barrier."""

    def __init__(self, n):
        h = C.c_void_p()
        check(lib().hx_loopback_create(n, C.byref(h)))
        self._h = h

    def __del__(self):
        try:
            lib().hx_loopback_destroy(self._h)
        except Exception:
            pass


def nccl_unique_id():
    """128-byte ncclUniqueId (rank 0 creates it; share it with the other ranks)."""
    buf = (C.c_char * 128)()
    check(lib().hx_nccl_get_unique_id(buf))
    return bytes(buf)
