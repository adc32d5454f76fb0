"""The reference's analytic decode model, restated for the B200 measurements.

Algorithmic bytes of the decode path (roofline.hpp:17-48), the alpha-beta
collective costs and the fragment-exchange payload (comm.hpp:28-69), the
HOP-B batchwise overlap schedule (overlap.hpp:37-69) and the per-layer /
whole-model composition decode_ttl (latency.cpp:45-250). bench.py takes its
byte counts from here and tools/calibrate.py feeds a MEASURED HardwareSpec
through decode_ttl; tests/test_analytic.py pins every function against the
reference's own library (tests/golden/analytic.json, oracle/gen_analytic_golden.cpp).

Specs are the host mirror's dataclasses (model.py: ModelSpec, HardwareSpec,
ParallelismConfig); a workload is (batch, kv_seq_len).
"""
import math
from dataclasses import dataclass, field
from typing import List


def ceil_div(a, b):
    return -(-a // b)


def _k_eff(model):
    return 1 if model.attention == "mla" else model.kv_heads


def _kv_width(model):
    return model.kv_latent_dim if (model.attention == "mla" and model.kv_latent_dim > 0) else model.head_size


# ---------------------------------------------------------------- roofline.hpp:17-48
def kv_bytes(model, batch, seq, tpa, kvp, bytes_per_param):
    """KV bytes one GPU streams per layer: B * 2 * ceil(K/tpa) * Hsz_kv * S/kvp * b."""
    if tpa < 1 or kvp < 1:
        raise ValueError("tpa and kvp must be >= 1")
    return batch * 2.0 * ceil_div(_k_eff(model), tpa) * _kv_width(model) * (seq / kvp) * bytes_per_param


def weight_bytes(model, tpa, tpf, bytes_per_param):
    """Per-layer weight bytes per GPU: Q and O projections 2*H*(Q/tpa)*Hsz, K/V
    2*H*ceil(K/tpa)*Hsz_kv, gated FFN gate_factor*H*F/tpf."""
    if tpa < 1 or tpf < 1:
        raise ValueError("tpa and tpf must be >= 1")
    if model.query_heads % tpa:
        raise ValueError("tpa must divide query_heads")
    h = float(model.hidden_dim)
    attn = 2.0 * h * (model.query_heads // tpa) * model.head_size + \
        2.0 * h * ceil_div(_k_eff(model), tpa) * _kv_width(model)
    return (attn + model.ffn_gate_factor * h * model.ffn_dim / tpf) * bytes_per_param


def kv_read_time(model, batch, seq, tpa, kvp, hw):
    return kv_bytes(model, batch, seq, tpa, kvp, hw.bytes_per_param) / hw.mem_bw


def weight_read_time(model, tpa, tpf, hw):
    return weight_bytes(model, tpa, tpf, hw.bytes_per_param) / hw.mem_bw


# ---------------------------------------------------------------- comm.hpp:28-69
def comm_time(kind, group, payload, hw):
    """Alpha-beta cost on a switched domain; kind in all_to_all / all_reduce /
    all_gather / broadcast; payload = bytes each participant holds."""
    if group < 1:
        raise ValueError("group_size must be >= 1")
    if payload < 0:
        raise ValueError("payload must be >= 0 bytes")
    if group == 1:
        return 0.0
    g = float(group)
    wire = payload * (g - 1.0) / g / hw.link_bw
    if kind == "all_to_all":
        return hw.link_latency + wire
    if kind == "all_reduce":
        return hw.link_latency * 2.0 * (g - 1.0) + 2.0 * wire
    if kind == "all_gather":
        return hw.link_latency * (g - 1.0) + wire
    if kind == "broadcast":
        return hw.link_latency + payload / hw.link_bw
    raise ValueError(f"unknown collective {kind}")


def a2a_payload_per_destination(model, batch, kvp, tpa, hw):
    """Bytes one KVP rank ships to one peer: B * H/(kvp*tpa) * (1 + 1/Hsz) * b."""
    if kvp < 1 or tpa < 1:
        raise ValueError("kvp and tpa must be >= 1")
    if model.hidden_dim % (kvp * tpa):
        raise ValueError("kvp*tpa must divide hidden_dim")
    return batch * (model.hidden_dim / (kvp * tpa)) * (1.0 + 1.0 / model.head_size) * hw.bytes_per_param


def a2a_total_send_bytes(model, batch, kvp, tpa, hw):
    return a2a_payload_per_destination(model, batch, kvp, tpa, hw) * (kvp - 1)


# ---------------------------------------------------------------- overlap.hpp:37-69
@dataclass
class Timeline:
    requests: int
    compute: float
    comm: float
    enabled: bool
    comm_start: List[float] = field(default_factory=list)
    comm_end: List[float] = field(default_factory=list)
    total: float = 0.0


def hopb_schedule(requests, compute, comm, enabled):
    """R requests of `compute` then `comm` each. Off: back to back. On:
    request i's exchange starts at max(end of its compute, end of i-1's
    exchange) while compute runs densely -> total = max(R c + t, c + R t)."""
    if requests < 1:
        raise ValueError("requests must be >= 1")
    if compute < 0 or comm < 0:
        raise ValueError("per-request times must be >= 0")
    tl = Timeline(requests, compute, comm, enabled)
    prev = 0.0
    for i in range(requests):
        if enabled:
            ce = (i + 1) * compute
            start = ce if i == 0 else max(ce, prev)
        else:
            start = i * (compute + comm) + compute
        prev = start + comm
        tl.comm_start.append(start)
        tl.comm_end.append(prev)
    tl.total = tl.comm_end[-1]
    return tl


# ---------------------------------------------------------------- latency.cpp:45-250
@dataclass
class Breakdown:
    qkv_proj: float = 0.0
    kv_read: float = 0.0
    attn_compute: float = 0.0
    a2a_comm: float = 0.0
    a2a_exposed: float = 0.0
    post_proj: float = 0.0
    attn_allreduce: float = 0.0
    ffn_weight_read: float = 0.0
    ffn_compute: float = 0.0
    moe_comm: float = 0.0
    ttl: float = 0.0


def _require_valid(cfg, model, hw):
    from .model import validate_config
    model.validate()
    v = validate_config(cfg, model, hw)
    if not v:
        raise ValueError(f"invalid config {cfg}: {v.rule}")


def _att_batch(cfg, batch):
    return ceil_div(batch, cfg.stage_pool()) if cfg.strategy == "ep_dp" else batch


def _roof(mem_s, flops, hw):
    return max(mem_s, flops / hw.compute_throughput)


def attention_phase(cfg, model, batch, seq, hw):
    _require_valid(cfg, model, hw)
    out = Breakdown()
    dp = cfg.strategy == "ep_dp"
    b = _att_batch(cfg, batch)
    h = float(model.hidden_dim)
    cols = (model.query_heads // cfg.tpa) * model.head_size + 2.0 * ceil_div(_k_eff(model), cfg.tpa) * _kv_width(model)
    out.qkv_proj = _roof(h * cols * hw.bytes_per_param / hw.mem_bw, 2.0 * b * h * cols, hw)
    out.kv_read = kv_read_time(model, b, seq, cfg.tpa, cfg.kvp, hw)
    # one query per KV head (latency.cpp:69-73 -- the reference's model; MLA's 128 heads are not counted)
    out.attn_compute = 2.0 * b * 2.0 * ceil_div(_k_eff(model), cfg.tpa) * _kv_width(model) * (seq / cfg.kvp) / \
        hw.compute_throughput
    if cfg.kvp > 1:
        per = a2a_payload_per_destination(model, batch, cfg.kvp, cfg.tpa, hw)
        out.a2a_comm = comm_time("all_to_all", cfg.kvp, per * cfg.kvp, hw)
    out.a2a_exposed = out.a2a_comm
    rows = h if dp else h / cfg.stage_pool()
    out.post_proj = _roof(rows * h * hw.bytes_per_param / hw.mem_bw, 2.0 * b * rows * h, hw)
    if not dp:
        out.attn_allreduce = comm_time("all_reduce", cfg.stage_pool(), batch * h * hw.bytes_per_param, hw)
    return out


def expected_activated_experts(moe, ep, batch):
    """E_local * (1 - (1 - 1/E)^(B k)) under uniform routing (latency.cpp:34-41)."""
    return (moe.total_experts // ep) * (1.0 - math.pow(1.0 - 1.0 / moe.total_experts,
                                                       batch * moe.active_experts_per_token))


def ffn_phase(cfg, model, batch, hw):
    _require_valid(cfg, model, hw)
    if batch < 1:
        raise ValueError("batch must be >= 1")
    out = Breakdown()
    h, b, gate, nb = float(model.hidden_dim), float(batch), float(model.ffn_gate_factor), hw.bytes_per_param
    act = b * h * nb
    if model.moe:
        m = model.moe
        fe, fs, tpf = float(m.expert_ffn_dim), float(m.shared_expert_ffn_dim), float(cfg.tpf)
        active = expected_activated_experts(m, cfg.ep, batch)
        out.ffn_weight_read = (active * gate * h * fe / tpf + gate * h * fs / tpf) * nb / hw.mem_bw
        pairs = b * m.active_experts_per_token / cfg.ep
        out.ffn_compute = (gate * 2.0 * pairs * h * fe / tpf + gate * 2.0 * b * h * fs / tpf) / hw.compute_throughput
        local = b * h * (cfg.ep - 1) / hw.compute_throughput if cfg.ep > 1 else 0.0
        out.moe_comm = comm_time("all_reduce", cfg.tpf, act, hw) + comm_time("all_gather", cfg.ep, act, hw) + local
    else:
        f, tpf = float(model.ffn_dim), float(cfg.tpf)
        out.ffn_weight_read = gate * h * f / tpf * nb / hw.mem_bw
        out.ffn_compute = gate * 2.0 * b * h * f / tpf / hw.compute_throughput
        out.moe_comm = comm_time("all_reduce", cfg.tpf, act, hw)
    return out


def per_gpu_memory_bytes(cfg, model, batch, seq, hw):
    _require_valid(cfg, model, hw)
    dp = cfg.strategy == "ep_dp"
    h = float(model.hidden_dim)
    params = h * (model.query_heads // cfg.tpa) * model.head_size + \
        2.0 * h * ceil_div(_k_eff(model), cfg.tpa) * _kv_width(model) + (h if dp else h / cfg.stage_pool()) * h
    gate = float(model.ffn_gate_factor)
    if model.moe:
        m = model.moe
        params += (m.total_experts // cfg.ep) * gate * h * m.expert_ffn_dim / cfg.tpf
        params += gate * h * m.shared_expert_ffn_dim / cfg.tpf
    else:
        params += gate * h * model.ffn_dim / cfg.tpf
    heads = float(ceil_div(_k_eff(model), cfg.tpa))
    tokens = _att_batch(cfg, batch) * float(seq) if dp else batch * (seq / cfg.kvp)
    kv = 2.0 * heads * _kv_width(model) * tokens
    return (params + kv) * (model.layers / cfg.pp) * hw.bytes_per_param


def decode_ttl(cfg, model, batch, seq, hw, hopb=True):
    """Whole-model time per decode step; fields are per-layer times as composed."""
    out = attention_phase(cfg, model, batch, seq, hw)
    ffn = ffn_phase(cfg, model, batch, hw)
    out.ffn_weight_read, out.ffn_compute, out.moe_comm = ffn.ffn_weight_read, ffn.ffn_compute, ffn.moe_comm
    attn_core = max(out.kv_read, out.attn_compute)
    ffn_core = max(out.ffn_weight_read, out.ffn_compute)
    r = float(batch)
    if hopb and cfg.strategy != "medha_kvp":
        out.a2a_exposed = max(0.0, hopb_schedule(batch, attn_core / r, out.a2a_comm / r, True).total - attn_core)
        out.attn_allreduce = max(0.0, hopb_schedule(batch, out.post_proj / r, out.attn_allreduce / r, True).total -
                                 out.post_proj)
    layer = out.qkv_proj + attn_core + out.a2a_exposed + out.post_proj + out.attn_allreduce + ffn_core + out.moe_comm
    act = r * model.hidden_dim * hw.bytes_per_param
    p2p = (cfg.pp - 1) * (hw.link_latency + act / hw.link_bw)
    out.ttl = model.layers * layer + p2p + comm_time("broadcast", cfg.kvp, act, hw)
    return out
