#!/usr/bin/env python
"""Helix decode-step benchmark (driver contract: one JSON line on rank 0).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Workload (BASELINE.json configs[1]): Llama-3-8B-shaped GQA decoder
(H=4096, Q=32, K=8, Hsz=128, F=14336, 32 layers, vocab 128256), batch 8,
131072-token synthetic KV per request, one B200, KVP=1. A step is one full
decode step of the stack (embedding -> 32 x [RMSNorm, QKV+append, Helix
attention, O-proj, RMSNorm, SwiGLU FFN] -> LM head -> greedy token) for all
8 requests; metric = tokens/s (aggregate) and TTL ms/token (= ms_per_step).
Synthetic bf16 weights/KV from the counter hash; KV per layer (4.3 GB) far
exceeds L2, so no flush is needed between steps.

`--impl reference` times the reference's own CPU implementation of the path
(DecodeHarness<double>::step, attention.hpp:460-510, built from /root/reference
sources into oracle/_ref/ref_bench) on the host cores with all threads.
"""
import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "TTL ms/token and tokens/s/GPU at 1M-token KV, KVP=1/2/4/8 on B200"
UNIT = "tokens/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--layers", type=int, default=32)
    ap.add_argument("--batch", type=int, default=8)
    ap.add_argument("--context", type=int, default=131072, help="KV tokens per request per GPU")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-context", type=int, default=131072,
                    help="context of the 1-thread cpu_baseline sample in our arm's line")
    ap.add_argument("--ref-context", type=int, default=32768,
                    help="context of the --impl reference sample (all host threads; scaled to the workload)")
    ap.add_argument("--profile-only", action="store_true", help="skip timing loops (for ncu)")
    ap.add_argument("--no-fp8", action="store_true", help="skip the FP8-KV variant of the headline workload")
    ap.add_argument("--no-slices", action="store_true",
                    help="skip the one-GPU-of-8 slices (C3 llama405b-like, C4 deepseek-r1-like)")
    ap.add_argument("--slice-context", type=int, default=125000,
                    help="KV tokens per request on this GPU for the slices (1M context / KVP 8)")
    return ap.parse_args()


def config_dict(a, n):
    return {"workload": "llama3-8b-shaped GQA decode (H=4096 Q=32 K=8 Hsz=128 F=14336 V=128256), "
                        f"{a.layers} layers, batch {a.batch}, {a.context} KV tokens/request/GPU, KVP={n}",
            "model": "llama3-8b-like", "global_batch": a.batch, "seq_len": a.context * n,
            "layers": a.layers, "parallelism": f"helix tpa=1 kvp={n} tpf={n}",
            "l2": "no flush needed: per-layer KV (4.3 GB) >> 126 MB L2"}


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    def __init__(self):
        self.samples = []
        self.proc = None

    def __enter__(self):
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={q}", "--format=csv,noheader,nounits",
                                          "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.samples.append([x.strip() for x in line.split(",")])

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self, device=0):
        rows = [r for r in self.samples if len(r) >= 9 and r[0] == str(device)]
        if not rows:
            return None
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        reasons = set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            for name, v in zip(names, r[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": float(rows[0][2]),
                "reasons": sorted(reasons), "samples": len(rows)}


def step_bytes_per_gpu(spec, batch, seq_global, kvp, layers, kv_elem=2, w_elem=2):
    """Algorithmic HBM bytes one GPU of a TPA = 1 x KVP = kvp Helix pool (TPF = kvp)
    streams for `layers` layers: KV = the reference's kv_read_time x mem_bw
    (roofline.hpp:17-27); weights = weight_read_time x mem_bw (roofline.hpp:33-48:
    QKV replicated per KVP rank, FFN over TPF) with the O-projection sharded over
    the pool as latency.cpp:85-94 has it (the roofline header counts it whole).
    Pinned to the reference's library by tests/test_analytic.py."""
    from paper_2507_07120_b200 import analytic as A
    kv = A.kv_bytes(spec, batch, seq_global, 1, kvp, kv_elem) * layers
    o_full = spec.hidden_dim * spec.query_heads * spec.head_size * w_elem
    w = (A.weight_bytes(spec, 1, kvp, w_elem) - o_full + o_full / kvp) * layers
    return kv, w


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return p["hbm_gbs"], "measured"
    except Exception:
        return 6650.0, "fallback"


def peak_tensor():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return p["bf16_tflops_sustained"], "measured (sustained)"
    except Exception:
        return 1393.0, "fallback"


def pool_slice(a, preset, S, ep, w_dtype="bf16", kv_dtype="bf16"):
    """One GPU of an N=8 Helix pool (TPA=1, KVP=8; FFN TPF=8, or EP=8 x TPF=1 for
    MoE) measured alone: rank 0 of an 8-rank loopback pool with the collectives
    switched off (a single B200 here), so the number is this GPU's compute per
    layer over its B x S-token KV shard; the reference's NVLink terms
    (latency.cpp:77-146) are not included. C3 = llama405b-like, C4 =
    deepseek-r1-like."""
    import ctypes
    import numpy as np
    import torch
    import paper_2507_07120_b200 as P
    from paper_2507_07120_b200.model import Loopback
    spec = P.model.PRESETS[preset]
    B, N, V = a.batch, 8, 4096
    mla = spec.attention == "mla"
    lb = Loopback(N)
    eng = P.HelixDecoder(spec, tpa=1, kvp=N, batch=B, capacity=S * N + 64 * N, layers=1, vocab=V,
                         use_graphs=True, pool=2, rank=0, loopback=lb, ep=ep, w_dtype=w_dtype, kv_dtype=kv_dtype)
    # HX_FLAG_SKIP_COMM: no a2a / all-reduce (no peers here) -- the step is then
    # CUDA-graph captured like the headline (and like the NCCL pool)
    P._lib.check(P.lib().hx_engine_set_flag(eng._h, 1, 3), eng._h)
    eng.init_weights(2507, qkv="hash")
    eng.fill_kv_hash(S * N, 2507)  # rank 0 keeps S of the S*N global tokens
    s_loc = int(P.lib().hx_effective_tokens(eng._h, 0, 0, 0))
    g = torch.Generator().manual_seed(7)
    host_tok = torch.randint(0, V, (B,), dtype=torch.int32, generator=g)
    tok = host_tok.cuda()
    nxt = torch.zeros(B, dtype=torch.int32, device="cuda")
    for _ in range(a.warmup):
        eng.step_device(tok.data_ptr(), nxt.data_ptr())
    eng.step(host_tok.numpy())  # the profile pass below replays these (distinct) request tokens
    eng.synchronize()
    prof = np.zeros(10)
    reps = max(3, a.steps)
    P.lib().hx_profile_step(eng._h, reps, prof.ctypes.data_as(ctypes.POINTER(ctypes.c_double)))
    eng.synchronize()
    # timed steps (eager; CUDA events on the engine stream)
    stream = torch.cuda.ExternalStream(eng.stream())
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(stream)
    for _ in range(a.steps):
        eng.step_device(tok.data_ptr(), nxt.data_ptr())
    e1.record(stream)
    e1.synchronize()
    ms = e0.elapsed_time(e1) / a.steps
    info = eng.info()
    att_ms = prof[2]
    H, Q, Hsz = spec.hidden_dim, spec.query_heads, spec.head_size
    hbm, _ = peaks()
    out = {"ms_per_layer": ms, "graph_replay": True, "kv_tokens_per_request_on_this_gpu": s_loc,
           "breakdown_ms": {k: float(v) for k, v in zip(
               ["embed", "qkv", "attention", "split_reduce", "o_proj", "gate_up_or_router_to_gate_up",
                "down_or_down_combine", "lm_head", "merge"], prof)}}
    if mla:
        active = int(P.lib().hx_moe_active_experts(eng._h))
        f8 = kv_dtype == "fp8"
        kv_bytes = B * s_loc * 576 * (1 if f8 else 2)
        flops = B * s_loc * Q * (576 + 512) * 2
        tc, tc_kind = peak_tensor()
        if f8:  # kind::f8f6f4 issues at twice the kind::f16 rate (B200 dense fp8 = 2x bf16)
            tc, tc_kind = 2 * tc, "2x " + tc_kind + " bf16 (fp8 rate)"

        out["workload"] = ("deepseek-r1-like layer, one GPU of KVP=8 x EP=8 (tpf=1): 128 heads x %d latent tokens x "
                           "B=%d; 32/256 experts top-8 + shared 2048/8; collectives off (1 GPU)" % (s_loc, B))
        out["mla_attention"] = {
            "kernel": ("mla_decode_kernel<fp8> (tcgen05 kind::f8f6f4 cta_group::2, e4m3 latents / q / P"
                       if f8 else "mla_decode_kernel (tcgen05 cta_group::2 CTA pair") +
                      ", TMEM accumulators, 2-SM TMA)",
            "launch_ms": att_ms, "algorithmic_kv_bytes": kv_bytes, "algorithmic_flops": flops,
            "roofline": {"bound": "tensor", "achieved": flops / (att_ms * 1e-3) / 1e12, "peak": tc,
                         "unit": "TFLOP/s", "frac": flops / (att_ms * 1e-3) / 1e12 / tc, "peak_kind": tc_kind,
                         "hbm_achieved_gbs": kv_bytes / (att_ms * 1e-3) / 1e9,
                         "hbm_frac": kv_bytes / (att_ms * 1e-3) / 1e9 / hbm,
                         "t_roof_ms": max(kv_bytes / hbm / 1e6, flops / tc / 1e9),
                         "traffic": ncu_traffic("mla_fp8" if f8 else "mla")}}
        out["moe"] = {"local_experts": spec.moe.total_experts // ep, "active_local_experts_last_step": active,
                      "expert_bytes_streamed": active * 3 * H * spec.moe.expert_ffn_dim * W_ELEM_BYTES[w_dtype]}
    else:
        K = spec.kv_heads
        ekv, ew = KV_ELEM_BYTES[kv_dtype], W_ELEM_BYTES[w_dtype]
        # roofline.hpp:17-48: QKV duplicated per KVP rank, O and FFN sharded over N
        kv_bytes, w_bytes = step_bytes_per_gpu(spec, B, s_loc * N, N, 1, ekv, ew)
        out["workload"] = ("llama405b-like layer, one GPU of TPA=1 x KVP=8 (TPF=8): %d KV heads x %d tokens x B=%d; "
                           "QKV replicated, W_O rows and FFN features 1/8; collectives off (1 GPU)" % (K, s_loc, B))
        out["attention"] = {
            "kernel": {"fp8": "attn_decode_kernel<128,12,2,2,fp8,W16>", "fp4": "attn_decode_kernel<128,12,3,2,fp4,W16>",
                       "bf16": "attn_decode_kernel<128,8,2,2,W16>"}[kv_dtype]
                      + " (TMA bulk-copy page ring, mma.sync)", "launch_ms": att_ms,
            "algorithmic_kv_bytes": kv_bytes,
            "roofline": {"bound": "hbm", "achieved": kv_bytes / (att_ms * 1e-3) / 1e9, "peak": hbm, "unit": "GB/s",
                         "frac": kv_bytes / (att_ms * 1e-3) / 1e9 / hbm,
                         "traffic": ncu_traffic("attention_405b_slice" + ("" if kv_dtype == "bf16" else "_" + kv_dtype))}}
        out["layer_roofline"] = {"bound": "hbm", "algorithmic_bytes": kv_bytes + w_bytes, "weight_bytes": w_bytes,
                                 "t_roof_ms": (kv_bytes + w_bytes) / hbm / 1e6,
                                 "achieved_gbs": (kv_bytes + w_bytes) / (ms * 1e-3) / 1e9,
                                 "frac": (kv_bytes + w_bytes) / (ms * 1e-3) / 1e9 / hbm}
        out["ttl_ms_extrapolated_126_layers"] = ms * spec.layers
    out["engine"] = info
    eng.close()
    return out


def kvp_slices(a):
    """configs[1]'s model at KVP = 2/4/8 (weak scaling: S tokens per request per
    GPU, global context S x KVP; TPF = KVP): ONE GPU of the pool measured alone
    -- rank 0 of a loopback pool with both collectives switched off (so the
    step is CUDA-graph captured like the headline) -- plus the pool's
    communication from the reference's alpha-beta model (comm.hpp:28-45;
    fp32 payloads as this engine sends them; gb200-like link 900 GB/s,
    0.1 us) for the combined HBM + NVLink figure. The real NCCL numbers come
    from `bench.py --gpus N` on an N-GPU box."""
    import torch
    import paper_2507_07120_b200 as P
    from paper_2507_07120_b200.model import Loopback
    spec = P.model.PRESETS["llama3-8b-like"]
    B, S, L = a.batch, a.context, a.layers
    H, Q, K, Hsz, F, V = spec.hidden_dim, spec.query_heads, spec.kv_heads, spec.head_size, spec.ffn_dim, spec.vocab
    hbm, _ = peaks()
    out = {}
    for n in (2, 4, 8):
        lb = Loopback(n)
        eng = P.HelixDecoder(spec, tpa=1, kvp=n, batch=B, capacity=S * n + 64 * n, layers=L, pool=2, rank=0,
                             loopback=lb, use_graphs=True)
        P._lib.check(P.lib().hx_engine_set_flag(eng._h, 1, 3), eng._h)
        eng.init_weights(2507, qkv="hash")
        eng.fill_kv_hash(S * n, 2507)
        tok = [torch.randint(0, V, (B,), dtype=torch.int32, device="cuda"),
               torch.zeros(B, dtype=torch.int32, device="cuda")]
        for i in range(a.warmup):
            eng.step_device(tok[i % 2].data_ptr(), tok[(i + 1) % 2].data_ptr())
        stream = torch.cuda.ExternalStream(eng.stream())
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(stream)
        for i in range(a.steps):
            eng.step_device(tok[i % 2].data_ptr(), tok[(i + 1) % 2].data_ptr())
        e1.record(stream)
        e1.synchronize()
        ms = e0.elapsed_time(e1) / a.steps
        s_loc = int(P.lib().hx_effective_tokens(eng._h, 0, 0, 0))
        eng.close()
        kv, w = step_bytes_per_gpu(spec, B, s_loc * n, n, L)
        w += (V // n) * H * 2  # LM-head rows of this rank
        # reference comm model per layer: all-to-all of the fragment slices + two TP all-reduces
        per_dest = B * H / n * (1 + 1 / Hsz) * 4
        a2a = 1e-7 + per_dest * n * (n - 1) / n / 9e11
        ar = 1e-7 * 2 * (n - 1) + 2 * (B * H * 4) * (n - 1) / n / 9e11
        comm_ms = (a2a + 2 * ar) * L * 1e3
        t_roof = (kv + w) / hbm / 1e6
        out[str(n)] = {"kv_tokens_per_request_per_gpu": s_loc, "global_context": s_loc * n,
                       "ttl_ms_compute": ms, "comm_ms_modeled": comm_ms, "ttl_ms_with_modeled_comm": ms + comm_ms,
                       "tokens_per_s_per_gpu": B / ((ms + comm_ms) * 1e-3) / n,
                       "hbm_bytes_per_gpu": kv + w, "t_roof_ms": t_roof + comm_ms,
                       "roofline_frac": (t_roof + comm_ms) / (ms + comm_ms)}
    return out


W_ELEM_BYTES = {"bf16": 2.0, "fp8": 1.0, "fp4": 17.0 / 32.0}  # fp4: e2m1 nibble + one exponent byte per 32 inputs
KV_ELEM_BYTES = {"bf16": 2.0, "fp8": 1.0, "fp4": 17.5 / 32.0}  # fp4: e2m1 nibble + a K exponent byte / V f16 scale per 32
KV_KERNEL = {"bf16": "attn_decode_kernel<128,7,3,1,bf16>", "fp8": "attn_decode_kernel<128,10,4,1,fp8>",
             "fp4": "attn_decode_kernel<128,12,4,1,fp4> (query image in shared memory)"}


def fp8_kv_line(a, w_dtype="bf16", kv_dtype="fp8"):
    """the configs[1] workload with FP8 (e4m3) KV pages
    (kv_dtype="fp8", attention MMAs in f16 on the exact widened values), and
    with w_dtype="fp8" also e4m3 GEMV weights (per-output power-of-two scales).
    Same timing method as the headline (graph replay, CUDA events on the engine
    stream); separate keys, never the headline number (the headline stores KV
    and weights in bf16)."""
    import ctypes
    import numpy as np
    import torch
    import paper_2507_07120_b200 as P
    spec = P.model.PRESETS["llama3-8b-like"]
    B, S, L = a.batch, a.context, a.layers
    eng = P.HelixDecoder(spec, tpa=1, kvp=1, batch=B, capacity=S + 4 * (a.warmup + a.steps + 16) + 64, layers=L,
                         kv_dtype=kv_dtype, w_dtype=w_dtype)
    eng.init_weights(2507, qkv="hash")
    eng.fill_kv_hash(S, 2507)
    stream = torch.cuda.ExternalStream(eng.stream())
    tok = [torch.randint(0, spec.vocab, (B,), dtype=torch.int32, device="cuda"),
           torch.zeros(B, dtype=torch.int32, device="cuda")]
    for i in range(a.warmup):
        eng.step_device(tok[i % 2].data_ptr(), tok[(i + 1) % 2].data_ptr())
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for i in range(a.steps):
        eng.step_device(tok[i % 2].data_ptr(), tok[(i + 1) % 2].data_ptr())
    e1.record(stream)
    e1.synchronize()
    ms = e0.elapsed_time(e1) / a.steps
    prof = np.zeros(10)
    P.lib().hx_profile_step(eng._h, 2, prof.ctypes.data_as(ctypes.POINTER(ctypes.c_double)))
    att = prof[2] / L
    s_now = eng.total_tokens(0, 0)
    kv_bytes = B * spec.kv_heads * s_now * spec.head_size * 2 * KV_ELEM_BYTES[kv_dtype]  # K+V, algorithmic
    hbm, _ = peaks()
    info = eng.info()
    eng.close()
    return {"kv_dtype": {"fp8": "fp8_e4m3", "fp4": "fp4_e2m1 (32-dim blocks, pow2 scales)"}[kv_dtype],
            "w_dtype": {"fp8": "fp8_e4m3", "fp4": "fp4_e2m1 (32-input blocks, pow2 scales)"}.get(w_dtype, "bf16"),
            "weight_bytes_resident": info["weight_bytes_per_layer"] * L + info["head_bytes"], "ms_per_step": ms, "value": B / (ms * 1e-3), "unit": UNIT,
            "breakdown_ms": {k: float(v) for k, v in zip(
                ["embed", "qkv", "attention", "split_reduce", "o_proj", "gate_up", "down", "lm_head", "merge"], prof)},
            "attention_roofline": {"bound": "hbm", "kernel": KV_KERNEL[kv_dtype],
                                   "algorithmic_bytes_per_launch": kv_bytes, "launch_ms": att,
                                   "achieved": kv_bytes / (att * 1e-3) / 1e9, "peak": hbm, "unit": "GB/s",
                                   "frac": kv_bytes / (att * 1e-3) / 1e9 / hbm,
                                   "traffic": ncu_traffic("attention_" + kv_dtype)},
            "kv_bytes_per_layer": info["kv_bytes_per_layer"]}


def ncu_traffic(key="attention"):
    """DRAM bytes per launch (read + write) of the kernel from the committed
    `ncu --set full` capture (profiles/ncu_summary.json), or None."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_summary.json")) as f:
            return json.load(f).get(key, {}).get("dram_bytes_per_launch")
    except Exception:
        return None


# ----------------------------------------------------------------------------- CPU reference
def run_ref_bench(threads, context, steps, warmup, layers, batch, kvp=1, context_full=None):
    """The reference's DecodeHarness<double>::step (oracle/_ref/ref_bench) on
    `threads` host threads, one request harness per thread, each step one layer's
    attention of every thread's request at `context` tokens over a KVP=`kvp`
    sharded cache. Returns the measured sample and the throughput it implies for
    the full workload (batch requests x `layers` layers x `context_full` tokens;
    attention cost is linear in the context -- acceptance.cpp:82-116)."""
    context_full = context_full or context
    exe = os.path.join(ROOT, "oracle", "_ref", "ref_bench")
    if os.path.exists(exe):
        out = subprocess.run([exe, "32", "8", "128", "1", str(kvp), str(context), str(steps), str(threads),
                              str(warmup)], capture_output=True, text=True, check=True).stdout
        r = json.loads(out.strip().splitlines()[-1])
        t = r["seconds_per_step_per_request"]
        wall_step = r["wall_s"] / max(1, steps)
        kind = "reference"
    else:
        # oracle port (clean-room restatement) when the reference could not be built
        from tests import oracle_py as O
        h = O.Harness(32, 8, 128, 1, kvp, 16, 42)
        h.grow_random(context, O.Rng(1000))
        x = O.Rng(7).draws(4096)
        for _ in range(warmup):
            h.step(x)
        t0 = time.time()
        for _ in range(steps):
            h.step(x)
        t = (time.time() - t0) / steps
        wall_step = t
        threads, kind = 1, "port"
    scale = context_full / context
    # request-layer attention steps per second at the sample context -> full decode steps
    tok_s = threads / (t * layers * scale)
    sample = (f"DecodeHarness<double>::step (attention.hpp:460-510), Q=32 K=8 Hsz=128 KVP={kvp}, {context}-token "
              f"context, {steps} timed steps after {warmup} warm-up, {threads} request harnesses on {threads} host "
              f"threads; one sample step = one layer's attention for each thread's request; throughput scaled x"
              f"{layers} layers" + (f" and x{scale:g} to the {context_full}-token context" if scale != 1 else "") +
              " (the reference has no O-proj/FFN/LM-head numerics, so the CPU figure covers attention only)")
    return {"value": tok_s, "unit": UNIT, "cores": threads, "kind": kind, "sample": sample,
            "seconds_per_request_layer_step": t, "sample_ms_per_step": wall_step * 1e3,
            "ms_per_full_step_extrapolated": batch / tok_s * 1e3}


def reference_arm(a):
    """--impl reference: the reference's own CPU path on this box's host cores,
    rank 0 only (other ranks exit without work), exactly --steps timed sample
    steps after --warmup untimed ones (run_ref_bench)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    n = a.gpus
    threads = os.cpu_count() or 1
    ctx_full = a.context * n
    ctx = min(ctx_full, a.ref_context)
    # bound memory: K and V doubles of 8 heads x 128 per token per request (+ chunk slack)
    try:
        mem = os.sysconf("SC_PAGE_SIZE") * os.sysconf("SC_PHYS_PAGES")
        threads = max(1, min(threads, int(mem * 0.5 // (ctx * 8 * 128 * 2 * 8 * 1.5))))
    except (ValueError, OSError):
        pass
    cb = run_ref_bench(threads, ctx, a.steps, a.warmup, a.layers, a.batch, kvp=n, context_full=ctx_full)
    line = {"metric": METRIC, "value": cb["value"], "unit": UNIT, "n_gpus": n, "steps": a.steps,
            "warmup": a.warmup, "ms_per_step": cb["sample_ms_per_step"],
            "ms_per_full_step_extrapolated": cb["ms_per_full_step_extrapolated"], "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": config_dict(a, n), "impl": "reference",
            "cpu_baseline": {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample")},
            "e2e": {"value": cb["value"], "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------- our arm
def ours(a):
    import numpy as np
    import torch
    import paper_2507_07120_b200 as P

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    dev = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(dev)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", dev))
    spec = P.model.PRESETS["llama3-8b-like"]
    B, S, L = a.batch, a.context, a.layers
    total_steps = 6 * (a.warmup + a.steps) + 8
    # weak scaling: S KV tokens per request per GPU; KVP = N (global context S*N)
    S_glob = S * world
    cap = S_glob + 4 * (total_steps + 8) * world + 64
    if world > 1:
        from paper_2507_07120_b200.model import nccl_unique_id
        uid = [nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        eng = P.HelixDecoder(spec, tpa=1, kvp=world, batch=B, capacity=cap, layers=L, device=dev, pool=1,
                             rank=rank, nccl_id=uid[0], hopb=False)  # HOP-B measured below (profiles/r01_hopb_sweep.md)
    else:
        eng = P.HelixDecoder(spec, tpa=1, kvp=1, batch=B, capacity=cap, layers=L, device=dev)
    eng.init_weights(2507, qkv="hash")
    eng.fill_kv_hash(S_glob, 2507)
    info = eng.info()
    stream = torch.cuda.ExternalStream(eng.stream())

    def barrier():
        torch.cuda.synchronize()
        if dist is not None:
            dist.barrier()

    def max_over_ranks(v):
        if dist is None:
            return v
        t = torch.tensor([v], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    tok = [torch.randint(0, spec.vocab, (B,), dtype=torch.int32, device="cuda"),
           torch.zeros(B, dtype=torch.int32, device="cuda")]

    def dev_step(i):
        eng.step_device(tok[i % 2].data_ptr(), tok[(i + 1) % 2].data_ptr())

    def timed(n_steps, offset):
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for i in range(n_steps):
            dev_step(offset + i)
        e1.record(stream)
        e1.synchronize()
        barrier()
        return max_over_ranks(e0.elapsed_time(e1) / n_steps)

    for i in range(a.warmup):
        dev_step(i)
    import ctypes
    with ClockSampler() as clk:
        time.sleep(0.3)
        ms = timed(a.steps, a.warmup)
        hopb = None
        if world > 1:
            # exposed KVP exchange per mode (overlap.hpp:37-69): same resident pool, runtime
            # switches; "no a2a" keeps every slice on its rank (measurement only)
            def setf(flag, v):
                P._lib.check(P.lib().hx_engine_set_flag(eng._h, flag, v), eng._h)
            off = a.warmup + a.steps

            def run_mode(collective, hopb_on, skip_a2a):
                setf(3, int(collective))
                setf(2, int(hopb_on))
                setf(1, int(skip_a2a))
                for i in range(a.warmup):
                    dev_step(off + i)
                return timed(a.steps, off + a.warmup)
            hopb = {"headline": "device exchange, HOP-B off (the line's ms_per_step)"}
            for name, coll, hb in (("collective_a2a", 1, 0), ("device", 0, 0), ("device_hopb", 0, 1)):
                with_x = ms if name == "device" else run_mode(coll, hb, 0)
                no_x = run_mode(coll, hb, 1)
                hopb[name] = {"ms_per_step": with_x, "ms_per_step_no_a2a": no_x,
                              "exposed_a2a_ms": max(0.0, with_x - no_x)}
            setf(1, 0)
            setf(2, 0)
            setf(3, 0)
            e_c, e_h = hopb["collective_a2a"]["exposed_a2a_ms"], hopb["device_hopb"]["exposed_a2a_ms"]
            hopb["hopb_hidden_frac_vs_collective"] = (1.0 - e_h / e_c) if e_c > 0 else None
            hopb["hopb_net_ms_vs_device"] = hopb["device"]["ms_per_step"] - hopb["device_hopb"]["ms_per_step"]
    clocks = clk.summary(dev)
    # e2e through the public API: pinned host tokens in, host next tokens out, every
    # step -- after the clock sampler has stopped: its nvidia-smi polling contends
    # with the synchronous per-step driver calls (+0.5-1 ms/step measured; the same
    # loop without it: tools/launch_cost.py, 22.73 vs 22.67 ms pipelined)
    h_tok = torch.zeros(B, dtype=torch.int32).pin_memory()
    h_next = torch.zeros(B, dtype=torch.int32).pin_memory()
    h_tok.copy_(tok[0].cpu())
    ip = ctypes.POINTER(ctypes.c_int32)
    # untimed warm-up of this call path too: its first call captures and uploads
    # the CUDA graph for the engine's own token buffers (tens of ms, once)
    for i in range(a.warmup):
        rc = P.lib().hx_decode_step(eng._h, ctypes.cast(h_tok.data_ptr(), ip), ctypes.cast(h_next.data_ptr(), ip),
                                    None, None)
        P._lib.check(rc, eng._h)
        h_tok.copy_(h_next)
    barrier()
    e2 = torch.cuda.Event(enable_timing=True)
    e3 = torch.cuda.Event(enable_timing=True)
    w0 = time.perf_counter()
    e2.record(stream)
    for i in range(a.steps):
        rc = P.lib().hx_decode_step(eng._h, ctypes.cast(h_tok.data_ptr(), ip), ctypes.cast(h_next.data_ptr(), ip),
                                    None, None)
        P._lib.check(rc, eng._h)
        h_tok.copy_(h_next)
    e3.record(stream)
    e3.synchronize()
    wall_e2e = (time.perf_counter() - w0) / a.steps * 1e3
    ms_e2e = max_over_ranks(max(e2.elapsed_time(e3) / a.steps, wall_e2e))

    # per-kernel-kind breakdown (eager launches, CUDA events on the engine stream)
    prof = np.zeros(10)
    P.lib().hx_profile_step(eng._h, 2, prof.ctypes.data_as(ctypes.POINTER(ctypes.c_double)))
    step_prof = prof.sum()
    attn_ms_launch = prof[2] / L
    s_now = eng.total_tokens(0, 0)
    attn_bytes = B * spec.kv_heads * s_now * spec.head_size * 2 * 2  # K+V bf16, algorithmic
    weight_bytes = info["weight_bytes_per_layer"] * L + info["head_bytes"] // 2  # LM head read; embedding gather ~0
    hbm_peak, peak_kind = peaks()
    achieved = attn_bytes / (attn_ms_launch * 1e-3) / 1e9
    step_bytes = attn_bytes * L + weight_bytes
    value = B / (ms * 1e-3)
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": a.steps, "warmup": a.warmup,
        "ms_per_step": ms, "ttl_ms": ms, "tokens_per_s_per_gpu": value / world, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
        "config": config_dict(a, world),
        "e2e": {"value": B / (ms_e2e * 1e-3), "unit": UNIT, "h2d_bytes_per_step": 4 * B, "d2h_bytes_per_step": 4 * B,
                "ms_per_step": ms_e2e},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": hbm_peak, "unit": "GB/s",
                     "frac": achieved / hbm_peak, "traffic": ncu_traffic(), "kernel": "attn_decode_kernel<128,7,3>",
                     "algorithmic_bytes_per_launch": attn_bytes, "launch_ms": attn_ms_launch, "peak_kind": peak_kind,
                     "step_hbm_frac": step_bytes / (ms * 1e-3) / 1e9 / hbm_peak,
                     "step_algorithmic_bytes": step_bytes},
        "breakdown_ms": {k: float(v) for k, v in zip(
            ["embed", "qkv", "attention", "split_reduce", "o_proj", "gate_up", "down", "lm_head", "merge"], prof)},
        "profile_step_ms": step_prof,
        "gpu_launches": int(info["kernels_per_step"]) * a.steps,
        "clocks": clocks,
        "engine": info,
    }
    if hopb is not None:
        line["hopb"] = hopb
    if world > 1:
        # one GPU of the KVP = N pool (TPA = 1, TPF = N): HBM bytes it reads per step and the
        # NVLink bytes it sends (fp32 fragment slices to N-1 peers, two ring all-reduces of the
        # [B x H] fp32 partials per layer, latency.cpp:77-146); combined roofline = HBM time at
        # the measured peak + NVLink time at 900 GB/s per direction, nothing overlapped
        H, Q, K, Hsz, F, V = (spec.hidden_dim, spec.query_heads, spec.kv_heads, spec.head_size, spec.ffn_dim,
                              spec.vocab)
        s_loc = int(P.lib().hx_effective_tokens(eng._h, 0, 0, rank % world))
        kv, w = step_bytes_per_gpu(spec, B, s_loc * world, world, L)
        w += (V // world) * H * 2  # LM-head rows of this rank
        xchunk = int(P.lib().hx_exchange_layout(Q, Hsz, world, None))
        a2a = (world - 1) * B * xchunk * 4 * L
        ar = 2 * (2 * (world - 1) / world * B * H * 4) * L
        t_hbm, t_nvl = (kv + w) / (hbm_peak * 1e9), (a2a + ar) / 900e9
        line["pool"] = {"kvp": world, "tpa": 1, "tpf": world, "comm_ranks": info["comm_ranks"],
                        "nccl_version": info["nccl_version"], "kv_tokens_per_request_per_gpu": s_loc,
                        "global_context": s_loc * world, "ttl_ms": ms, "tokens_per_s_per_gpu": value / world,
                        "hbm_bytes_per_gpu_per_step": kv + w, "nvlink_bytes_per_gpu_per_step": a2a + ar,
                        "t_roof_ms": (t_hbm + t_nvl) * 1e3, "roofline_frac": (t_hbm + t_nvl) * 1e3 / ms}
    if not a.no_cpu_baseline and rank == 0 and world == 1:
        try:
            cb = run_ref_bench(1, min(a.cpu_context, S), 2, 0, L, B, context_full=S)
            line["cpu_baseline"] = {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample")}
        except Exception as ex:  # reported, never fatal for the GPU number
            line["cpu_baseline"] = {"error": str(ex)[:200]}
    if world == 1 and not a.no_fp8:
        eng.close()  # free the 150 GB pool
        try:
            line["fp8_kv"] = fp8_kv_line(a)
        except Exception as ex:  # reported, never fatal for the headline number
            line["fp8_kv"] = {"error": str(ex)[:300]}
        try:
            line["fp8_kv_w"] = fp8_kv_line(a, w_dtype="fp8")
        except Exception as ex:  # reported, never fatal for the headline number
            line["fp8_kv_w"] = {"error": str(ex)[:300]}
        try:  # FP4 (e2m1) KV -- the paper's evaluation precision -- with FP8 weights
            line["fp4_kv_fp8_w"] = fp8_kv_line(a, w_dtype="fp8", kv_dtype="fp4")
        except Exception as ex:  # reported, never fatal for the headline number
            line["fp4_kv_fp8_w"] = {"error": str(ex)[:300]}
        try:  # the paper's setting: weights AND KV in FP4
            line["fp4_kv_fp4_w"] = fp8_kv_line(a, w_dtype="fp4", kv_dtype="fp4")
        except Exception as ex:  # reported, never fatal for the headline number
            line["fp4_kv_fp4_w"] = {"error": str(ex)[:300]}
    if world == 1 and not a.no_slices:
        eng.close()  # free the 150 GB pool before the 8-GPU-pool slices
        try:
            line["kvp_slices"] = kvp_slices(a)
        except Exception as ex:  # reported, never fatal for the headline number
            line["kvp_slices"] = {"error": str(ex)[:300]}
        for key, preset, ctx, ep, wd, kd in (
                ("llama405b_slice", "llama405b-like", a.slice_context, 1, "bf16", "bf16"),
                ("deepseek_slice", "deepseek-r1-like", a.slice_context, 8, "bf16", "bf16"),
                ("llama405b_slice_fp8w", "llama405b-like", a.slice_context, 1, "fp8", "bf16"),
                ("deepseek_slice_fp8w", "deepseek-r1-like", a.slice_context, 8, "fp8", "bf16"),
                ("llama405b_slice_fp8", "llama405b-like", a.slice_context, 1, "fp8", "fp8"),
                ("llama405b_slice_fp4", "llama405b-like", a.slice_context, 1, "fp8", "fp4"),
                ("llama405b_slice_fp4w", "llama405b-like", a.slice_context, 1, "fp4", "fp4"),
                ("deepseek_slice_fp4w", "deepseek-r1-like", a.slice_context, 8, "fp4", "bf16"),
                ("deepseek_slice_fp8", "deepseek-r1-like", a.slice_context, 8, "fp8", "fp8")):
            try:
                line[key] = pool_slice(a, preset, ctx, ep, wd, kd)
                line[key]["w_dtype"] = wd
                line[key]["kv_dtype"] = kd
            except Exception as ex:  # reported, never fatal for the headline number
                line[key] = {"error": str(ex)[:300]}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.barrier()
        eng.close()
        dist.destroy_process_group()


def relaunch_under_torchrun(a):
    """`python bench.py --gpus N` (N > 1) outside torchrun: launch the N ranks
    here, one process per GPU, exactly as the driver does (torch.distributed.run,
    127.0.0.1 rendezvous), with NCCL's init log on so every communicator's
    nranks is visible in stderr."""
    import socket
    import torch
    have = torch.cuda.device_count()
    if have < a.gpus:
        print(json.dumps({"metric": METRIC, "error": f"--gpus {a.gpus} but {have} GPU(s) visible"}), flush=True)
        return 1
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={a.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd, env=env)


def main():
    a = parse()
    if a.impl == "reference":
        reference_arm(a)
        return 0
    world = os.environ.get("WORLD_SIZE")
    if world is None and a.gpus > 1:
        return relaunch_under_torchrun(a)
    if world is not None and int(world) != a.gpus:
        raise SystemExit(f"bench.py: --gpus {a.gpus} but WORLD_SIZE={world}")
    os.environ.setdefault("NCCL_DEBUG", "INFO")
    os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    ours(a)
    return 0


if __name__ == "__main__":
    sys.exit(main())
