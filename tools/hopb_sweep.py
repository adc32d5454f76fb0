"""C5: HOP-B sweep -- batch x context x KVP, overlap on vs off.

    python tools/hopb_sweep.py [--model llama405b-like] [--kvp 2 4 8]
                               [--contexts 131072 ...] [--batches 1 2 ...]
                               [--out gpurun_out/hopb_sweep.jsonl]

One GPU of a KVP-sharded Helix pool (TPA = 1, TPF = KVP; one layer of the
model) is measured alone: rank 0 of a KVP-rank loopback pool with the
collectives switched off, so every number here is this GPU's real compute:

  * attn_ms_off -- batched attention + split reduce, which stores every
    slice straight into the peers' receive buffers (HOP-B off: the exchange
    follows the whole batch);
  * attn_ms_on  -- HOP-B on as this engine implements it: ONE request-ordered
    attention launch that only counts each stream's finished splits, and the
    co-resident stream reducer that merges and pushes every stream as it
    completes while later requests stream (overlap.hpp:37-69 at stream
    granularity; here the slices stay on this rank); serialised by the
    profiling events, so an upper bound;
  * layer_ms_off / layer_ms_on -- the whole layer (QKV .. FFN), eager launches,
    the two modes interleaved over 4 rounds, best round each (clocks drift
    down over a run; back-to-back measurement biased the second mode).

The all-to-all itself needs peers (one B200 here), so its duration comes from
the reference's own alpha-beta model (comm.hpp:28-45, a2a_payload_per_destination
:60-69; payload in fp32 as this engine sends it) with the reference's
gb200-like link figures (900 GB/s, 0.1 us) -- "modeled" in the output -- and
the exposed time with and without HOP-B from the reference's hopb_schedule
(overlap.hpp:37-69, composition latency.cpp:216-234) applied to the MEASURED
per-request compute. On a multi-GPU box `bench.py --gpus N` measures the real
NCCL exposure (its `hopb` key) on the same engine.

Points whose KV shard does not fit (1-layer slice: KV + weights > 170 GB) are
reported as skipped.
"""
import argparse
import ctypes
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from types import SimpleNamespace

from paper_2507_07120_b200 import analytic as A  # pinned to the reference library (tests/test_analytic.py)
from paper_2507_07120_b200.model import HARDWARE_PRESETS


def hopb_schedule(requests, compute, comm, enabled):
    """overlap.hpp:37-69: total span of R requests' compute + comm."""
    return A.hopb_schedule(requests, compute, comm, enabled).total


def a2a_time(hidden, head_size, batch, kvp, bytes_per_elem=4):
    """comm_time(AllToAll, kvp, per_dest * kvp) with the reference payload (comm.hpp:28-69)
    on the reference's gb200-like link (presets/gb200-like.json: 900 GB/s, 0.1 us)."""
    hw = HARDWARE_PRESETS["gb200-like"]
    hw = SimpleNamespace(**{**hw.__dict__, "bytes_per_param": bytes_per_elem})
    per_dest = A.a2a_payload_per_destination(SimpleNamespace(hidden_dim=hidden, head_size=head_size), batch, kvp, 1,
                                             hw)
    return A.comm_time("all_to_all", kvp, per_dest * kvp, hw)


def point(P, Loopback, spec, kvp, S, B, steps=5, rounds=4):
    import numpy as np
    import torch
    s_loc = S // kvp
    K, Hsz, H, F = spec.kv_heads, spec.head_size, spec.hidden_dim, spec.ffn_dim
    kv_bytes = B * s_loc * 2 * K * Hsz * 2
    w_bytes = H * (spec.query_heads * Hsz + 2 * K * Hsz) * 2 + (H // kvp) * H * 2 + 3 * H * F // kvp * 2
    if kv_bytes + w_bytes > 170e9:
        return {"kvp": kvp, "context": S, "batch": B, "skipped": "KV shard + weights exceed 170 GB"}
    lb = Loopback(kvp)
    eng = P.HelixDecoder(spec, tpa=1, kvp=kvp, batch=B, capacity=S + 64 * kvp, layers=1, vocab=4096,
                         use_graphs=False, pool=2, rank=0, loopback=lb, hopb=True)
    lib = P.lib()
    lib.hx_engine_set_flag(eng._h, 1, 3)  # no peers on one GPU: slices stay on this rank, all-reduces off
    eng.init_weights(2507, qkv="hash")
    eng.fill_kv_hash(S, 2507)
    tok = torch.randint(0, 4096, (B,), dtype=torch.int32, device="cuda")
    nxt = torch.zeros(B, dtype=torch.int32, device="cuda")
    stream = torch.cuda.ExternalStream(eng.stream())
    out = {"kvp": kvp, "context": S, "batch": B, "kv_tokens_per_gpu": s_loc}
    # The two modes are measured interleaved (off, on, off, on, ...) and each
    # keeps its best round: HBM-bound steps heat the part and the clocks drift
    # down over a run, so measuring one mode after the other biases the second
    # by up to ~10% (the first version of this sweep did exactly that).
    for hopb in (0, 1):  # warm both modes (first call of each captures nothing: eager)
        lib.hx_engine_set_flag(eng._h, 2, hopb)
        for _ in range(2):
            eng.step_device(tok.data_ptr(), nxt.data_ptr())
    best = {0: float("inf"), 1: float("inf")}
    for rnd in range(rounds):
        for hopb in ((0, 1) if rnd % 2 == 0 else (1, 0)):
            lib.hx_engine_set_flag(eng._h, 2, hopb)
            eng.step_device(tok.data_ptr(), nxt.data_ptr())
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record(stream)
            for _ in range(steps):
                eng.step_device(tok.data_ptr(), nxt.data_ptr())
            e1.record(stream)
            e1.synchronize()
            best[hopb] = min(best[hopb], e0.elapsed_time(e1) / steps)
    for hopb in (0, 1):
        lib.hx_engine_set_flag(eng._h, 2, hopb)
        prof = np.zeros(10)
        lib.hx_profile_step(eng._h, 3, prof.ctypes.data_as(ctypes.POINTER(ctypes.c_double)))
        key = "on" if hopb else "off"
        # off: batched attention (kind 2) + split reduce with the device push (kind 3);
        # on: the request-ordered attention (kind 2) + the co-resident stream reducer
        # (kind 3, serialised here by the profiling events); both then the flag wait (kind 9)
        out[f"attn_ms_{key}"] = float(prof[2] + prof[3])
        out[f"attn_kernel_ms_{key}"] = float(prof[2])
        out[f"reduce_ms_{key}"] = float(prof[3])
        out[f"flag_wait_ms_{key}"] = float(prof[9])
        out[f"layer_ms_{key}"] = best[hopb]
    streams = eng.info()["attn_streams"]
    eng.close()
    t = a2a_time(H, Hsz, B, kvp) * 1e3  # ms, whole batch, reference alpha-beta model
    # off: the exchange follows the whole batch's attention (fully exposed);
    # on: each stream's slices leave as the stream completes -- the reference's
    # hopb_schedule at the kernel's exchange granularity (R = streams)
    span_on = hopb_schedule(streams, out["attn_ms_on"] / streams, t / streams, True)
    # both modes end with the same one-CTA flag wait (device-initiated exchange)
    exp_on = max(0.0, span_on - out["attn_ms_on"]) + out["flag_wait_ms_on"]
    exp_off = t + out["flag_wait_ms_off"]
    out.update({
        "streams": streams, "a2a_ms_modeled": t, "exposed_a2a_ms_off": exp_off, "exposed_a2a_ms_on": exp_on,
        "a2a_hidden_frac": (1.0 - max(0.0, span_on - out["attn_ms_on"]) / t) if t > 0 else None,
        # what HOP-B buys end to end at this point, its compute price included: the
        # measured layer (interleaved, best round) plus the modeled exchange exposure
        "hopb_gain_ms": (out["layer_ms_off"] + t) - (out["layer_ms_on"] + max(0.0, span_on - out["attn_ms_on"])),
    })
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="llama405b-like")
    ap.add_argument("--kvp", type=int, nargs="+", default=[2, 4, 8])
    ap.add_argument("--contexts", type=int, nargs="+",
                    default=[131072, 262144, 524288, 1048576, 2097152, 4194304])
    ap.add_argument("--batches", type=int, nargs="+", default=[1, 2, 4, 8, 16, 32, 64])
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "hopb_sweep.jsonl"))
    a = ap.parse_args()
    import paper_2507_07120_b200 as P
    from paper_2507_07120_b200.model import Loopback
    spec = P.model.PRESETS[a.model]
    os.makedirs(os.path.dirname(a.out), exist_ok=True)
    with open(a.out, "w") as f:
        for kvp in a.kvp:
            for S in a.contexts:
                for B in a.batches:
                    try:
                        r = point(P, Loopback, spec, kvp, S, B)
                    except Exception as ex:  # recorded, the sweep goes on
                        r = {"kvp": kvp, "context": S, "batch": B, "error": str(ex)[:200]}
                    r["model"] = a.model
                    f.write(json.dumps(r) + "\n")
                    f.flush()
                    print(json.dumps(r), flush=True)


if __name__ == "__main__":
    main()
