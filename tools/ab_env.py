"""Interleaved A/B of an engine environment switch on configs[1]'s model
(llama3-8b-like, B = 8, 131072 KV tokens/request, a few layers): two engines
built with the variable unset/"0" (A) and set to the given value (B), timed in
alternating rounds (clocks drift down over a run of HBM-bound steps, so
back-to-back measurement biases whichever runs second); best round per engine.

    python tools/ab_env.py HX_LOCAL_STREAM_REDUCE 1 [--layers 8] [--kv bf16] [--rounds 6]
    python tools/ab_env.py HX_FUSED_COMBINE 1 --slice [--layers 4]   # C3: llama405b-like rank 0 of a KVP=8 pool
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("var")
    ap.add_argument("value")
    ap.add_argument("--layers", type=int, default=8)
    ap.add_argument("--context", type=int, default=131072)
    ap.add_argument("--kv", default="bf16")
    ap.add_argument("--w", default="bf16")
    ap.add_argument("--rounds", type=int, default=6)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--g16", action="store_true", help="the C3 per-GPU attention shape: 128 query / 8 KV heads")
    ap.add_argument("--slice", action="store_true",
                    help="bench.py's C3 slice: llama405b-like rank 0 of a TPA=1 x KVP=8 loopback pool, "
                         "collectives off, --context tokens per request on this GPU")
    ap.add_argument("--hopb", action="store_true", help="--slice with HOP-B on")
    ap.add_argument("--profile", action="store_true", help="also print both engines' hx_profile_step breakdowns")
    a = ap.parse_args()
    import torch
    import paper_2507_07120_b200 as P
    spec = P.model.PRESETS["llama3-8b-like"]
    if a.g16:
        spec = P.model.ModelSpec("g16", 1, 16384, 128, 8, 128, 1024, 3, "gqa", 0, vocab=4096)
    B = 8
    engines = []
    vocab = spec.vocab
    for v in ("0", a.value):
        os.environ[a.var] = v
        if a.slice:
            from paper_2507_07120_b200.model import Loopback
            spec, N, vocab = P.model.PRESETS["llama405b-like"], 8, 4096
            g = P.HelixDecoder(spec, tpa=1, kvp=N, batch=B, capacity=(a.context + 64) * N, layers=a.layers,
                               vocab=vocab, use_graphs=True, pool=2, rank=0, loopback=Loopback(N), hopb=a.hopb,
                               kv_dtype=a.kv, w_dtype=a.w)
            P._lib.check(P.lib().hx_engine_set_flag(g._h, 1, 3), g._h)  # collectives off (no peers)
            g.init_weights(2507, qkv="hash")
            g.fill_kv_hash(a.context * N, 2507)
        else:
            g = P.HelixDecoder(spec, batch=B, capacity=a.context + 64, layers=a.layers, kv_dtype=a.kv, w_dtype=a.w)
            g.init_weights(2507, qkv="hash")
            g.fill_kv_hash(a.context, 2507)
        engines.append(g)
    tok = torch.randint(0, vocab, (B,), dtype=torch.int32, device="cuda")
    nxt = torch.zeros(B, dtype=torch.int32, device="cuda")
    for g in engines:
        for _ in range(3):
            g.step_device(tok.data_ptr(), nxt.data_ptr())
    best = [float("inf"), float("inf")]
    for r in range(a.rounds):
        for i in ((0, 1) if r % 2 == 0 else (1, 0)):
            g = engines[i]
            s = torch.cuda.ExternalStream(g.stream())
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record(s)
            for _ in range(a.steps):
                g.step_device(tok.data_ptr(), nxt.data_ptr())
            e1.record(s)
            e1.synchronize()
            best[i] = min(best[i], e0.elapsed_time(e1) / a.steps)
    prof = []
    if a.profile:  # hx_profile_step: per-phase launch times (bench.py pool_slice breakdown order)
        import ctypes
        import numpy as np
        names = ["embed", "qkv", "attention", "split_reduce", "o_proj", "gate_up", "down", "lm_head", "merge"]
        for g in engines:
            pr = np.zeros(10)
            P.lib().hx_profile_step(g._h, 5, pr.ctypes.data_as(ctypes.POINTER(ctypes.c_double)))
            g.synchronize()
            prof.append({k: round(float(v), 4) for k, v in zip(names, pr)})
    print(json.dumps({"var": a.var, "A_ms": best[0], "B_ms": best[1], "B_over_A": best[1] / best[0], "profile": prof,
                      "layers": a.layers, "kv": a.kv, "w": a.w, "slice": a.slice, "hopb": a.hopb}))


if __name__ == "__main__":
    main()
