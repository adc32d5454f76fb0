"""Interleaved A/B of an engine environment switch on configs[1]'s model
(llama3-8b-like, B = 8, 131072 KV tokens/request, a few layers): two engines
built with the variable unset/"0" (A) and set to the given value (B), timed in
alternating rounds (clocks drift down over a run of HBM-bound steps, so
back-to-back measurement biases whichever runs second); best round per engine.

    python tools/ab_env.py HX_LOCAL_STREAM_REDUCE 1 [--layers 8] [--kv bf16] [--rounds 6]
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
    a = ap.parse_args()
    import torch
    import paper_2507_07120_b200 as P
    spec = P.model.PRESETS["llama3-8b-like"]
    if a.g16:
        spec = P.model.ModelSpec("g16", 1, 16384, 128, 8, 128, 1024, 3, "gqa", 0, vocab=4096)
    B = 8
    engines = []
    for v in ("0", a.value):
        os.environ[a.var] = v
        g = P.HelixDecoder(spec, batch=B, capacity=a.context + 64, layers=a.layers, kv_dtype=a.kv, w_dtype=a.w)
        g.init_weights(2507, qkv="hash")
        g.fill_kv_hash(a.context, 2507)
        engines.append(g)
    tok = torch.randint(0, spec.vocab, (B,), dtype=torch.int32, device="cuda")
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
    print(json.dumps({"var": a.var, "A_ms": best[0], "B_ms": best[1], "B_over_A": best[1] / best[0],
                      "layers": a.layers, "kv": a.kv, "w": a.w}))


if __name__ == "__main__":
    main()
