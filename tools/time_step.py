"""Time decode steps of configs[1]'s model (or the G16 shape) for one engine
configuration -- for A/B runs across processes (process-wide switches such as
HX_W8_CTAS). Prints one JSON line: best-of-rounds ms per step.
    python tools/time_step.py [--kv fp4] [--w fp4] [--layers 4] [--rounds 5]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--layers", type=int, default=4)
    ap.add_argument("--context", type=int, default=131072)
    ap.add_argument("--kv", default="bf16")
    ap.add_argument("--w", default="bf16")
    ap.add_argument("--rounds", type=int, default=5)
    ap.add_argument("--steps", type=int, default=5)
    a = ap.parse_args()
    import torch
    import paper_2507_07120_b200 as P
    spec = P.model.PRESETS["llama3-8b-like"]
    B = 8
    g = P.HelixDecoder(spec, batch=B, capacity=a.context + a.rounds * a.steps + 64, layers=a.layers, kv_dtype=a.kv,
                       w_dtype=a.w)
    g.init_weights(2507, qkv="hash")
    g.fill_kv_hash(a.context, 2507)
    tok = torch.randint(0, spec.vocab, (B,), dtype=torch.int32, device="cuda")
    nxt = torch.zeros(B, dtype=torch.int32, device="cuda")
    for _ in range(3):
        g.step_device(tok.data_ptr(), nxt.data_ptr())
    s = torch.cuda.ExternalStream(g.stream())
    best = float("inf")
    for _ in range(a.rounds):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(s)
        for _ in range(a.steps):
            g.step_device(tok.data_ptr(), nxt.data_ptr())
        e1.record(s)
        e1.synchronize()
        best = min(best, e0.elapsed_time(e1) / a.steps)
    print(json.dumps({"ms": best, "env": {k: v for k, v in os.environ.items() if k.startswith("HX_")}}))


if __name__ == "__main__":
    main()
