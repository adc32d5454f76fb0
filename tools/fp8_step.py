"""A few decode steps of configs[1]'s model (llama3-8b-like, B = 8, 131072 KV
tokens/request) with FP8 KV pages and/or FP8 weights -- the workload for ncu
captures of the FP8 kernels (profiles/). Usage:
    python tools/fp8_step.py [--layers 2] [--kv fp8|bf16] [--w fp8|bf16] [--steps 3]
"""
import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--layers", type=int, default=2)
    ap.add_argument("--context", type=int, default=131072)
    ap.add_argument("--kv", default="fp8")
    ap.add_argument("--w", default="fp8")
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--g16", action="store_true", help="405B-like attention shard: 128 query / 8 KV heads (G = 16)")
    a = ap.parse_args()
    import paper_2507_07120_b200 as P
    spec = P.model.PRESETS["llama3-8b-like"]
    if a.g16:  # the C3 per-GPU attention shape (one GPU of KVP = 8: 8 KV heads, G = 16), small FFN
        spec = P.model.ModelSpec("g16", 1, 16384, 128, 8, 128, 1024, 3, "gqa", 0, vocab=4096)
    B = 8
    eng = P.HelixDecoder(spec, tpa=1, kvp=1, batch=B, capacity=a.context + 64, layers=a.layers,
                         kv_dtype=a.kv, w_dtype=a.w)
    eng.init_weights(2507, qkv="hash")
    eng.fill_kv_hash(a.context, 2507)
    tokens = (np.arange(B) * 131 + 7) % spec.vocab
    for _ in range(a.steps):
        tokens, _, _ = eng.step(tokens)
    print("ok", eng.info())
    eng.close()


if __name__ == "__main__":
    main()
