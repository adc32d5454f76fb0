"""MLA attention kernel measurement at the C4 (deepseek-r1-like, KVP=8) per-GPU
shard: B=8 requests x 131072 latent tokens (1M context / KVP 8) of 576 bf16,
128 query heads. Hidden width is shrunk (H = 128 x 8) so the decode step is
dominated by the attention kernel; per-kernel times come from hx_profile_step."""
import ctypes
import json
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import paper_2507_07120_b200 as P  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 8
S = int(sys.argv[2]) if len(sys.argv) > 2 else 131072
spec = P.model.ModelSpec("mla-bench", 1, 1024, 128, 1, 8, 1024, 3, "mla", 288, vocab=1000)
g = P.HelixDecoder(spec, tpa=1, kvp=1, batch=B, capacity=S + 64, layers=1, vocab=1000)
g.init_weights(1, qkv="hash")
t0 = time.time()
g.fill_kv_hash(S, 1)
print("fill", time.time() - t0, "s", file=sys.stderr)
toks = np.arange(B) % 1000
for _ in range(3):
    g.step(toks)
ms = np.zeros(10)
reps = 10
P.lib().hx_profile_step(g._h, reps, ms.ctypes.data_as(ctypes.POINTER(ctypes.c_double)))
att = ms[2]
red = ms[3]
kv_bytes = B * S * 576 * 2
flops = B * S * 128 * (576 + 512) * 2
print(json.dumps({"B": B, "S": S, "attention_ms": att, "split_reduce_ms": red,
                  "kv_GBps": kv_bytes / att / 1e6, "TFLOPs": flops / att / 1e9,
                  "hbm_frac": kv_bytes / att / 1e6 / 6556.2, "tensor_frac_sustained": flops / att / 1e9 / 1393.0,
                  "info": g.info()}))
