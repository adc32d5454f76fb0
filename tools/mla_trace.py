"""Per-tile event trace of the MLA kernel's first CTA pair (debug build):

    HX_NVCC_FLAGS=-DHX_MLA_TRACE python -m paper_2507_07120_b200.build   # (touch csrc/mla.cu first)
    KV=fp8 python tools/mla_trace.py      # or KV=bf16

Runs two eager decode steps of the C4 shard (deepseek-r1-like rank 0 of KVP = 8 x
EP = 8, B = 8, 125,000 latent tokens); the kernel prints softmax / MMA-issue event
times (ns, %globaltimer) per 256-token tile.
"""
import sys, os, torch
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), '..'))
import paper_2507_07120_b200 as P
from paper_2507_07120_b200.model import Loopback
kv = os.environ.get("KV", "fp8")
spec = P.model.PRESETS["deepseek-r1-like"]
B, N, S = 8, 8, 125000
eng = P.HelixDecoder(spec, tpa=1, kvp=N, batch=B, capacity=S * N + 64 * N, layers=1, vocab=4096, use_graphs=False,
                     pool=2, rank=0, loopback=Loopback(N), ep=8, kv_dtype=kv)
P._lib.check(P.lib().hx_engine_set_flag(eng._h, 1, 3), eng._h)
eng.init_weights(2507, qkv="hash")
eng.fill_kv_hash(S * N, 2507)
tok = torch.arange(B, dtype=torch.int32, device="cuda")
nxt = torch.zeros(B, dtype=torch.int32, device="cuda")
for _ in range(2):
    eng.step_device(tok.data_ptr(), nxt.data_ptr())
torch.cuda.synchronize()
