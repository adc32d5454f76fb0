import sys
import numpy as np
sys.path.insert(0, ".")
import paper_2507_07120_b200 as P
from tests import oracle_py as O


def rel(a, b):
    return float(np.abs(a - b).max() / max(1e-12, np.abs(b).max()))


for batch in [int(a) for a in sys.argv[1:]]:
    spec = P.model.ModelSpec("t", 1, 128, 4, 2, 32, 256, 3, "gqa", 0, vocab=500)
    g = P.HelixDecoder(spec, batch=batch, capacity=128, layers=1, vocab=500, use_graphs=False)
    g.init_weights(31, qkv="hash")
    g.fill_kv_hash(40, 31)
    o = O.Model(128, 4, 2, 32, 256, 1, 500, batch=batch, seed=31, qkv_hash=True, bf16=True)
    for b in range(batch):
        o.grow_hash(0, b, 40)
    toks = np.arange(batch) * 7 % 500
    nxt, logits, hidden = g.step(toks, want_logits=True, want_hidden=True)
    lo, ho, no = o.step(toks)
    per_b = [rel(hidden[1][b], ho[1][b]) for b in range(batch)]
    bad = [b for b in range(batch) if per_b[b] > 2e-3]
    print(batch, "h0", rel(hidden[0], ho[0]), "h1", rel(hidden[1], ho[1]), "logits", rel(logits, lo), "bad rows", bad[:20])
