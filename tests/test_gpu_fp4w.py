"""GPU parity of FP4 (e2m1) GEMV weights -- the paper's evaluation precision
("all model weights, KV states ... FP4"; w_dtype="fp4").

Every GEMV weight (QKV / MLA W_q + latent projection, O, gate/up, down, MoE
router and experts, LM head) is stored in MX-style e2m1 blocks: 32 consecutive
inputs of one output feature share a power-of-two scale; the oracle quantises
its double hash draws identically (layer_oracle.cpp quantize_fp4_cols, pinned on
CPU in tests/test_fp4_oracle.py), so GPU and oracle multiply the SAME weights.
The GEMV widens e2m1 exactly to f16 (cvt.rn.f16x2.e2m1x2) and applies the block
scale in f16 (exact), activations as two f16 terms (22 bits): the comparison
bounds are the bf16 / FP8 paths' -- 2e-3 on the first step's hidden states and
logits (fp32 accumulation over K, exact-weight operands).
"""
import threading

import numpy as np
import pytest

from tests import oracle_py as O

pytestmark = pytest.mark.gpu


def rel_err(got, want):
    return float(np.abs(got - want).max() / max(1e-12, np.abs(want).max()))


@pytest.mark.parametrize("q,k,hsz,kvp,B,kv", [(8, 2, 32, 2, 3, "bf16"), (32, 2, 64, 1, 8, "bf16"),
                                              (16, 1, 128, 4, 16, "bf16"), (8, 2, 64, 2, 5, "fp8")])
def test_fp4_weights_decode_step_matches_oracle(q, k, hsz, kvp, B, kv):
    import paper_2507_07120_b200 as P
    H, F, L, V = q * hsz, 384, 2, 700
    spec = P.model.ModelSpec("w4", L, H, q, k, hsz, F, 3, "gqa", 0, vocab=V)
    g = P.HelixDecoder(spec, tpa=1, kvp=kvp, batch=B, capacity=2100, layers=L, vocab=V, kv_dtype=kv, w_dtype="fp4")
    assert g.info()["w_dtype"] == 2
    g.init_weights(17, qkv="hash")
    g.fill_kv_hash(2000, 17)
    o = O.Model(H, q, k, hsz, F, L, V, tpa=1, kvp=kvp, batch=B, seed=17, qkv_hash=True, kv_fp8=kv == "fp8",
                w_fp4=True)
    for l in range(L):
        for b in range(B):
            o.grow_hash(l, b, 2000)
    tokens = (np.arange(B) * 131 + 1) % V
    for step in range(2):
        nxt, logits, hidden = g.step(tokens, want_logits=True, want_hidden=True)
        lo, ho, no = o.step(tokens)
        tol = 2e-3 if step == 0 else 2e-2
        e_h, e_l = rel_err(hidden, ho), rel_err(logits, lo)
        print(f"fp4w q={q} k={k} hsz={hsz} kvp={kvp} B={B} kv={kv} step={step} hidden={e_h:.2e} logits={e_l:.2e}")
        assert e_h <= tol and e_l <= tol
        tokens = no
    g.close()


@pytest.mark.parametrize("tpa,kvp", [(1, 2), (2, 2)])
def test_fp4_weights_loopback_pool(tpa, kvp):
    """Distributed layout (TPA-sharded QKV heads, TP-sharded O-proj rows / FFN
    columns / vocabulary): the 32-input blocks of a sharded matrix start at
    multiples of 32 of its full input range, so every rank's shard carries the
    oracle's quantisation."""
    import paper_2507_07120_b200 as P
    from paper_2507_07120_b200.model import Loopback
    H, Q, K, D, F, L, V, B = 512, 16, 2, 32, 512, 2, 400, 2
    n = tpa * kvp
    spec = P.model.ModelSpec("w4d", L, H, Q, K, D, F, 3, "gqa", 0, vocab=V)
    lb = Loopback(n)
    engines = [P.HelixDecoder(spec, tpa=tpa, kvp=kvp, batch=B, capacity=3000, layers=L, vocab=V, use_graphs=False,
                              pool=2, rank=r, loopback=lb, w_dtype="fp4") for r in range(n)]
    for e in engines:
        e.init_weights(3, qkv="hash")
        e.fill_kv_hash(2500, 3)
    o = O.Model(H, Q, K, D, F, L, V, tpa=tpa, kvp=kvp, batch=B, seed=3, qkv_hash=True, w_fp4=True)
    for l in range(L):
        for b in range(B):
            o.grow_hash(l, b, 2500)
    tokens = np.array([4, 399])
    res = [None] * n
    errors = []

    def run(r):
        try:
            res[r] = engines[r].step(tokens, want_logits=True, want_hidden=True)
        except Exception as ex:  # surfaced below
            errors.append(ex)
    th = [threading.Thread(target=run, args=(r,), daemon=True) for r in range(n)]
    [t.start() for t in th]
    [t.join(timeout=120) for t in th]
    assert not errors, errors
    lo, ho, no = o.step(tokens)
    for r in range(n):
        e_h = rel_err(res[r][2], ho)
        print(f"rank {r}: hidden {e_h:.2e}")
        assert e_h <= 2e-3
        np.testing.assert_array_equal(res[r][0], no)
    for e in engines:
        e.close()


def test_fp4_weights_weight_bytes():
    """e2m1 codes + one exponent byte per 32 inputs: 17/32 byte per weight."""
    import paper_2507_07120_b200 as P
    spec = P.model.ModelSpec("w4", 1, 1024, 8, 2, 128, 1024, 3, "gqa", 0, vocab=512)
    a = P.HelixDecoder(spec, batch=2, capacity=64, layers=1, vocab=512)
    b = P.HelixDecoder(spec, batch=2, capacity=64, layers=1, vocab=512, w_dtype="fp4")
    assert b.info()["weight_bytes_per_layer"] * 64 == a.info()["weight_bytes_per_layer"] * 17
    a.close()
    b.close()


@pytest.mark.parametrize("E,k,Fe,shared,B,kvp", [(8, 2, 128, 0, 3, 1), (16, 4, 64, 256, 5, 2), (32, 6, 128, 0, 16, 2)])
def test_fp4_weights_moe_matches_oracle(E, k, Fe, shared, B, kvp):
    """Routed MoE with FP4 router / expert / shared-expert weights: grouped
    expert GEMVs stream each expert's image with its inline block scales."""
    import paper_2507_07120_b200 as P
    H, Q, K, D, L, V = 256, 8, 2, 32, 2, 1000
    spec = P.model.ModelSpec("moe", L, H, Q, K, D, 512, 3, "gqa", 0, P.model.MoESpec(E, k, Fe, shared), vocab=V)
    seed = 900 + E
    g = P.HelixDecoder(spec, tpa=1, kvp=kvp, batch=B, capacity=256, layers=L, vocab=V, w_dtype="fp4")
    g.init_weights(seed, qkv="hash")
    o = O.Model(H, Q, K, D, shared, L, V, tpa=1, kvp=kvp, chunk=16, batch=B, seed=seed, qkv_hash=True,
                moe=(E, k, Fe), w_fp4=True)
    g.fill_kv_hash(37, seed)
    for l in range(L):
        for b in range(B):
            o.grow_hash(l, b, 37)
    tokens = (np.arange(B) * 131 + 7) % V
    compared = 0
    # Two steps: from step 1 on each side attends over its OWN appended K/V (GPU:
    # fp32 projection -> bf16; oracle: double -> bf16), and an element on the other
    # side of a bf16 rounding boundary moves the peaked (unit-scale hash weights)
    # softmax of that request: request 9 of the E=32, B=16 case reaches 4e-4 at
    # step 1 and 2.3e-2 at step 2 for any B >= 10 (the bf16-weight MoE test sees
    # the same effect at other seeds). Exact-operand parity of the attention is
    # tests/test_gpu_fp8.py's step_append comparison.
    for step in range(2):
        nxt, logits, hidden = g.step(tokens, want_logits=True, want_hidden=True)
        lo, ho, no = o.step(tokens)
        if not o.route_gaps().min() > 1e-4:
            break  # a router near-tie: the two sides may legally diverge from here
        tol = 2e-3 if step == 0 else 2e-2
        e_h, e_l = rel_err(hidden, ho), rel_err(logits, lo)
        print(f"E={E} k={k} shared={shared} B={B} step={step} hidden={e_h:.2e} logits={e_l:.2e}")
        assert e_h <= tol and e_l <= tol
        compared += 1
        tokens = no
    assert compared >= 1
    g.close()


@pytest.mark.parametrize("moe", [False, True])
def test_fp4_weights_mla_matches_oracle(moe):
    """MLA (W_q and the latent projection in FP4; W_UK / W_UV bf16), alone and
    with a routed MoE FFN -- the deepseek-shaped layer in miniature."""
    import paper_2507_07120_b200 as P
    H, Q, HSZ, L, V, LAT = 256, 16, 16, 2, 500, 288
    m = P.model.MoESpec(8, 2, 64, 64) if moe else None
    spec = P.model.ModelSpec("mla", L, H, Q, 1, HSZ, 256, 3, "mla", LAT, m, vocab=V)
    B, ctx, seed = 3, 333, 11
    g = P.HelixDecoder(spec, tpa=1, kvp=2, batch=B, capacity=ctx + 8, layers=L, vocab=V, w_dtype="fp4")
    g.init_weights(seed, qkv="hash")
    g.fill_kv_hash(ctx, seed)
    o = O.Model(H, Q, 1, HSZ, 64 if moe else 256, L, V, tpa=1, kvp=2, chunk=16, batch=B, seed=seed, qkv_hash=True,
                moe=(8, 2, 64) if moe else None, kv_latent=LAT, w_fp4=True)
    for l in range(L):
        for b in range(B):
            o.grow_hash(l, b, ctx)
    tokens = np.array([1, 2, 3])
    compared = 0
    for step in range(2):
        nxt, logits, hidden = g.step(tokens, want_logits=True, want_hidden=True)
        lo, ho, no = o.step(tokens)
        if moe and not o.route_gaps().min() > 1e-4:
            break  # a router near-tie: the two sides may legally diverge from here
        tol = 5e-3 if step == 0 else 2e-2
        e_h, e_l = rel_err(hidden, ho), rel_err(logits, lo)
        print(f"mla moe={moe} step={step} hidden={e_h:.2e} logits={e_l:.2e}")
        assert e_h <= tol and e_l <= tol
        compared += 1
        tokens = no
    assert compared >= 1, "router near-tie on the first step at this seed; pick another"
    g.close()


@pytest.mark.parametrize("what", ["batch", "mt19937"])
def test_fp4_weights_rejections(what):
    import paper_2507_07120_b200 as P
    if what == "batch":
        spec = P.model.ModelSpec("w4", 1, 256, 8, 2, 32, 256, 3, "gqa", 0, vocab=300)
        with pytest.raises(ValueError, match="batch <= 16"):
            P.HelixDecoder(spec, batch=32, capacity=64, layers=1, vocab=300, w_dtype="fp4")
    else:
        spec = P.model.ModelSpec("w4", 1, 256, 8, 2, 32, 256, 3, "gqa", 0, vocab=300)
        g = P.HelixDecoder(spec, batch=1, capacity=64, layers=1, vocab=300, w_dtype="fp4")
        with pytest.raises(Exception, match="hash"):
            g.init_weights(1)
        g.close()
