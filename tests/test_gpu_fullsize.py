"""Parity at the BASELINE configs' full sizes through size-independent
properties (the double oracle cannot run these sizes in test time):

* KVP invariance -- the Helix decomposition is exact (attention.hpp:413-417:
  sharded attention + LSE merge reproduces monolithic attention), so the same
  model over the same global token stream must give the same hidden states
  and logits whether its KV sits in one shard or is round-robin sharded over
  a KVP pool (here: the local pool on one GPU, every shard a separate page
  pool with its own split/merge path). Only fp32 summation order differs.
* Determinism -- every reduction runs in a fixed order, so repeating a step
  on an identical state is bit-identical.

Shapes: configs[1] layer (llama3-8b-like, B = 8, S = 131072), configs[2]
layer (llama405b-like, B = 8, S = 1M global = 125k per KVP-8 shard), configs[3]
layer (deepseek-r1-like MLA, B = 8, 1M global). Vocab is reduced (LM-head
rows are independent), one layer each.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def rel_err(got, want):
    return float(np.abs(got - want).max() / max(1e-12, np.abs(want).max()))


def _run(P, spec, kvp, S, B, tokens, ep=1, kv_dtype="bf16", steps=1):
    g = P.HelixDecoder(spec, tpa=1, kvp=kvp, batch=B, capacity=S + 64 * kvp, layers=1, vocab=2048,
                       kv_dtype=kv_dtype)
    g.init_weights(2507, qkv="hash")
    g.fill_kv_hash(S, 2507)
    outs = []
    for _ in range(steps):
        nxt, logits, hidden = g.step(tokens, want_logits=True, want_hidden=True)
        outs.append((nxt, logits, hidden))
    g.close()
    return outs


@pytest.mark.parametrize("preset,S,kvps", [
    ("llama3-8b-like", 131072, (1, 4)),
    ("llama405b-like", 1000000, (1, 8)),
])
def test_kvp_invariance_full_size(preset, S, kvps):
    import paper_2507_07120_b200 as P
    spec = P.model.PRESETS[preset]
    B = 8
    tokens = (np.arange(B) * 211 + 5) % 2048
    ref = _run(P, spec, kvps[0], S, B, tokens, steps=2)
    got = _run(P, spec, kvps[1], S, B, tokens, steps=2)
    for step in range(2):
        e_h = rel_err(got[step][2], ref[step][2])
        e_l = rel_err(got[step][1], ref[step][1])
        print(f"{preset} S={S} kvp {kvps[0]} vs {kvps[1]} step {step}: hidden {e_h:.2e} logits {e_l:.2e}")
        assert e_h <= 1e-3 and e_l <= 1e-3


def test_mla_kvp_invariance_full_size():
    import paper_2507_07120_b200 as P
    spec = P.model.PRESETS["deepseek-r1-like"]
    B, S = 8, 1000000
    tokens = (np.arange(B) * 97 + 3) % 2048
    # MoE routing is part of the layer; a near-tie in the router could legally pick
    # another expert set under a different summation order -- compare attention-
    # dominated hidden states with the routed FFN included, at a loose bound
    ref = _run(P, spec, 1, S, B, tokens)
    got = _run(P, spec, 8, S, B, tokens)
    e_h = rel_err(got[0][2], ref[0][2])
    print(f"deepseek-r1-like S={S} kvp 1 vs 8: hidden {e_h:.2e}")
    assert e_h <= 5e-3


@pytest.mark.parametrize("kv_dtype", ["bf16", "fp8"])
def test_decode_step_is_deterministic_full_size(kv_dtype):
    """Same state, same step -> bit-identical logits and hidden states."""
    import paper_2507_07120_b200 as P
    spec = P.model.PRESETS["llama3-8b-like"]
    B, S = 8, 131072
    tokens = (np.arange(B) * 13 + 1) % 2048
    a = _run(P, spec, 1, S, B, tokens, kv_dtype=kv_dtype)
    b = _run(P, spec, 1, S, B, tokens, kv_dtype=kv_dtype)
    np.testing.assert_array_equal(a[0][1], b[0][1])
    np.testing.assert_array_equal(a[0][2], b[0][2])
    np.testing.assert_array_equal(a[0][0], b[0][0])


def test_fp8_vs_bf16_full_size():
    """FP8 pages change only the KV storage rounding: the step stays close to
    bf16's. With the hash QKV weights (unit scale, like the reference's
    U[-1,1) draws) the logits have a std of ~40, so the softmax is peaked and
    e4m3's 2^-4 relative rounding of K and V moves the layer output by ~10%;
    the bound only rules out a broken FP8 path (exact parity against an
    e4m3-storage oracle is tests/test_gpu_fp8.py)."""
    import paper_2507_07120_b200 as P
    spec = P.model.PRESETS["llama3-8b-like"]
    B, S = 8, 131072
    tokens = (np.arange(B) * 17 + 2) % 2048
    a = _run(P, spec, 1, S, B, tokens, kv_dtype="bf16")
    b = _run(P, spec, 1, S, B, tokens, kv_dtype="fp8")
    e_h = rel_err(b[0][2], a[0][2])
    print(f"fp8 vs bf16 hidden {e_h:.2e}")
    assert e_h <= 0.25
