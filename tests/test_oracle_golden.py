"""Pin the CPU oracle (clean-room restatement of attention.hpp) against golden
vectors produced by the REFERENCE's own header (oracle/gen_golden.cpp, run over
/root/reference/proj/include/helixsim/attention.hpp unmodified + the in-repo
Eigen shim). CPU only."""
import json
import os

import numpy as np
import pytest

from tests import oracle_py as O

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "reference_harness.json")


def _load():
    with open(GOLDEN) as f:
        return json.load(f)


def _num(v):
    return float("-inf") if v == "-inf" else float("inf") if v == "inf" else float(v)


def rel_err(got, want):
    # helixsim.cpp:381-384 / test_attention.cpp:25-28
    scale = max(1e-12, np.abs(want).max())
    return np.abs(got - want).max() / scale


CASES = _load()["cases"]


@pytest.mark.parametrize("case", CASES, ids=[c["name"] for c in CASES])
def test_restatement_reproduces_reference_harness(case):
    h = O.Harness(case["query_heads"], case["kv_heads"], case["head_size"], case["tpa"], case["kvp"],
                  case["chunk"], case["seed"])
    rng = O.Rng(case["grow_seed"])
    h.grow_random(case["context"], rng)
    hidden = case["query_heads"] * case["head_size"]
    shape = (case["query_heads"], case["head_size"])
    for s in case["steps"]:
        x = rng.draws(hidden)  # random_matrix(rng, hidden, 1): same stream as the reference
        np.testing.assert_array_equal(x, np.array(s["x"]))  # RNG stream is bit-identical
        want_ref = np.array(s["reference"]).reshape(shape)
        want_step = np.array(s["step"]).reshape(shape)
        ref = h.reference(x)
        got, _ = h.step(x)
        assert rel_err(ref, want_ref) <= 1e-12
        assert rel_err(got, want_step) <= 1e-12
        # and the reference's own exactness contract (test_attention.cpp:302-303)
        assert rel_err(got, ref) <= 1e-10
    assert [h.effective_tokens(r) for r in range(case["kvp"])] == case["effective_tokens"]
    ranks, _ = h.token_order()
    assert ranks.tolist() == case["token_rank"]
    assert h.max_min_gap() == case["max_min_gap"]
    np.testing.assert_array_equal(h.transcript().reshape(-1), np.array(case["transcript"], dtype=np.int64))
    k0 = h.cache_rows(0, 0, 0)
    v0 = h.cache_rows(0, 0, 1)
    assert rel_err(k0, np.array(case["rank0_head0_keys"]).reshape(k0.shape)) <= 1e-12
    assert rel_err(v0, np.array(case["rank0_head0_values"]).reshape(v0.shape)) <= 1e-12


def test_merge_matches_reference_fragments():
    m = _load()["merge"]
    w = m["width"]
    q = np.array(m["q"])
    outs, lses = [], []
    for f in m["fragments"]:
        keys = np.array(f["keys"]).reshape(-1, w)
        values = np.array(f["values"]).reshape(-1, w)
        out, lse = O.partial_head_attention(q, keys, values)
        assert lse == _num(f["lse"]) or abs(lse - _num(f["lse"])) <= 1e-12 * abs(lse)
        assert rel_err(out, np.array(f["out"])) <= 1e-12 if keys.shape[0] else np.all(out == 0)
        outs.append(out)
        lses.append(lse)
    merged, lse = O.merge_head_fragments(np.array(outs), np.array(lses))
    assert rel_err(merged, np.array(m["merged_out"])) <= 1e-12
    assert abs(lse - m["merged_lse"]) <= 1e-12 * abs(lse)
    assert rel_err(merged, np.array(m["reference"])) <= 1e-10
    # permutation invariance is bitwise (attention.hpp:85-88)
    perm = np.random.default_rng(7).permutation(len(outs))
    m2, l2 = O.merge_head_fragments(np.array(outs)[perm], np.array(lses)[perm])
    assert np.array_equal(m2, merged) and l2 == lse


def test_transcript_contract_worked_shape():
    # test_attention.cpp:318-348
    h = O.Harness(4, 2, 8, 2, 4, 16, 42)
    rng = O.Rng(113)
    h.grow_random(48, rng)
    x = rng.draws(32)
    h.step(x)
    t = h.transcript()
    b = t[t[:, 0] == 0]
    a = t[t[:, 0] == 1]
    assert len(b) == 7 and np.all(b[:, 1] == 0) and np.all(b[:, 3] == 32) and np.all(b[:, 4] == 0)
    assert len(a) == 24 and np.all(a[:, 1] != a[:, 2]) and np.all(a[:, 3] == 4) and np.all(a[:, 4] == 1)


def test_shape_validation_messages():
    # test_attention.cpp:382-395 + the reference's messages (attention.hpp:431-437, 461-464)
    with pytest.raises(ValueError, match="multiple of kv_heads"):
        O.Harness(4, 3, 8, 1, 1, 16, 1)
    with pytest.raises(ValueError, match="tpa must divide kv_heads"):
        O.Harness(4, 2, 8, 4, 1, 16, 1)
    with pytest.raises(ValueError, match="divide the hidden width"):
        O.Harness(4, 2, 8, 2, 3, 16, 1)
    h = O.Harness(4, 2, 8, 2, 2, 16, 1)
    with pytest.raises(ValueError, match="nonempty context"):
        h.step(np.zeros(32))
    h.grow_random(4, O.Rng(116))
    with pytest.raises(ValueError, match="wrong width"):
        h.step(np.zeros(31))


def test_bf16_rounding_is_rne():
    vals = np.array([1.0, 1.00390625, 1.005859375, -0.333333333, 1e-20, 0.0])
    r = O.round_bf16(vals)
    assert r[0] == 1.0 and r[1] == 1.0  # tie 1+2^-8 -> even (1.0)
    assert r[2] == 1.0078125
    assert abs(r[3] - (-0.333984375)) < 1e-12
    f32 = np.float32(vals[3])
    # agrees with the bit-level RNE of torch/CUDA for representable cases
    b = np.array([f32]).view(np.uint32)[0]
    b = (b + 0x7FFF + ((b >> 16) & 1)) & 0xFFFF0000
    assert np.array([b], dtype=np.uint32).view(np.float32)[0] == np.float32(r[3])


def test_oracle_moe_routing_invariants():
    """MoE oracle: k distinct in-range experts per (layer, request), listed by
    descending router logit (margins >= 0); top_k == E selects every expert."""
    for E, k in [(8, 3), (4, 4)]:
        m = O.Model(64, 4, 2, 16, 0, 2, 50, batch=3, seed=5, qkv_hash=True, bf16=True, moe=(E, k, 32))
        for l in range(2):
            for b in range(3):
                m.grow_hash(l, b, 9)
        lo, ho, no = m.step(np.array([1, 2, 3]))
        r = m.routes()
        assert r.shape == (2, 3, k)
        for l in range(2):
            for b in range(3):
                assert len(set(r[l, b])) == k and r[l, b].min() >= 0 and r[l, b].max() < E
        g = m.route_gaps()
        assert (g >= 0).all()
        assert np.isfinite(lo).all() and np.abs(ho[-1] - ho[0]).max() > 0


@pytest.mark.parametrize("kvp", [2, 3])
def test_oracle_mla_sharding_invariance(kvp):
    """MLA through the reference's shard_attention + merge_fragments: hidden
    states and logits do not depend on the KVP width (the Helix exactness
    property, attention.hpp:118-175), to rounding."""
    def run(k):
        m = O.Model(128, 8, 1, 16, 64, 2, 50, kvp=k, batch=2, seed=4, qkv_hash=True, bf16=True, kv_latent=288)
        for l in range(2):
            for b in range(2):
                m.grow_hash(l, b, 37 + 5 * b)
        out = []
        toks = np.array([1, 2])
        for _ in range(2):
            lo, ho, no = m.step(toks)
            out.append((lo, ho))
            toks = no
        return out
    a, b = run(1), run(kvp)
    for (la, ha), (lb, hb) in zip(a, b):
        assert np.abs(la - lb).max() <= 1e-10 * np.abs(la).max()
        assert np.abs(ha - hb).max() <= 1e-10 * np.abs(ha).max()
