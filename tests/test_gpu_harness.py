"""GPU parity of the DecodeHarness path (C-ABI -> CUDA) against the CPU oracle.

Two comparisons per step:
  * against the oracle run on the SAME bf16-stored operands (weights, grown KV,
    appended KV rounded to bf16 exactly as the GPU stores them, x rounded to
    fp32): the tolerance bounds the GPU arithmetic itself;
  * against the reference's own double-precision outputs (golden vectors from
    attention.hpp): bounds the effect of bf16 storage.
"""
import json
import os

import numpy as np
import pytest

from tests import oracle_py as O

pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "reference_harness.json")
with open(GOLDEN) as f:
    CASES = json.load(f)["cases"]

# GPU arithmetic vs the bf16-operand oracle (fp32 accumulate, hi/mid/lo query
# split, hi/lo P and x splits): relative to max |out| (reference rel_error).
TOL_ARITH = 2e-4
# bf16 storage of W/KV vs the reference's double harness.
TOL_BF16 = 5e-2


def rel_err(got, want):
    scale = max(1e-12, np.abs(want).max())
    return float(np.abs(got - want).max() / scale)


def appended_rows(g, case, request=0):
    """K/V rows the GPU stored for the newest token (round-robin closed form)."""
    t = g.total_tokens(request) - 1
    c, kvp = case["chunk"], case["kvp"]
    rank = (t // c) % kvp
    row = (t // (c * kvp)) * c + t % c
    ks, vs = [], []
    for h in range(case["kv_heads"]):
        k, v = g.context(rank, h, request)
        ks.append(k[row])
        vs.append(v[row])
    return np.array(ks, dtype=np.float64), np.array(vs, dtype=np.float64)


def assert_within_one_bf16_ulp(got_bf16, want_double):
    """GPU rounds its fp32 projection to bf16; the oracle's double projection
    rounds to the same or the adjacent bf16 value."""
    want = O.round_bf16(want_double)
    ulp = np.ldexp(1.0, np.frexp(np.maximum(np.abs(want), 1e-30))[1] - 8)
    assert np.all(np.abs(got_bf16 - want) <= ulp * 1.0000001), np.abs(got_bf16 - want).max()


@pytest.fixture(scope="module")
def P():
    import paper_2507_07120_b200 as P
    return P


@pytest.mark.parametrize("case", CASES, ids=[c["name"] for c in CASES])
def test_harness_matches_oracle_and_reference(P, case):
    dims = (case["query_heads"], case["kv_heads"], case["head_size"])
    hidden = dims[0] * dims[2]
    g = P.DecodeHarness(dims, case["tpa"], case["kvp"], case["chunk"], case["seed"], batch=1,
                        capacity=case["context"] + 8)
    o = O.Harness(*dims, case["tpa"], case["kvp"], case["chunk"], case["seed"], bf16=True)
    rg, ro = P.Rng(case["grow_seed"]), O.Rng(case["grow_seed"])
    g.grow_random(case["context"], rg)
    o.grow_random(case["context"], ro)
    # grown cache is bit-identical (bf16 of the same mt19937_64 doubles)
    for r in range(case["kvp"]):
        assert g.effective_tokens(r) == o.effective_tokens(r)
        for h in range(case["kv_heads"]):
            k, v = g.context(r, h)
            np.testing.assert_array_equal(k, o.cache_rows(r, h, 0).astype(np.float32))
            np.testing.assert_array_equal(v, o.cache_rows(r, h, 1).astype(np.float32))
    errs = []
    for s in case["steps"]:
        x = np.array([rg.unit_draw() for _ in range(hidden)])
        np.testing.assert_array_equal(x, np.array(s["x"]))  # same stream as the reference
        x32 = x.astype(np.float32).astype(np.float64)
        got = g.step(x32)
        k_gpu, v_gpu = appended_rows(g, case)
        _, k_ref, v_ref = o.project(x32)
        assert_within_one_bf16_ulp(k_gpu, k_ref)
        assert_within_one_bf16_ulp(v_gpu, v_ref)
        # attention parity on identical stored operands (feed the GPU's bf16 rows)
        want_arith, _ = o.step_append(x32, k_gpu, v_gpu)
        want_ref = np.array(s["step"]).reshape(dims[0], dims[2])
        e_a, e_r = rel_err(got, want_arith), rel_err(got, want_ref)
        errs.append((e_a, e_r))
    print(case["name"], errs)
    for e_a, e_r in errs:
        assert e_a <= TOL_ARITH, f"arith err {errs}"
        assert e_r <= TOL_BF16, f"bf16 storage err {errs}"

    # round-robin bookkeeping and transcript follow the reference exactly
    assert g.total_tokens() == case["context"] + len(case["steps"])
    assert [g.effective_tokens(r) for r in range(case["kvp"])] == case["effective_tokens"]
    assert g.max_min_gap() == case["max_min_gap"]
    np.testing.assert_array_equal(g.transcript().reshape(-1), np.array(case["transcript"], dtype=np.int64))


def test_harness_shape_errors_match_reference(P):
    with pytest.raises(ValueError, match="multiple of kv_heads"):
        P.DecodeHarness((4, 3, 8), 1, 1, 16, 1)
    with pytest.raises(ValueError, match="tpa must divide kv_heads"):
        P.DecodeHarness((4, 2, 8), 4, 1, 16, 1)
    with pytest.raises(ValueError, match="divide the hidden width"):
        P.DecodeHarness((4, 2, 8), 2, 3, 16, 1)
    h = P.DecodeHarness((4, 2, 8), 2, 2, 16, 1)
    with pytest.raises(ValueError, match="nonempty context"):
        h.step(np.zeros(32))
    h.grow_random(4, P.Rng(116))
    with pytest.raises(ValueError, match="wrong width"):
        h.step(np.zeros(31))


def test_batched_requests_are_independent(P):
    """B requests in one GPU step == B reference harnesses (same seeded weights)."""
    dims, tpa, kvp, B = (16, 4, 128), 1, 2, 4
    g = P.DecodeHarness(dims, tpa, kvp, 16, 9, batch=B, capacity=300)
    oracles = [O.Harness(*dims, tpa, kvp, 16, 9, bf16=True) for _ in range(B)]
    for b in range(B):
        n = 100 + 37 * b  # ragged contexts
        g.grow_random(n, P.Rng(500 + b), request=b)
        oracles[b].grow_random(n, O.Rng(500 + b))
    rx = np.random.default_rng(3)
    case = {"chunk": 16, "kvp": kvp, "kv_heads": 4}
    for step in range(3):
        x = rx.uniform(-1, 1, size=(B, 16 * 128)).astype(np.float32)
        got = g.step(x)
        for b in range(B):
            k_gpu, v_gpu = appended_rows(g, case, b)
            want, _ = oracles[b].step_append(x[b].astype(np.float64), k_gpu, v_gpu)
            assert rel_err(got[b], want) <= TOL_ARITH


@pytest.mark.parametrize("dims,tpa,kvp,chunk,ctx", [
    ((16, 4, 16), 1, 16, 4, 300),     # kvp = 16: past the register-resident merge (MAXK = 8)
    ((32, 8, 16), 2, 16, 16, 700),    # two TPA groups x 16 KVP ranks = 32 slots
    ((64, 2, 8), 1, 64, 1, 200),      # kvp = 64 = validate_config max_gpus, chunk 1, empty ranks
])
def test_wide_kvp_local_pool_matches_oracle(P, dims, tpa, kvp, chunk, ctx):
    """kvp > 8 merges (local memory, merge.cuh MAXK = 64) against the oracle,
    including ranks whose shard is still empty (lse = -inf)."""
    g = P.DecodeHarness(dims, tpa, kvp, chunk, 77, batch=1, capacity=ctx + 8)
    o = O.Harness(*dims, tpa, kvp, chunk, 77, bf16=True)
    rg, ro = P.Rng(5), O.Rng(5)
    g.grow_random(ctx, rg)
    o.grow_random(ctx, ro)
    case = {"chunk": chunk, "kvp": kvp, "kv_heads": dims[1]}
    rx = np.random.default_rng(11)
    for _ in range(3):
        x = rx.uniform(-1, 1, size=dims[0] * dims[2]).astype(np.float32).astype(np.float64)
        got = g.step(x)
        k_gpu, v_gpu = appended_rows(g, case)
        want, _ = o.step_append(x, k_gpu, v_gpu)
        assert rel_err(got, want) <= TOL_ARITH
    assert [g.effective_tokens(r) for r in range(kvp)] == [o.effective_tokens(r) for r in range(kvp)]


def test_short_context_in_a_large_engine_plans_from_the_live_context(P):
    """The attention split plan follows the live context (engine.cpp
    live_splits), not the capacity: a 1M-token engine serving a 600-token
    context launches few, full-size work items -- and stays exact as the
    context grows across plan buckets."""
    dims = (32, 8, 128)
    g = P.DecodeHarness(dims, 1, 1, 16, 3, batch=2, capacity=1 << 20)
    o = [O.Harness(*dims, 1, 1, 16, 3, bf16=True) for _ in range(2)]
    for b in range(2):
        g.grow_random(600 + 300 * b, P.Rng(40 + b), request=b)
        o[b].grow_random(600 + 300 * b, O.Rng(40 + b))
    assert g.info()["attn_splits"] <= 2, g.info()  # 57 pages: items of >= 32 pages
    rx = np.random.default_rng(5)
    case = {"chunk": 16, "kvp": 1, "kv_heads": 8}
    for step in range(3):
        x = rx.uniform(-1, 1, size=(2, 4096)).astype(np.float32)
        got = g.step(x)
        for b in range(2):
            k_gpu, v_gpu = appended_rows(g, case, b)
            want, _ = o[b].step_append(x[b].astype(np.float64), k_gpu, v_gpu)
            assert rel_err(got[b], want) <= TOL_ARITH
