"""The drop-in's exact (fp64) path on the GPU against the reference's own
numbers: DecodeHarness with kv_dtype="f64" (HX_KV_F64) and the free functions
behind include/helixsim/exact_b200.hpp, held to the reference's tolerances
(test_attention.cpp: 1e-12 primitives, 1e-10 decode steps) -- and the
reference's OWN test file compiled unmodified against the drop-in header
(oracle/_ref/test_attention_b200, built by `make -C oracle ref`)."""
import json
import os
import subprocess

import numpy as np
import pytest

from tests import oracle_py as O

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
with open(os.path.join(ROOT, "tests", "golden", "reference_harness.json")) as f:
    CASES = json.load(f)["cases"]


def rel_err(got, want):
    return float(np.abs(np.asarray(got) - np.asarray(want)).max() / max(1e-12, np.abs(want).max()))


@pytest.fixture(scope="module")
def P():
    import paper_2507_07120_b200 as P
    return P


@pytest.mark.parametrize("case", CASES, ids=[c["name"] for c in CASES])
def test_exact_harness_matches_reference_golden(P, case):
    """Every golden decode case of the reference (attention.hpp's own double
    outputs) within its 1e-10 step tolerance; cache and transcript exact."""
    dims = (case["query_heads"], case["kv_heads"], case["head_size"])
    g = P.DecodeHarness(dims, case["tpa"], case["kvp"], case["chunk"], case["seed"], capacity=case["context"] + 8,
                        kv_dtype="f64")
    rg = P.Rng(case["grow_seed"])
    g.grow_random(case["context"], rg)
    o = O.Harness(*dims, case["tpa"], case["kvp"], case["chunk"], case["seed"], bf16=False)
    o.grow_random(case["context"], O.Rng(case["grow_seed"]))
    for r in range(case["kvp"]):
        for h in range(case["kv_heads"]):
            k, v = g.context(r, h)
            np.testing.assert_array_equal(k, o.cache_rows(r, h, 0))  # the reference's doubles, unrounded
            np.testing.assert_array_equal(v, o.cache_rows(r, h, 1))
    for s in case["steps"]:
        x = np.array([rg.unit_draw() for _ in range(dims[0] * dims[2])])
        want = np.array(s["step"]).reshape(dims[0], dims[2])
        mono = g.reference(x)  # same pre-append context as step() (test_attention.cpp:299-301)
        got = g.step(x)
        assert rel_err(got, want) <= 1e-10
        assert rel_err(got, mono) <= 1e-10
    assert g.total_tokens() == case["context"] + len(case["steps"])
    np.testing.assert_array_equal(g.transcript().reshape(-1), np.array(case["transcript"], dtype=np.int64))


def test_exact_harness_headline_shape_matches_double_oracle(P):
    """Q = 32, K = 8, Hsz = 128 (configs[1]'s attention), 8k context, KVP 4 x TPA 2."""
    dims, tpa, kvp, ctx = (32, 8, 128), 2, 4, 8192
    g = P.DecodeHarness(dims, tpa, kvp, 16, 42, capacity=ctx + 8, kv_dtype="f64")
    o = O.Harness(*dims, tpa, kvp, 16, 42, bf16=False)
    g.grow_random(ctx, P.Rng(1000))
    o.grow_random(ctx, O.Rng(1000))
    rx = np.random.default_rng(4)
    for _ in range(2):
        x = rx.uniform(-1, 1, 4096)
        want, _ = o.step(x)
        assert rel_err(g.step(x), want) <= 1e-10


def test_free_functions_match_the_oracle(P):
    """partial_head_attention / reference_attention / merge_head_fragments on
    caller operands (attention.hpp:43-137) within 1e-12, identities bitwise."""
    from paper_2507_07120_b200 import exact as X
    rng = np.random.default_rng(101)
    for width, tokens in ((16, 64), (24, 96), (128, 1000), (8, 1)):
        q = rng.uniform(-1, 1, width)
        k, v = rng.uniform(-1, 1, (tokens, width)), rng.uniform(-1, 1, (tokens, width))
        out, lse = X.partial_head_attention(q, k, v)
        w_out, w_lse = O.partial_head_attention(q, k, v)
        assert rel_err(out, w_out) <= 1e-12 and abs(lse - w_lse) <= 1e-12 * max(1.0, abs(w_lse))
        # a single full shard merges to the reference bitwise (test_attention.cpp:95-106)
        m, ml = X.merge_head_fragments(out[None, :], np.array([lse]))
        np.testing.assert_array_equal(m, X.reference_attention(q, k, v))
        assert ml == lse
    # one token: the output IS its value row (test_attention.cpp:63-72)
    q, k1, v1 = rng.uniform(-1, 1, 8), rng.uniform(-1, 1, (1, 8)), rng.uniform(-1, 1, (1, 8))
    np.testing.assert_array_equal(X.reference_attention(q, k1, v1), v1[0])
    # empty shard: the identity element; reference_attention throws
    out, lse = X.partial_head_attention(q, np.zeros((0, 8)), np.zeros((0, 8)))
    assert lse == -np.inf and not out.any()
    with pytest.raises(ValueError, match="attention needs >= 1 context token"):
        X.reference_attention(q, np.zeros((0, 8)), np.zeros((0, 8)))


def test_merge_is_bitwise_order_invariant(P):
    """Canonical order (attention.hpp:90-102) incl. equal-lse ties broken by coefficients."""
    from paper_2507_07120_b200 import exact as X
    rng = np.random.default_rng(104)
    q = rng.uniform(-1, 1, 16)
    outs, lses = [], []
    for tokens in (40, 1, 17, 0, 64, 0, 5):
        k, v = rng.uniform(-1, 1, (tokens, 16)), rng.uniform(-1, 1, (tokens, 16))
        o, l = X.partial_head_attention(q, k, v)
        outs.append(o)
        lses.append(l)
    outs.append(outs[2] * 0.5)  # an exact lse tie with a different coefficient vector
    lses.append(lses[2])
    outs, lses = np.array(outs), np.array(lses)
    base = X.merge_head_fragments(outs, lses)
    w_out, w_lse = O.merge_head_fragments(outs, lses)
    assert rel_err(base[0], w_out) <= 1e-12
    perm_rng = np.random.default_rng(7)
    for _ in range(10):
        p = perm_rng.permutation(len(lses))
        m = X.merge_head_fragments(outs[p], lses[p])
        np.testing.assert_array_equal(m[0], base[0])
        assert m[1] == base[1]
    with pytest.raises(ValueError, match="all fragments empty"):
        X.merge_head_fragments(np.zeros((2, 4)), np.array([-np.inf, -np.inf]))


def test_reference_test_file_passes_against_the_dropin():
    """/root/reference/proj/tests/test_attention.cpp, unmodified, compiled with
    tests/cpp/dropin first on the include path (its `#include
    "helixsim/attention.hpp"` resolves to exact_b200.hpp) and linked to
    libhelix_b200.so: all of the reference's own cases pass on the GPU."""
    exe = os.path.join(ROOT, "oracle", "_ref", "test_attention_b200")
    if not os.path.exists(exe):
        pytest.skip("built from /root/reference sources by `make -C oracle ref` (not present here)")
    out = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    print(out.stdout[-2000:])
    assert out.returncode == 0, out.stdout[-4000:] + out.stderr[-2000:]
    assert "failed: 0" in out.stdout.splitlines()[-1]
