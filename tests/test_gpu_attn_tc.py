"""The experimental tcgen05 GQA kernel for quantised KV pages (attention_tc.cu,
opt-in with HX_ATTN_TC=1 -- the engine reads it at construction) against the
legacy kernel on the same engine contents: both compute on identical stored
operands (e4m3 / e2m1 x 2^e values are exact in f16, q and P split into two
f16 terms, fp32 accumulation), so hidden states and logits agree to the usual
2e-4 arithmetic bound, and the greedy ids are equal. Shapes: head size 128,
GQA groups of 4 (8-row items) and 16 (16-row items), contexts spanning several
128-token tiles per item, partial last tiles and pages, and two requests of
different lengths (ragged).
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

TOL = 2e-4


def rel(a, b):
    return float(np.abs(a - b).max() / max(1e-12, np.abs(b).max()))


def run(monkeypatch, tc, spec, kv, ctx):
    import paper_2507_07120_b200 as P
    monkeypatch.setenv("HX_ATTN_TC", "1" if tc else "0")
    g = P.HelixDecoder(spec, batch=2, capacity=ctx + 64, layers=1, vocab=300, use_graphs=False, kv_dtype=kv)
    g.init_weights(11, qkv="hash")
    g.fill_kv_hash(ctx, 11)
    toks = np.array([5, 77])
    out = []
    for _ in range(3):  # the second and third steps attend over the appended rows too
        nxt, logits, hidden = g.step(toks, want_logits=True, want_hidden=True)
        out.append((nxt.copy(), logits.copy(), hidden.copy()))
        toks = nxt
    del g
    return out


@pytest.mark.parametrize("kv", ["fp8", "fp4"])
@pytest.mark.parametrize("q_heads,kv_heads", [(8, 2), (16, 1)])
@pytest.mark.parametrize("ctx", [1000, 5003])
def test_tc_kernel_matches_legacy(monkeypatch, kv, q_heads, kv_heads, ctx):
    import paper_2507_07120_b200 as P
    spec = P.model.ModelSpec("tc", 1, 128 * q_heads, q_heads, kv_heads, 128, 512, 3, "gqa", 0, vocab=300)
    legacy = run(monkeypatch, False, spec, kv, ctx)
    tc = run(monkeypatch, True, spec, kv, ctx)
    for (n0, l0, h0), (n1, l1, h1) in zip(legacy, tc):
        assert rel(h1, h0) < TOL
        assert rel(l1, l0) < TOL
        np.testing.assert_array_equal(n1, n0)
