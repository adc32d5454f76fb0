"""GPU parity of FP8 (e4m3) KV pages (kv_dtype="fp8").

The oracle stores the KV in e4m3 exactly as the GPU does (round_e4m3: RNE,
saturating at +-448 -- checked against torch.float8_e4m3fn in
tests/test_fp8_oracle.py); weights stay bf16. Comparisons:
  * grown caches read back bit-identically (same mt19937_64 / hash values,
    same rounding), appended K/V within one e4m3 ulp of the oracle's double
    projection (the GPU rounds its fp32 projection);
  * attention on identical stored operands: the e4m3 values are exact in f16,
    q is split into three f16 terms and P into two, fp32 accumulation -> the
    same 2e-4 bound as the bf16 path;
  * full decode steps (hidden states / logits) 2e-3 on the first step;
  * against the reference's double harness the e4m3 storage itself costs
    ~2^-4 relative per element; bounded here at 0.15 (reported).
"""
import json
import os
import threading

import numpy as np
import pytest

from tests import oracle_py as O

pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "reference_harness.json")
with open(GOLDEN) as f:
    CASES = json.load(f)["cases"]

TOL_ARITH = 2e-4
TOL_FP8_STORAGE = 0.15


def rel_err(got, want):
    return float(np.abs(got - want).max() / max(1e-12, np.abs(want).max()))


def e4m3_ulp(x):
    a = np.maximum(np.abs(x), 2.0 ** -6)
    return np.ldexp(1.0, np.floor(np.log2(a)).astype(int) - 3)


def appended_rows(g, case, request=0):
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


@pytest.mark.parametrize("case", [c for c in CASES if c["context"] > 0][:8], ids=lambda c: c["name"])
def test_fp8_harness_matches_oracle(case):
    import paper_2507_07120_b200 as P
    dims = (case["query_heads"], case["kv_heads"], case["head_size"])
    hidden = dims[0] * dims[2]
    g = P.DecodeHarness(dims, case["tpa"], case["kvp"], case["chunk"], case["seed"], batch=1,
                        capacity=case["context"] + 8, kv_dtype="fp8")
    assert g.info()["kv_dtype"] == 1
    o = O.Harness(*dims, case["tpa"], case["kvp"], case["chunk"], case["seed"], bf16=True, kv_fp8=True)
    rg, ro = P.Rng(case["grow_seed"]), O.Rng(case["grow_seed"])
    g.grow_random(case["context"], rg)
    o.grow_random(case["context"], ro)
    for r in range(case["kvp"]):
        for h in range(case["kv_heads"]):
            k, v = g.context(r, h)
            np.testing.assert_array_equal(k, o.cache_rows(r, h, 0).astype(np.float32))
            np.testing.assert_array_equal(v, o.cache_rows(r, h, 1).astype(np.float32))
    errs = []
    for s in case["steps"]:
        x = np.array([rg.unit_draw() for _ in range(hidden)])
        x32 = x.astype(np.float32).astype(np.float64)
        got = g.step(x32)
        k_gpu, v_gpu = appended_rows(g, case)
        _, k_ref, v_ref = o.project(x32)
        want_k, want_v = O.round_e4m3(k_ref), O.round_e4m3(v_ref)
        assert np.all(np.abs(k_gpu - want_k) <= e4m3_ulp(want_k) * 1.0000001)
        assert np.all(np.abs(v_gpu - want_v) <= e4m3_ulp(want_v) * 1.0000001)
        want_arith, _ = o.step_append(x32, k_gpu, v_gpu)
        want_ref = np.array(s["step"]).reshape(dims[0], dims[2])
        errs.append((rel_err(got, want_arith), rel_err(got, want_ref)))
    print(case["name"], errs)
    for e_a, e_r in errs:
        assert e_a <= TOL_ARITH, errs
        assert e_r <= TOL_FP8_STORAGE, errs


@pytest.mark.parametrize("q,k,hsz,kvp", [(8, 2, 32, 2), (32, 2, 64, 1), (16, 1, 128, 4)])
def test_fp8_decode_step_matches_oracle(q, k, hsz, kvp):
    """Hash-filled FP8 cache, full decode step; includes GQA groups of 16 (two query chunks)."""
    import paper_2507_07120_b200 as P
    H, F, L, V, B = q * hsz, 256, 2, 700, 3
    spec = P.model.ModelSpec("fp8", L, H, q, k, hsz, F, 3, "gqa", 0, vocab=V)
    g = P.HelixDecoder(spec, tpa=1, kvp=kvp, batch=B, capacity=2100, layers=L, vocab=V, kv_dtype="fp8")
    g.init_weights(17, qkv="hash")
    g.fill_kv_hash(2000, 17)
    o = O.Model(H, q, k, hsz, F, L, V, tpa=1, kvp=kvp, batch=B, seed=17, qkv_hash=True, bf16=True, kv_fp8=True)
    for l in range(L):
        for b in range(B):
            o.grow_hash(l, b, 2000)
    tokens = np.array([1, 50, 699])
    for step in range(2):
        nxt, logits, hidden = g.step(tokens, want_logits=True, want_hidden=True)
        lo, ho, no = o.step(tokens)
        tol = 2e-3 if step == 0 else 2e-2
        e_h, e_l = rel_err(hidden, ho), rel_err(logits, lo)
        print(f"q={q} k={k} hsz={hsz} kvp={kvp} step={step} hidden={e_h:.2e} logits={e_l:.2e}")
        assert e_h <= tol and e_l <= tol
        tokens = no
    g.close()


def test_fp8_hash_fill_reads_back_exactly():
    """Device hash fill rounds to e4m3 exactly as the oracle (layer_oracle grow_hash)."""
    import ctypes
    import paper_2507_07120_b200 as P
    K, D = 2, 32
    spec = P.model.ModelSpec("fp8", 1, 256, 8, K, D, 256, 3, "gqa", 0, vocab=300)
    g = P.HelixDecoder(spec, tpa=1, kvp=2, batch=2, capacity=600, layers=1, vocab=300, kv_dtype="fp8")
    g.init_weights(5, qkv="hash")
    g.fill_kv_hash(530, 5)
    fp = ctypes.POINTER(ctypes.c_float)
    for b in range(2):
        for rank in range(2):
            toks = [t for t in range(530) if (t // 16) % 2 == rank]
            for h in range(K):
                k = np.zeros((len(toks), D), dtype=np.float32)
                v = np.zeros((len(toks), D), dtype=np.float32)
                assert P.lib().hx_read_kv(g._h, 0, b, rank, h, k.ctypes.data_as(fp), v.ctypes.data_as(fp)) == 0
                for row in (0, 1, 17, len(toks) - 1):
                    t = toks[row]
                    idx = [(((b * K + h) << 32) + t) * D + d for d in range(D)]
                    wk = np.array([O.hash_unit(5, (10 << 32) | 0, i) for i in idx])
                    wv = np.array([O.hash_unit(5, (11 << 32) | 0, i) for i in idx])
                    np.testing.assert_array_equal(k[row], O.round_e4m3(wk).astype(np.float32))
                    np.testing.assert_array_equal(v[row], O.round_e4m3(wv).astype(np.float32))
    g.close()


def test_fp8_loopback_pool_hopb():
    """One-rank-per-thread pool with FP8 pages and HOP-B per-request launches."""
    import paper_2507_07120_b200 as P
    from paper_2507_07120_b200.model import Loopback
    H, Q, K, D, F, L, V, B, kvp = 512, 16, 2, 32, 256, 1, 400, 2, 2
    spec = P.model.ModelSpec("fp8d", L, H, Q, K, D, F, 3, "gqa", 0, vocab=V)
    lb = Loopback(kvp)
    engines = [P.HelixDecoder(spec, tpa=1, kvp=kvp, batch=B, capacity=3000, layers=L, vocab=V, use_graphs=False,
                              hopb=True, pool=2, rank=r, loopback=lb, kv_dtype="fp8") for r in range(kvp)]
    for e in engines:
        e.init_weights(3, qkv="hash")
        e.fill_kv_hash(2500, 3)
    o = O.Model(H, Q, K, D, F, L, V, tpa=1, kvp=kvp, batch=B, seed=3, qkv_hash=True, bf16=True, kv_fp8=True)
    for b in range(B):
        o.grow_hash(0, b, 2500)
    tokens = np.array([4, 399])
    res = [None] * kvp
    errors = []

    def run(r):
        try:
            res[r] = engines[r].step(tokens, want_logits=True, want_hidden=True)
        except Exception as ex:  # surfaced below
            errors.append(ex)
    th = [threading.Thread(target=run, args=(r,), daemon=True) for r in range(kvp)]
    [t.start() for t in th]
    [t.join(timeout=120) for t in th]
    assert not errors, errors
    lo, ho, no = o.step(tokens)
    for r in range(kvp):
        assert rel_err(res[r][2], ho) <= 2e-3
    for e in engines:
        e.close()


def test_fp4_rejects_mla():
    """MLA latents are bf16 or FP8 (tests/test_gpu_mla_fp8.py); FP4 pages are GQA-only."""
    import paper_2507_07120_b200 as P
    spec = P.model.ModelSpec("mla", 1, 256, 16, 1, 16, 256, 3, "mla", 288, vocab=300)
    with pytest.raises(ValueError, match="FP4"):
        P.HelixDecoder(spec, batch=1, capacity=64, layers=1, vocab=300, kv_dtype="fp4")
