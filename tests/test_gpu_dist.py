"""Distributed Helix pool on ONE B200: tpa*kvp engines in loopback mode (one
host thread per rank, HX_POOL_LOOPBACK) run the same sharded code as the NCCL
process-per-GPU pool -- per-rank KV shard, TPA-group QKV slice, fragment pack
+ all-to-all + fused LSE merge into the O-proj, TP O-proj/FFN with
AllReduce, vocabulary-sharded LM head with max-AllReduce -- and are checked
against the CPU oracle (oracle/layer_oracle.hpp). Only the NCCL transport
calls themselves are not exercised here."""
import threading

import numpy as np
import pytest

from tests import oracle_py as O

pytestmark = pytest.mark.gpu


def rel_err(got, want):
    return float(np.abs(got - want).max() / max(1e-12, np.abs(want).max()))


@pytest.mark.parametrize("tpa,kvp,hopb", [(1, 2, False), (2, 2, False), (1, 4, True), (2, 1, False), (2, 2, True),
                                              (1, 16, False)])
def test_loopback_pool_matches_oracle(tpa, kvp, hopb):
    import paper_2507_07120_b200 as P
    from paper_2507_07120_b200.model import Loopback
    H, Q, K, D, F, L, V, B = 256, 8, 2, 32, 512, 2, 1000, 3
    spec = P.model.ModelSpec("test", L, H, Q, K, D, F, 3, "gqa", 0, vocab=V)
    n = tpa * kvp
    lb = Loopback(n)
    engines = [P.HelixDecoder(spec, tpa=tpa, kvp=kvp, chunk_size=16, batch=B, capacity=400, layers=L, vocab=V,
                              use_graphs=False, hopb=hopb, pool=2, rank=r, loopback=lb) for r in range(n)]
    o = O.Model(H, Q, K, D, F, L, V, tpa=tpa, kvp=kvp, chunk=16, batch=B, seed=4321, bf16=True)
    # launches per step (engine.cpp launches_per_step): embed + LM head x2 + argmax; per layer
    # QKV x2, attention [+ split reduce with the device push under HOP-B off], flag wait,
    # O x2 (the LSE combine fused into the O-projection GEMV), residual, gate/up x2, down x2, residual
    info = engines[0].info()
    assert info["exchange"] == (3 if hopb else 2)
    assert info["kernels_per_step"] == 4 + L * (10 + 3)  # attention, split reduce or HOP-B stream reducer, flag wait
    for e in engines:
        e.init_weights(4321, qkv="mt19937")
    for l in range(L):
        for b in range(B):
            cnt = 40 + 13 * b + 7 * l
            for e in engines:  # every rank replays the same stream; each keeps its own shard
                e.grow_random(l, b, cnt, P.Rng(100 * l + b))
            o.grow_random(l, b, cnt, O.Rng(100 * l + b))
    tokens = np.array([5, 17, 999])
    for step in range(2):
        results = [None] * n
        errors = []

        def run(r):
            try:
                results[r] = engines[r].step(tokens, want_logits=True, want_hidden=True)
            except Exception as ex:  # surfaced below
                errors.append(ex)
        th = [threading.Thread(target=run, args=(r,), daemon=True) for r in range(n)]
        [t.start() for t in th]
        [t.join(timeout=120) for t in th]
        assert not any(t.is_alive() for t in th), "loopback ranks did not finish (collective deadlock)"
        assert not errors, errors
        lo, ho, no = o.step(tokens)
        tol = 2e-3 if step == 0 else 2e-2
        vl = engines[0].vocab_local
        for r in range(n):
            nxt, logits, hidden = results[r]
            assert rel_err(hidden, ho) <= tol, (r, rel_err(hidden, ho))
            shard = lo[:, r * vl: min(V, (r + 1) * vl)]
            assert rel_err(logits[:, :shard.shape[1]], shard) <= tol
            scale = np.abs(lo).max()
            for b in range(B):
                top2 = np.sort(lo[b])[-2:]
                if top2[1] - top2[0] > 1e-3 * scale:
                    assert nxt[b] == no[b]
        # all ranks agree bit-for-bit (identical all-reduce results)
        for r in range(1, n):
            np.testing.assert_array_equal(results[r][0], results[0][0])
            np.testing.assert_array_equal(results[r][2], results[0][2])
        tokens = no
    for e in engines:
        e.close()


def test_loopback_hopb_long_context_group16():
    """HOP-B at a long context with many small work items (HX_ATTN_SPLIT): the
    request-ordered attention launch reduces and pushes every stream from
    inside the kernel -- every split of every stream must be counted exactly
    once. GQA group 16 runs the W16 consumers (each KV page read once for 16
    query heads)."""
    import paper_2507_07120_b200 as P
    from paper_2507_07120_b200.model import Loopback
    H, Q, K, D, F, L, V, B, kvp = 1024, 32, 2, 32, 512, 1, 500, 4, 2
    S = 40000
    spec = P.model.ModelSpec("test16", L, H, Q, K, D, F, 3, "gqa", 0, vocab=V)
    lb = Loopback(kvp)
    import os
    old = os.environ.get("HX_ATTN_SPLIT")
    os.environ["HX_ATTN_SPLIT"] = "8,8"  # small items: per-request split count (156) != batched (148)
    try:
        engines = [P.HelixDecoder(spec, tpa=1, kvp=kvp, chunk_size=16, batch=B, capacity=S + 64, layers=L, vocab=V,
                                  use_graphs=False, hopb=True, pool=2, rank=r, loopback=lb) for r in range(kvp)]
    finally:
        if old is None:
            del os.environ["HX_ATTN_SPLIT"]
        else:
            os.environ["HX_ATTN_SPLIT"] = old
    assert engines[0].info()["exchange"] == 3  # HOP-B: reduce + push inside the attention kernel
    o = O.Model(H, Q, K, D, F, L, V, tpa=1, kvp=kvp, chunk=16, batch=B, seed=77, qkv_hash=True, bf16=True)
    for e in engines:
        e.init_weights(77, qkv="hash")
        e.fill_kv_hash(S, 77)
    for b in range(B):
        o.grow_hash(0, b, S)
    tokens = np.array([1, 2, 3, 499])
    results = [None] * kvp
    errors = []

    def run(r):
        try:
            results[r] = engines[r].step(tokens, want_logits=True, want_hidden=True)
        except Exception as ex:  # surfaced below
            errors.append(ex)
    th = [threading.Thread(target=run, args=(r,), daemon=True) for r in range(kvp)]
    [t.start() for t in th]
    [t.join(timeout=300) for t in th]
    assert not any(t.is_alive() for t in th), "loopback ranks did not finish"
    assert not errors, errors
    lo, ho, no = o.step(tokens)
    for r in range(kvp):
        assert rel_err(results[r][2], ho) <= 2e-3, (r, rel_err(results[r][2], ho))
    for e in engines:
        e.close()


def test_loopback_pool_large_batch_tcgen05():
    """Batch 20 (> 16): the sharded pool's GEMVs (TP partial stores, residual adds
    after the AllReduce) run on tcgen05 with the tcgen05 x-fragment layout."""
    import paper_2507_07120_b200 as P
    from paper_2507_07120_b200.model import Loopback
    H, Q, K, D, F, L, V, B, kvp = 256, 8, 2, 32, 512, 1, 1000, 20, 2
    spec = P.model.ModelSpec("test", L, H, Q, K, D, F, 3, "gqa", 0, vocab=V)
    lb = Loopback(kvp)
    engines = [P.HelixDecoder(spec, tpa=1, kvp=kvp, chunk_size=16, batch=B, capacity=300, layers=L, vocab=V,
                              use_graphs=False, pool=2, rank=r, loopback=lb) for r in range(kvp)]
    o = O.Model(H, Q, K, D, F, L, V, tpa=1, kvp=kvp, chunk=16, batch=B, seed=55, qkv_hash=True, bf16=True)
    for e in engines:
        e.init_weights(55, qkv="hash")
        e.fill_kv_hash(200, 55)
    for b in range(B):
        o.grow_hash(0, b, 200)
    tokens = (np.arange(B) * 37 + 1) % V
    results = [None] * kvp
    errors = []

    def run(r):
        try:
            results[r] = engines[r].step(tokens, want_logits=True, want_hidden=True)
        except Exception as ex:  # surfaced below
            errors.append(ex)
    th = [threading.Thread(target=run, args=(r,), daemon=True) for r in range(kvp)]
    [t.start() for t in th]
    [t.join(timeout=120) for t in th]
    assert not errors, errors
    lo, ho, no = o.step(tokens)
    for r in range(kvp):
        assert rel_err(results[r][2], ho) <= 2e-3, (r, rel_err(results[r][2], ho))
    for e in engines:
        e.close()


@pytest.mark.parametrize("hopb,graphs", [(False, False), (True, False), (False, True), (True, True)])
def test_nccl_pool_single_rank_matches_local(hopb, graphs):
    """The NCCL transport itself on the one GPU available: a one-rank NCCL pool
    (ncclCommInitRank + ncclCommSplit, grouped send/recv all-to-all to itself,
    ncclAllReduce sum and max) runs the distributed code path end to end and
    must agree with the local pool on the same weights and cache."""
    import paper_2507_07120_b200 as P
    from paper_2507_07120_b200.model import nccl_unique_id
    H, Q, K, D, F, L, V, B = 256, 8, 2, 32, 512, 2, 1000, 3
    spec = P.model.ModelSpec("test", L, H, Q, K, D, F, 3, "gqa", 0, vocab=V)
    outs = []
    for pool in (0, 1):
        kw = dict(pool=1, rank=0, nccl_id=nccl_unique_id(), hopb=hopb) if pool else {}
        g = P.HelixDecoder(spec, tpa=1, kvp=1, batch=B, capacity=400, layers=L, vocab=V, use_graphs=graphs, **kw)
        g.init_weights(77, qkv="hash")
        g.fill_kv_hash(300, 77)
        g.step(np.array([3, 4, 5]))  # a first step (captures the graph when enabled)
        outs.append(g.step(np.array([3, 4, 5]), want_logits=True, want_hidden=True))
        g.close()
    assert rel_err(outs[1][2], outs[0][2]) <= 1e-5
    assert rel_err(outs[1][1], outs[0][1]) <= 1e-5
    np.testing.assert_array_equal(outs[1][0], outs[0][0])


def _gpu_count():
    try:
        import torch
        return torch.cuda.device_count()
    except Exception:
        return 0


def _nccl_pool_rank(rank, n, uid, hopb, graphs, q):
    """One process = one GPU = one rank of the KVP = n pool (HX_POOL_NCCL)."""
    try:
        import paper_2507_07120_b200 as P
        H, Q, K, D, F, L, V, B = 256, 8, 2, 32, 512, 2, 1000, 3
        spec = P.model.ModelSpec("test", L, H, Q, K, D, F, 3, "gqa", 0, vocab=V)
        g = P.HelixDecoder(spec, tpa=1, kvp=n, batch=B, capacity=400, layers=L, vocab=V, device=rank,
                           use_graphs=graphs, hopb=hopb, pool=1, rank=rank, nccl_id=uid)
        assert g.info()["comm_ranks"] == n
        g.init_weights(77, qkv="hash")
        g.fill_kv_hash(300, 77)
        out = [g.step(np.array([3, 4, 5]), want_logits=True, want_hidden=True)]
        out.append(g.step(out[0][0], want_logits=True, want_hidden=True))
        g.close()
        q.put((rank, out, None))
    except Exception as ex:  # reported to the parent
        q.put((rank, None, repr(ex)))


@pytest.mark.skipif(_gpu_count() < 2, reason="needs >= 2 GPUs (one process per GPU)")
@pytest.mark.parametrize("hopb,graphs", [(False, True), (True, False), (True, True)])
def test_nccl_pool_two_gpus_matches_oracle(hopb, graphs):
    """A real two-process NCCL pool (KVP = 2, TPF = 2): grouped send/recv
    all-to-all of the fragment slices between GPUs, ncclAllReduce of the TP
    partials, vocab-sharded argmax -- against the oracle's sharded decode."""
    import multiprocessing as mp
    from paper_2507_07120_b200.model import nccl_unique_id
    n = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    uid = nccl_unique_id()
    procs = [ctx.Process(target=_nccl_pool_rank, args=(r, n, uid, hopb, graphs, q)) for r in range(n)]
    [p.start() for p in procs]
    res = {}
    for _ in range(n):
        r, out, err = q.get(timeout=300)
        assert err is None, (r, err)
        res[r] = out
    [p.join(timeout=60) for p in procs]
    H, Q, K, D, F, L, V, B = 256, 8, 2, 32, 512, 2, 1000, 3
    o = O.Model(H, Q, K, D, F, L, V, tpa=1, kvp=n, chunk=16, batch=B, seed=77, qkv_hash=True, bf16=True)
    for l in range(L):
        for b in range(B):
            o.grow_hash(l, b, 300)
    tokens = np.array([3, 4, 5])
    for step in range(2):
        lo, ho, no = o.step(tokens)
        tol = 2e-3 if step == 0 else 2e-2
        for r in range(n):
            nxt, logits, hidden = res[r][step]
            assert rel_err(hidden, ho) <= tol, (r, step, rel_err(hidden, ho))
        np.testing.assert_array_equal(res[1][step][2], res[0][step][2])
        tokens = no


@pytest.mark.parametrize("pool,kvp,hopb", [(0, 2, False), (0, 4, False), (2, 2, False), (2, 2, True), (2, 4, False)])
def test_fused_combine_is_bit_identical_to_merge_kernel(pool, kvp, hopb, monkeypatch):
    """The LSE combine inside the O-projection GEMV (GemvParams::merge, gemv.cu
    merge_prologue) merges in the same canonical order as the merge kernels it
    replaces (misc.cu xprep_merge_local / xprep_merge_recv): decode steps are
    bit-identical with HX_FUSED_COMBINE=0, and one launch per layer shorter."""
    import paper_2507_07120_b200 as P
    from paper_2507_07120_b200.model import Loopback
    H, Q, K, D, F, L, V, B = 256, 8, 2, 32, 512, 2, 1000, 3
    spec = P.model.ModelSpec("test", L, H, Q, K, D, F, 3, "gqa", 0, vocab=V)
    out, launches = {}, {}
    for mode in ("0", "1"):
        monkeypatch.setenv("HX_FUSED_COMBINE", mode)
        n = kvp if pool else 1
        lb = Loopback(n) if pool else None
        kw = dict(pool=2, loopback=lb) if pool else {}
        engines = [P.HelixDecoder(spec, tpa=1, kvp=kvp, chunk_size=16, batch=B, capacity=400, layers=L, vocab=V,
                                  use_graphs=False, hopb=hopb, rank=r, **kw) for r in range(n)]
        launches[mode] = engines[0].info()["kernels_per_step"]
        for e in engines:
            e.init_weights(77, qkv="hash")
            e.fill_kv_hash(150 + 17 * kvp, 77)
        tokens = np.array([5, 17, 999])
        res = []
        for step in range(2):
            results = [None] * n
            errors = []

            def run(r):
                try:
                    results[r] = engines[r].step(tokens, want_logits=True, want_hidden=True)
                except Exception as ex:  # surfaced below
                    errors.append(ex)
            th = [threading.Thread(target=run, args=(r,), daemon=True) for r in range(n)]
            [t.start() for t in th]
            [t.join(timeout=120) for t in th]
            assert not any(t.is_alive() for t in th) and not errors, errors
            res.append(results[0])
            tokens = results[0][0]
        out[mode] = res
        for e in engines:
            e.close()
    assert launches["0"] == launches["1"] + L
    for a, b in zip(out["0"], out["1"]):
        for x, y in zip(a, b):
            np.testing.assert_array_equal(x, y)
