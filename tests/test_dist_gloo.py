"""Multi-process (world_size 2 and 4, gloo, CPU) check of the Helix fragment
exchange that the NCCL engine performs: every rank computes its KV shard's
(partial O, lse) fragment with the CPU oracle, packs it with the PRODUCT's
exchange layout (hx_exchange_layout -- the same host function the engine's
pack kernel and O-proj merge are planned from), exchanges slices with a real
all-to-all, merges its slice in canonical order, and the gathered slices must
equal the monolithic step (attention.hpp:460-510) to 1e-12."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _layout(q_per_group, hsz, kvp):
    import ctypes as C
    from paper_2507_07120_b200._lib import lib
    out = (C.c_int64 * (4 * kvp))()
    chunk = lib().hx_exchange_layout(q_per_group, hsz, kvp, out)
    assert chunk > 0
    return chunk, np.array(out[:], dtype=np.int64).reshape(kvp, 4)


def _worker(rank, world, port, dims, tpa, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from tests import oracle_py as O
    Q, K, D = dims
    kvp = world // tpa
    g, r = rank // kvp, rank % kvp
    h = O.Harness(Q, K, D, tpa, kvp, 16, 42)
    rng = O.Rng(112)
    h.grow_random(70, rng)
    x = rng.draws(Q * D)
    qall, _, _ = h.project(x)
    q_per_group, kv_per_group, q_per_kv = Q // tpa, K // tpa, Q // K
    # this rank's fragment: its shard, its group's heads (shard_attention, attention.hpp:375-396)
    frag_o = np.zeros((q_per_group, D))
    frag_lse = np.zeros(q_per_group)
    for kh in range(kv_per_group):
        keys = h.cache_rows(r, g * kv_per_group + kh, 0)
        vals = h.cache_rows(r, g * kv_per_group + kh, 1)
        for qi in range(q_per_kv):
            row = kh * q_per_kv + qi
            head = g * q_per_group + row
            o, lse = O.partial_head_attention(qall[head * D:(head + 1) * D], keys, vals)
            frag_o[row], frag_lse[row] = o, lse
    chunk, lay = _layout(q_per_group, D, kvp)
    flat = frag_o.reshape(-1)
    send = np.zeros((world, chunk))  # only the KVP group's peers receive data
    for p in range(kvp):
        e0, cnt, h0, nh = lay[p]
        send[g * kvp + p, :cnt] = flat[e0:e0 + cnt]
        send[g * kvp + p, cnt:cnt + nh] = frag_lse[h0:h0 + nh]
    recv = torch.zeros(world * chunk, dtype=torch.float64)
    dist.all_to_all_single(recv, torch.from_numpy(send.reshape(-1)).clone())
    recv = recv.numpy().reshape(world, chunk)[g * kvp:(g + 1) * kvp]
    e0, cnt, h0, nh = lay[r]
    merged = np.zeros(cnt)
    for e in range(cnt):
        head = (e0 + e) // D
        outs = recv[:, e:e + 1]
        lses = recv[:, cnt + head - h0]
        m, _ = O.merge_head_fragments(outs, lses)
        merged[e] = m[0]
    gathered = [torch.zeros(cnt, dtype=torch.float64) for _ in range(world)]
    dist.all_gather(gathered, torch.from_numpy(merged))
    if rank == 0:
        full = np.concatenate([t.numpy() for t in gathered])  # rank order == (g, r) order == flattened heads
        want, _ = h.step(x)
        err = np.abs(full - want.reshape(-1)).max() / np.abs(want).max()
        q.put(float(err))
    dist.destroy_process_group()


@pytest.mark.parametrize("dims,tpa,world", [((4, 2, 8), 1, 2), ((4, 2, 8), 2, 4), ((8, 4, 16), 1, 4), ((16, 4, 8), 2, 2)])
def test_exchange_across_processes(dims, tpa, world):
    ctx = mp.get_context("spawn")
    q = ctx.SimpleQueue()
    mp.start_processes(_worker, args=(world, _free_port(), dims, tpa, q), nprocs=world, join=True,
                       start_method="spawn")
    assert q.get() <= 1e-12
