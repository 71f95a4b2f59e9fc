"""world_size-2 gloo tests of the multi-GPU host logic (run on CPU).

* stream / KV-head sharding covers every stream exactly once;
* the sequence split + all-gather + LSE merge reproduces attention over the
  whole sequence (partials computed by the oracle's attend on each rank's
  shard, exchanged over torch.distributed, merged by sharding.gather_and_merge).
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2603_16435_b200 import sharding


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_stream_shards_partition():
    for n in (1, 7, 256):
        for w in (1, 2, 3, 8):
            covered = [i for r in range(w) for i in sharding.stream_shard(n, w, r)]
            assert covered == list(range(n))


def test_sequence_shards_layout():
    sh = sharding.sequence_shards(4, 1000, 16, 4)
    assert sh[0].init == (0, 4) and all(s.init == (0, 0) for s in sh[1:])
    assert sh[-1].local == (0, 16) and all(s.local == (0, 0) for s in sh[:-1])
    assert sum(s.comp[1] - s.comp[0] for s in sh) == 1000
    assert sum(s.tokens for s in sh) == 1020


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import oracle as O

    rng = O.Rng(99)
    ks = rng.stack(3, 32, 16, O.KEY)
    vs = rng.stack(2, 32, 16, O.VALUE)
    n_init, n_comp, n_local = 3, 301, 9
    ik, iv = rng.matrix(n_init, 16), rng.matrix(n_init, 16)
    lk, lv = rng.matrix(n_local, 16), rng.matrix(n_local, 16)
    g = np.random.default_rng(5)
    kcodes = g.integers(0, 32, (n_comp, 3)).astype(np.uint32)
    vcodes = g.integers(0, 32, (n_comp, 2)).astype(np.uint32)
    queries = rng.matrix(4, 16)
    shard = sharding.sequence_shards(n_init, n_comp, n_local, world)[rank]
    c0, c1 = shard.comp
    outs, lses = [], []
    for qi in range(4):
        o, lse = O.attend_segments(
            ks, vs, ik[slice(*shard.init)], iv[slice(*shard.init)], ks.pack(kcodes[c0:c1]), vs.pack(vcodes[c0:c1]),
            c1 - c0, lk[slice(*shard.local)], lv[slice(*shard.local)], queries[qi])
        outs.append(o)
        lses.append(lse)
    o_local = torch.tensor(np.stack(outs), dtype=torch.float64)
    l_local = torch.tensor(lses, dtype=torch.float64)
    o, lse = sharding.gather_and_merge(o_local, l_local)
    if rank == 0:
        ref = [O.attend_segments(ks, vs, ik, iv, ks.pack(kcodes), vs.pack(vcodes), n_comp, lk, lv, queries[qi])
               for qi in range(4)]
        err = max(float(np.abs(o[qi].numpy() - ref[qi][0]).max()) for qi in range(4))
        lerr = max(abs(float(lse[qi]) - ref[qi][1]) for qi in range(4))
        q.put((err, lerr))
    dist.barrier()
    dist.destroy_process_group()


def test_sequence_split_lse_combine_gloo():
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=240)
        assert p.exitcode == 0
    err, lerr = q.get(timeout=10)
    assert err < 1e-5 and lerr < 1e-9


def test_lse_merge_matches_monolithic_softmax():
    torch.manual_seed(0)
    logits = torch.randn(3, 50, dtype=torch.float64)
    v = torch.randn(50, 8, dtype=torch.float64)
    full_w = torch.softmax(logits, -1)
    o_full = full_w @ v
    lse_full = torch.logsumexp(logits, -1)
    parts = [(0, 20), (20, 21), (21, 50)]
    o_p = torch.stack([torch.softmax(logits[:, a:b], -1) @ v[a:b] for a, b in parts])
    l_p = torch.stack([torch.logsumexp(logits[:, a:b], -1) for a, b in parts])
    # an empty shard contributes nothing
    o_p = torch.cat([o_p, torch.zeros(1, 3, 8, dtype=torch.float64)])
    l_p = torch.cat([l_p, torch.full((1, 3), float("-inf"), dtype=torch.float64)])
    o, lse = sharding.lse_merge(o_p, l_p)
    assert torch.allclose(o, o_full) and torch.allclose(lse, lse_full)
