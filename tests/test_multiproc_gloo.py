"""World-size-2 gloo tests (CPU) of the multi-GPU host logic: sharding plans,
the all-gather layout, and MagicPIG.decode_sharded's collective sequence, with
the device ops replaced by oracle stand-ins (test infrastructure only)."""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import synth
from paper_2410_16179_b200 import sharding


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _init(rank, world, port):
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)


def test_sequence_shard_partition():
    for n in [1, 1000, 1024, 16384, 131072 + 37]:
        for P in [1, 2, 3, 4, 8]:
            covered = []
            for r in range(P):
                lo, ln = sharding.sequence_shard(n, P, r)
                covered.extend(range(lo, lo + ln))
                if r < P - 1 and ln:
                    assert lo % 1024 == 0
            assert covered == list(range(n))


def test_head_shard_partition():
    for H in [1, 8, 64]:
        for P in [1, 2, 4, 8]:
            heads = []
            for r in range(P):
                h0, h1 = sharding.head_shard(H, P, r)
                heads.extend(range(h0, h1))
            assert heads == list(range(H))


def _worker_gather(rank, world, port, q):
    _init(rank, world, port)
    t = torch.arange(6, dtype=torch.int64).reshape(2, 3) + 100 * rank
    g = sharding.all_gather_stacked(t)
    q.put((rank, g.numpy()))
    dist.destroy_process_group()


def test_all_gather_stacked_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker_gather, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = [q.get(timeout=120) for _ in ps]
    for p in ps:
        p.join(timeout=120)
    for rank, g in res:
        assert g.shape == (2, 2, 3)
        for r in range(2):
            np.testing.assert_array_equal(g[r], np.arange(6).reshape(2, 3) + 100 * r)


def _worker_decode(rank, world, port, q, case):
    """Sequence-sharded decode through MagicPIG.decode_sharded with oracle stand-ins."""
    _init(rank, world, port)
    import paper_2410_16179_b200.index as index
    from paper_2410_16179_b200 import binding
    k, v, qq, W, K, L, sink, local = case
    n = k.shape[0]
    G = qq.shape[0]
    full = oracle.decode_unit(k, v, qq, W, K, L, 1, 1, 2, sink, local)
    lo, ln = sharding.sequence_shard(n, world, rank, align=256)

    def fake_decode(self, qt, kt, vt, out=None, partial=None, s_count=None, s_mask=None):
        # per-shard partial state of the unsharded sample (global S and log u)
        for g in range(G):
            e = oracle.estimate(qq[g], k[lo:lo + ln], v[lo:lo + ln], full["in_s"][g, lo:lo + ln],
                                full["logu"][g, lo:lo + ln])
            partial[g, 0] = e["m"]
            partial[g, 1] = e["s"]
            partial[g, 2:] = torch.from_numpy(e["a"])
        return partial

    def fake_merge(parts, out):
        P, BH, _ = parts.shape
        for r in range(BH):
            out.view(BH, -1)[r] = torch.from_numpy(oracle.merge_partials(parts[:, r].double().numpy()))

    index.MagicPIG.decode = fake_decode
    binding.merge_partials = fake_merge
    index.B_.merge_partials = fake_merge
    obj = index.MagicPIG.__new__(index.MagicPIG)
    qt = torch.zeros((1, G, 128), dtype=torch.bfloat16)
    kt = torch.zeros((1, 1, ln, 128), dtype=torch.bfloat16)
    out = obj.decode_sharded(qt, kt, kt)
    q.put((rank, out.numpy()[0], full["out"]))
    dist.destroy_process_group()


@pytest.mark.parametrize("n", [700, 1300])
def test_decode_sharded_gloo(n):
    wl = synth.Workload("gloo", 905, B=1, Hq=2, Hkv=1, n=n, K=6, L=20)
    k, v, qq = synth.make_unit(wl, 0, 0)
    W = synth.make_projections(6, 20, 1)
    case = (k, v, qq, W, 6, 20, 4, 64)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker_decode, args=(r, 2, port, q, case)) for r in range(2)]
    for p in ps:
        p.start()
    res = [q.get(timeout=300) for _ in ps]
    for p in ps:
        p.join(timeout=120)
    outs = {}
    for rank, out, ref in res:
        np.testing.assert_allclose(out, ref, rtol=1e-5, atol=1e-6)
        outs[rank] = out
    np.testing.assert_array_equal(outs[0], outs[1])  # bit-identical on every rank
