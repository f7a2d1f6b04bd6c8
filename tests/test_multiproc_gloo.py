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


# ---------------------------------------------------------------------------- build_sharded's exchanges
def _q64_int(x: float) -> int:
    """trunc(x * 2^64) of an exactly representable double, as a Python int (test stand-in arithmetic)."""
    from fractions import Fraction
    f = Fraction(x) * (1 << 64)
    t = abs(f.numerator) // f.denominator
    return t if f >= 0 else -t


def _pair(v: int):
    u = v & ((1 << 128) - 1)
    lo, hi = u & ((1 << 64) - 1), u >> 64
    return [lo - (1 << 64) if lo >= (1 << 63) else lo, hi - (1 << 64) if hi >= (1 << 63) else hi]


def _unpair(p) -> int:
    return oracle.i128([int(p[0]) & ((1 << 64) - 1), int(p[1]) & ((1 << 64) - 1)])


def _worker_build(rank, world, port, q, case):
    """MagicPIG.build_sharded's collective sequence (all-gather of the exact centering sums, device
    reduction, all-gather of the local MIPS radii, device max) with the device ops replaced by exact
    Python-integer stand-ins: every rank must end with the unsharded c and r^2."""
    _init(rank, world, port)
    import paper_2410_16179_b200.index as index
    from fractions import Fraction
    k, sink, local = case
    n, d = k.shape
    lo, ln = sharding.sequence_shard(n, world, rank, align=256)
    kf = synth.bf16_bits_to_f32(k).astype(np.float64)

    def in_d(i):
        return not (i < sink or i >= n - local)

    def fake_key_stats(cfg, kt, seq_offset, n_global, ks, cnt, ws):
        for j in range(d):
            s = sum(_q64_int(kf[seq_offset + i, j]) for i in range(kt.shape[2]) if in_d(seq_offset + i))
            ks[0, 0, j] = torch.tensor(_pair(s), dtype=torch.int64)
        cnt[0, 0] = sum(1 for i in range(kt.shape[2]) if in_d(seq_offset + i))

    def fake_reduce(mode, parts_sum, parts_cnt, P, B, Hkv, out_sum, out_cnt):
        if mode == 0:
            for j in range(d):
                out_sum[0, 0, j] = torch.tensor(_pair(sum(_unpair(parts_sum[p, 0, 0, j]) for p in range(P))),
                                                dtype=torch.int64)
            out_cnt[0, 0] = int(parts_cnt[:, 0, 0].sum())
        else:
            out_sum[0, 0] = torch.tensor(_pair(max(_unpair(parts_sum[p, 0, 0]) for p in range(P))),
                                         dtype=torch.int64)

    def fake_key_norms(cfg, kt, seq_offset, n_global, key_sum, count, center, r2, ws):
        cnt = int(count[0, 0])
        for j in range(d):
            mean = float(Fraction(_unpair(key_sum[0, 0, j]), 1 << 64)) / cnt if cnt else 0.0
            center[0, 0, j] = float(np.float32(mean))
        c = center[0, 0].numpy().astype(np.float64)
        best = 0
        for i in range(kt.shape[2]):
            if not in_d(seq_offset + i):
                continue
            x = synth.bf16_bits_to_f32(synth.bf16_bits_from_f32((kf[seq_offset + i] - c).astype(np.float32)))
            best = max(best, sum(_q64_int(float(xx) * float(xx)) for xx in x.astype(np.float64)))
        r2[0, 0] = torch.tensor(_pair(best), dtype=torch.int64)

    seen = {}

    def fake_build_tables(cfg, kt, seq_offset, n_global, W, center, r2, codes, key_norm, ws):
        seen["c"] = center[0, 0].numpy().copy()
        seen["r2"] = _unpair(r2[0, 0])

    index.B_.key_stats = fake_key_stats
    index.B_.reduce_stats = fake_reduce
    index.B_.key_norms = fake_key_norms
    index.B_.build_tables = fake_build_tables
    index.B_.codes_words = lambda cfg, B, H, n: 1
    index.B_.build_workspace_bytes = lambda cfg, B, H, n: 1
    index.B_.new_workspace = lambda nb, dev: torch.zeros(1, dtype=torch.uint8)
    obj = index.MagicPIG.__new__(index.MagicPIG)
    obj.cfg, obj.W, obj.buckets, obj._ws_build = None, None, False, None
    kt = torch.from_numpy(k[lo:lo + ln].view(np.int16)).view(torch.bfloat16).reshape(1, 1, ln, d)
    obj.build_sharded(kt, lo, n)
    q.put((rank, seen["c"], seen["r2"], (obj.seq_offset, obj.n_global, obj.shape)))
    dist.destroy_process_group()


@pytest.mark.parametrize("n", [600, 1000])
def test_build_sharded_gloo(n):
    wl = synth.Workload("gloob", 906, B=1, Hq=1, Hkv=1, n=n, K=6, L=20)
    k, _, _ = synth.make_unit(wl, 0, 0)
    sink, local = 4, 64
    ref = oracle.key_transform(k, sink, local, 1, 1)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker_build, args=(r, 2, port, q, (k, sink, local))) for r in range(2)]
    for p in ps:
        p.start()
    res = [q.get(timeout=300) for _ in ps]
    for p in ps:
        p.join(timeout=120)
    for rank, c, r2, meta in res:
        np.testing.assert_array_equal(c, ref["c"])  # global centering vector, bit for bit
        assert r2 == ref["r2_q"]                    # global MIPS radius (exact fixed point)
        lo, ln = sharding.sequence_shard(n, 2, rank, align=256)
        assert meta == (lo, n, (1, 1, ln))
