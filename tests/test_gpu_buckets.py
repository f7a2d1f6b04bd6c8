"""GPU parity of the bucketed hash tables (the paper's HT as inverted lists, P:102,
P:107) against the CPU oracle: the bucket contents
are exactly the keys with that code, and decoding through the buckets gives the
same S (bit-exact) and outputs within 2e-3 as the oracle (reading R18)."""
from __future__ import annotations

import numpy as np
import pytest

import oracle
import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

TOL = 2e-3


def _dev():
    if not torch.cuda.is_available():
        pytest.fail("GPU tests need a CUDA device (no fallback)")
    return torch.device("cuda:0")


def _bf(a):
    return torch.from_numpy(np.ascontiguousarray(a).view(np.int16)).view(torch.bfloat16).to(_dev())


def _pkg():
    import paper_2410_16179_b200 as pkg
    return pkg


def _rel_err(got, ref):
    den = np.max(np.abs(ref))
    return float(np.max(np.abs(got - ref)) / den) if den > 0 else float(np.max(np.abs(got)))


CASES = [
    # name, n, B, Hq, Hkv, K, L, center, mips, minc, sink, local
    ("C1", 1024, 1, 1, 1, 10, 150, 1, 1, 2, 4, 64),
    ("ragged", 2500, 1, 4, 1, 10, 150, 1, 1, 2, 4, 64),
    ("mips0", 3000, 1, 4, 2, 10, 150, 1, 0, 2, 4, 64),
    ("k8l75", 2049, 2, 8, 2, 8, 75, 1, 1, 2, 4, 64),
    ("k11l300", 1500, 1, 2, 1, 11, 300, 1, 1, 2, 4, 64),
    ("k3l5", 700, 1, 2, 2, 3, 5, 1, 1, 2, 0, 0),
    ("minc1", 1300, 1, 4, 1, 9, 20, 1, 1, 1, 4, 24),
    ("k14", 900, 1, 2, 1, 14, 6, 1, 1, 2, 2, 8),
    ("allstatic", 60, 1, 4, 1, 10, 150, 1, 1, 2, 4, 64),
    ("tiny", 37, 1, 1, 1, 2, 3, 1, 1, 2, 1, 1),
    ("manyunits", 3000, 16, 32, 8, 8, 20, 1, 1, 2, 4, 64),
    ("longg8", 20000, 1, 8, 1, 6, 16, 1, 1, 2, 4, 64),
    ("ids16max", 65536, 1, 2, 1, 7, 10, 1, 1, 2, 4, 64),  # largest n with uint16 ids (id 65535)
    ("ids32", 70001, 1, 2, 1, 6, 12, 1, 1, 2, 4, 64),     # n > 65536: int32 ids
]


def _build(wl, k, W):
    pkg = _pkg()
    tk = _bf(k)
    mp = pkg.MagicPIG(torch.from_numpy(W).to(_dev()), K=wl.K, L=wl.L, center=wl.center, mips=wl.mips,
                      min_collisions=wl.min_collisions, sink=wl.sink, local=wl.local, buckets=True).build(tk)
    return mp, tk


@pytest.mark.parametrize("case", CASES, ids=[c[0] for c in CASES])
def test_bucketed_decode_parity(case):
    name, n, B, Hq, Hkv, K, L, center, mips, minc, sink, local = case
    wl = synth.Workload(name, 1700 + CASES.index(case), B=B, Hq=Hq, Hkv=Hkv, n=n, K=K, L=L, center=center,
                        mips=mips, min_collisions=minc, sink=sink, local=local)
    k, v, q = synth.make_batch(wl)
    W = synth.make_projections(K, L, mips)
    mp, tk = _build(wl, k, W)
    tv, tq = _bf(v), _bf(q)
    s_count = torch.zeros((B, Hq), dtype=torch.int32, device=_dev())
    nw = (n + 31) // 32
    sm = torch.zeros((B, Hq, nw), dtype=torch.int32, device=_dev())
    out = mp.decode(tq, tk, tv, s_count=s_count, s_mask=sm)
    torch.cuda.synchronize()
    assert mp.status() == 0 and mp.status("build") == 0
    out, s_count, sm = out.cpu().numpy(), s_count.cpu().numpy(), sm.cpu().numpy().view(np.uint32)
    refs = oracle.decode_batch(k, v, q, W, K, L, center, mips, minc, sink, local)
    G = Hq // Hkv
    for b in range(B):
        for h in range(Hkv):
            ref = refs[b][h]
            for g in range(G):
                row = h * G + g
                assert int(s_count[b, row]) == int(ref["s_count"][g]), (b, row)
                bits = np.unpackbits(sm[b, row].view(np.uint8), bitorder="little")[:n]
                np.testing.assert_array_equal(bits, (ref["in_s"][g] == 1).astype(np.uint8))
                if ref["s_count"][g] > 0 or np.any(ref["in_s"][g] == 2):
                    assert _rel_err(out[b, row], ref["out"][g]) <= TOL


def test_bucket_contents_are_the_code_classes():
    """offsets/ids of every table: bucket c holds exactly the keys whose oracle code for that table is c."""
    pkg = _pkg()
    wl = synth.Workload("bk", 1800, B=1, Hq=2, Hkv=2, n=1900, K=7, L=12)
    k, v, q = synth.make_batch(wl)
    W = synth.make_projections(wl.K, wl.L, wl.mips)
    mp, _ = _build(wl, k, W)
    tables = mp.buf.tables.cpu().numpy()
    nb = 1 << wl.K
    # n <= 65536: the ids are uint16 (the paper's int16 table entries), ceil(L*n/2) words
    per_unit = wl.L * (nb + 1) + (wl.L * wl.n + 1) // 2
    assert tables.size == pkg.binding.bucket_tables_words(mp.cfg, 1, 2, wl.n) == 2 * per_unit
    for h in range(2):
        t_ = oracle.key_transform(k[0, h], wl.sink, wl.local, 1, 1)
        codes = oracle.encode_keys(t_["xbar"], W, wl.K, wl.L)  # [n][L]
        tu = tables[h * per_unit:(h + 1) * per_unit]
        offs = tu[:wl.L * (nb + 1)].reshape(wl.L, nb + 1)
        ids = np.ascontiguousarray(tu[wl.L * (nb + 1):]).view(np.uint16)[:wl.L * wl.n].reshape(wl.L, wl.n)
        for t in range(wl.L):
            assert offs[t, 0] == 0 and offs[t, nb] == wl.n and np.all(np.diff(offs[t]) >= 0)
            for c in np.unique(codes[:, t]):
                got = np.sort(ids[t, offs[t, c]:offs[t, c + 1]])
                np.testing.assert_array_equal(got, np.nonzero(codes[:, t] == c)[0])


def test_bucketed_equals_dense_at_c2_shape():
    """C2 shape (8 units x 4 heads, n = 16384): the bucketed and the dense decode give the same S and
    bit-identical outputs (same gather, same merge order)."""
    pkg = _pkg()
    wl = synth.CONFIGS["C2"]
    k, v, q = synth.make_batch(wl)
    W = synth.make_projections(wl.K, wl.L, wl.mips)
    tW = torch.from_numpy(W).to(_dev())
    tk, tv, tq = _bf(k), _bf(v), _bf(q)
    res = []
    for bk in (False, True):
        mp = pkg.MagicPIG(tW, K=wl.K, L=wl.L, buckets=bk).build(tk)
        sm = torch.zeros((wl.B, wl.Hq, wl.n // 32), dtype=torch.int32, device=_dev())
        out = mp.decode(tq, tk, tv, s_mask=sm)
        torch.cuda.synchronize()
        res.append((out.cpu(), sm.cpu()))
    assert torch.equal(res[0][1], res[1][1])
    assert torch.equal(res[0][0], res[1][0])


def test_bucket_limits():
    pkg = _pkg()
    cfg = pkg.make_config(K=16, L=9)
    assert pkg.binding.bucket_tables_words(cfg, 1, 1, 1000) == 0
    W = torch.zeros((129, 16 * 9), dtype=torch.float32, device=_dev())
    mp = pkg.MagicPIG(W, K=16, L=9, buckets=True)
    with pytest.raises(pkg.MagicPIGError):
        mp.build(torch.zeros((1, 1, 1000, 128), dtype=torch.bfloat16, device=_dev()))


def test_bucketed_sequence_sharding_emulated():
    """Sequence shards on one GPU with bucketed tables per shard: the union of the shards' S equals the
    unsharded S, and the fixed-order merge of the shard partials equals the unsharded estimate (P12)."""
    pkg = _pkg()
    Bd = pkg.binding
    wl = synth.Workload("bshard", 1850, B=1, Hq=4, Hkv=2, n=5000, K=10, L=150)
    k, v, q = synth.make_batch(wl)
    W = synth.make_projections(wl.K, wl.L, 1)
    tW = torch.from_numpy(W).to(_dev())
    tk_full, tv_full, tq = _bf(k), _bf(v), _bf(q)
    full = pkg.MagicPIG(tW, K=wl.K, L=wl.L, buckets=True).build(tk_full)
    sm_full = torch.zeros((1, 4, (wl.n + 31) // 32), dtype=torch.int32, device=_dev())
    out_full = full.decode(tq, tk_full, tv_full, s_mask=sm_full)
    cfg = full.cfg
    dev = _dev()
    cuts = [0, 1024 + 300, 2900, 5000]
    P = len(cuts) - 1
    ks_all = torch.zeros((P, 1, 2, 128, 2), dtype=torch.int64, device=dev)
    cnt_all = torch.zeros((P, 1, 2), dtype=torch.int64, device=dev)
    shards = []
    for p in range(P):
        a, b = cuts[p], cuts[p + 1]
        tk = _bf(k[:, :, a:b])
        ws = Bd.new_workspace(Bd.build_workspace_bytes(cfg, 1, 2, b - a), dev)
        Bd.key_stats(cfg, tk, a, wl.n, ks_all[p], cnt_all[p], ws)
        shards.append((a, b, tk, _bf(v[:, :, a:b]), ws))
    key_sum = torch.zeros((1, 2, 128, 2), dtype=torch.int64, device=dev)
    count = torch.zeros((1, 2), dtype=torch.int64, device=dev)
    Bd.reduce_stats(0, ks_all, cnt_all, P, 1, 2, key_sum, count)
    center = torch.zeros((1, 2, 128), dtype=torch.float32, device=dev)
    r2_all = torch.zeros((P, 1, 2, 2), dtype=torch.int64, device=dev)
    for p, (a, b, tk, tv, ws) in enumerate(shards):
        Bd.key_norms(cfg, tk, a, wl.n, key_sum, count, center, r2_all[p], ws)
    r2 = torch.zeros((1, 2, 2), dtype=torch.int64, device=dev)
    Bd.reduce_stats(1, r2_all, None, P, 1, 2, r2, None)
    parts = torch.zeros((P, 4, 130), dtype=torch.float32, device=dev)
    masks = []
    for p, (a, b, tk, tv, ws) in enumerate(shards):
        codes = torch.zeros((Bd.codes_words(cfg, 1, 2, b - a),), dtype=torch.int32, device=dev)
        knorm = torch.zeros((1, 2, b - a), dtype=torch.float32, device=dev)
        Bd.build_tables(cfg, tk, a, wl.n, tW, center, r2, codes, knorm, ws)
        tables = torch.zeros((Bd.bucket_tables_words(cfg, 1, 2, b - a),), dtype=torch.int32, device=dev)
        Bd.build_buckets(cfg, codes, 1, 2, b - a, tables)
        wsd = Bd.new_workspace(Bd.decode_workspace_bytes(cfg, 1, 4, 2, b - a), dev)
        sm = torch.zeros((1, 4, (b - a + 31) // 32), dtype=torch.int32, device=dev)
        Bd.decode_buckets(cfg, tq, tables, center, knorm, tk, tv, a, wl.n, tW, wsd, partial=parts[p], s_mask=sm)
        masks.append((a, b, sm))
    out = torch.zeros((1, 4, 128), dtype=torch.float32, device=dev)
    Bd.merge_partials(parts, out)
    torch.cuda.synchronize()
    full_mask = sm_full.cpu().numpy().view(np.uint32)
    for a, b, sm in masks:
        mk = sm.cpu().numpy().view(np.uint32)
        for row in range(4):
            got = np.unpackbits(mk[0, row].view(np.uint8), bitorder="little")[: b - a]
            want = np.unpackbits(full_mask[0, row].view(np.uint8), bitorder="little")[a:b]
            np.testing.assert_array_equal(got, want)
    for row in range(4):
        assert _rel_err(out.cpu().numpy()[0, row], out_full.cpu().numpy()[0, row]) <= 2e-4


def test_bucketed_session_matches_decode():
    pkg = _pkg()
    wl = synth.Workload("bsess", 1860, B=1, Hq=8, Hkv=2, n=3000, K=10, L=150)
    k, v, q = synth.make_batch(wl)
    W = synth.make_projections(wl.K, wl.L, wl.mips)
    mp, tk = _build(wl, k, W)
    tv, tq = _bf(v), _bf(q)
    ref = mp.decode(tq, tk, tv).cpu()
    sess = pkg.session(mp, tk, tv, wl.Hq)
    sess.q_host.copy_(tq.cpu())
    got = sess.step()
    torch.cuda.synchronize()
    assert torch.equal(got, ref)
