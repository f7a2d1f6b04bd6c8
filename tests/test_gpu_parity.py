"""GPU parity tests (-m gpu): the CUDA path through the C ABI vs the CPU oracle
on the same seeded inputs.  Bit-exact: centering vector, MIPS radius, key
codes, query codes, collision counts, sampled sets S.  Outputs: per (sequence,
query head) max_d |o_gpu - o_ref| / max_d |o_ref| <= 2e-3 (north_star; DESIGN.md
reading R18)."""
from __future__ import annotations

import json
import os

import numpy as np
import pytest

import oracle
import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

TOL = 2e-3


@pytest.fixture(params=[9, 8, 7, 6, 5], ids=["k9", "k8", "k7", "k6", "k5"], autouse=True)
def decode_kernel(request):
    """Every parity test runs on five decode paths: 9 = kernel 7's pipeline with the K/V rows gathered
    by plain 16-B loads straight into the mma fragments (no shared-memory staging), 8 = Query kernel + select (per-piece S_g u T
    lists) + the tcgen05 estimator (TMA gather4 tiles, TMEM accumulators), 7 = the same with the
    mma.sync estimator (every warp a contiguous range), 6 = Query kernel + estimator kernel with a
    producer warp, and 5 = the persistent fused kernel (which falls back to the cluster-per-chunk
    kernel 4 when its shared memory does not fit); they must agree with the oracle independently."""
    if not torch.cuda.is_available():
        pytest.fail("GPU tests need a CUDA device (no fallback)")
    pkg = _pkg()
    pkg.binding.set_decode_kernel(request.param)
    yield request.param
    pkg.binding.set_decode_kernel(0)


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


def _run_gpu(wl, k, v, q, W, s_mask=True):
    pkg = _pkg()
    B, Hkv, n, _ = k.shape
    Hq = q.shape[1]
    tk, tv, tq = _bf(k), _bf(v), _bf(q)
    tW = torch.from_numpy(W).to(_dev())
    mp = pkg.MagicPIG(tW, K=wl.K, L=wl.L, center=wl.center, mips=wl.mips, min_collisions=wl.min_collisions,
                      sink=wl.sink, local=wl.local).build(tk)
    s_count = torch.zeros((B, Hq), dtype=torch.int32, device=_dev())
    nw = (n + 31) // 32
    sm = torch.zeros((B, Hq, max(nw, 1)), dtype=torch.int32, device=_dev()) if s_mask else None
    part = torch.zeros((B * Hq, 130), dtype=torch.float32, device=_dev())
    out = mp.decode(tq, tk, tv, s_count=s_count, s_mask=sm)
    mp.decode(tq, tk, tv, partial=part)
    canon = torch.zeros((B, Hkv, max(n, 1), wl.L), dtype=torch.int16, device=_dev())
    pkg.binding.export_codes(mp.cfg, mp.buf.codes, B, Hkv, n, canon)
    torch.cuda.synchronize()
    st_b, st_d = mp.status("build"), mp.status("decode")
    res = {
        "out": out.cpu().numpy(), "s_count": s_count.cpu().numpy(),
        "s_mask": sm.cpu().numpy().view(np.uint32) if s_mask else None,
        "codes": canon.cpu().numpy().view(np.uint16)[:, :, :n], "center": mp.buf.center.cpu().numpy(),
        "r2": mp.buf.r2.cpu().numpy(), "partial": part.cpu().numpy(), "status_build": st_b,
        "status_decode": st_d, "mp": mp, "tq": tq, "tk": tk, "tv": tv, "tW": tW,
    }
    return res


def _q64(pair):
    v = (int(pair[0]) & ((1 << 64) - 1)) | ((int(pair[1]) & ((1 << 64) - 1)) << 64)
    return v - (1 << 128) if v >= (1 << 127) else v


def _check_unit(wl, res, ref, b, h, n, check_codes=True):
    G = wl.G
    assert ref["status"] in (0, oracle.OR_EDEGENERATE), ref["status"]
    if check_codes:
        np.testing.assert_array_equal(res["codes"][b, h], ref["codes"], err_msg="key codes differ")
    np.testing.assert_array_equal(res["center"][b, h], ref["c"], err_msg="centering vector differs")
    for g in range(G):
        row = h * G + g
        assert int(res["s_count"][b, row]) == int(ref["s_count"][g]), (b, row)
        if res["s_mask"] is not None:
            bits = np.unpackbits(res["s_mask"][b, row].view(np.uint8), bitorder="little")[:n]
            np.testing.assert_array_equal(bits, (ref["in_s"][g] == 1).astype(np.uint8), err_msg=f"S differs {b},{row}")
        if ref["s_count"][g] > 0 or np.any(ref["in_s"][g] == 2):
            err = _rel_err(res["out"][b, row], ref["out"][g])
            assert err <= TOL, (b, row, err)


CASES = [
    # name, n, B, Hq, Hkv, K, L, center, mips, minc, sink, local
    ("C1", 1024, 1, 1, 1, 10, 150, 1, 1, 2, 4, 64),
    ("ragged", 2500, 1, 4, 1, 10, 150, 1, 1, 2, 4, 64),
    ("mips0", 3000, 1, 4, 2, 10, 150, 1, 0, 2, 4, 64),
    ("k8l75", 2049, 2, 8, 2, 8, 75, 1, 1, 2, 4, 64),
    ("k11l300", 1500, 1, 2, 1, 11, 300, 1, 1, 2, 4, 64),
    ("k7", 1800, 1, 8, 1, 7, 35, 1, 1, 2, 4, 64),
    ("k3l5", 700, 1, 2, 2, 3, 5, 1, 1, 2, 0, 0),
    ("minc1", 1300, 1, 4, 1, 9, 20, 1, 1, 1, 4, 24),
    ("nocenter", 1111, 1, 1, 1, 10, 150, 0, 1, 2, 4, 64),
    ("k16", 1100, 1, 2, 1, 16, 9, 1, 1, 2, 2, 8),
    ("allstatic", 60, 1, 4, 1, 10, 150, 1, 1, 2, 4, 64),
    ("tiny", 37, 1, 1, 1, 2, 3, 1, 1, 2, 1, 1),
    # persistent kernel: CTAs spanning several units, and units spanning > 1 merge block
    ("manyunits", 3000, 16, 32, 8, 8, 20, 1, 1, 2, 4, 64),
    ("longunit", 40000, 1, 4, 1, 8, 20, 1, 1, 2, 4, 64),
    ("longg8", 20000, 1, 8, 1, 6, 16, 1, 1, 2, 4, 64),
]


@pytest.mark.parametrize("case", CASES, ids=[c[0] for c in CASES])
def test_build_and_decode_parity(case):
    name, n, B, Hq, Hkv, K, L, center, mips, minc, sink, local = case
    wl = synth.Workload(name, 700 + CASES.index(case), B=B, Hq=Hq, Hkv=Hkv, n=n, K=K, L=L, center=center,
                        mips=mips, min_collisions=minc, sink=sink, local=local)
    k, v, q = synth.make_batch(wl)
    W = synth.make_projections(K, L, mips)
    res = _run_gpu(wl, k, v, q, W)
    assert res["status_build"] == 0 and res["status_decode"] in (0,), (res["status_build"], res["status_decode"])
    refs = oracle.decode_batch(k, v, q, W, K, L, center, mips, minc, sink, local)
    for b in range(B):
        for h in range(Hkv):
            ref = refs[b][h]
            _check_unit(wl, res, ref, b, h, n)
            t = oracle.key_transform(k[b, h], sink, local, center, mips)
            assert _q64(res["r2"][b, h]) == t["r2_q"]


def test_query_codes_and_collision_counts():
    pkg = _pkg()
    wl = synth.Workload("qc", 801, B=2, Hq=8, Hkv=2, n=1500, K=10, L=150)
    k, v, q = synth.make_batch(wl)
    W = synth.make_projections(wl.K, wl.L, wl.mips)
    res = _run_gpu(wl, k, v, q, W, s_mask=False)
    mp = res["mp"]
    qc = torch.zeros((2, 8, wl.L), dtype=torch.int16, device=_dev())
    ws = pkg.binding.new_workspace(pkg.binding.decode_workspace_bytes(mp.cfg, 2, 8, 2, wl.n), _dev())
    pkg.binding.query_codes(mp.cfg, res["tq"], res["tW"], qc, ws)
    cnt = torch.zeros((2, 8, wl.n), dtype=torch.int16, device=_dev())
    pkg.binding.collision_counts(mp.cfg, res["tq"], mp.buf.codes, (2, 2, wl.n), res["tW"], cnt, ws)
    torch.cuda.synchronize()
    qc = qc.cpu().numpy().view(np.uint16)
    cnt = cnt.cpu().numpy().view(np.uint16)
    for b in range(2):
        for hq in range(8):
            ref = oracle.encode_query(q[b, hq], W, wl.K, wl.L, wl.mips)
            np.testing.assert_array_equal(qc[b, hq], ref)
            h = hq // 4
            t = oracle.key_transform(k[b, h], wl.sink, wl.local, 1, 1)
            if hq % 4 == 0:
                codes = oracle.encode_keys(t["xbar"], W, wl.K, wl.L)
            np.testing.assert_array_equal(cnt[b, hq], oracle.collision_counts(codes, ref))


def test_decode_on_imported_oracle_codes():
    """The decode kernel alone: codes computed by the oracle, packed on device."""
    pkg = _pkg()
    wl = synth.Workload("imp", 802, B=1, Hq=4, Hkv=1, n=3100, K=10, L=150)
    k, v, q = synth.make_batch(wl)
    W = synth.make_projections(wl.K, wl.L, wl.mips)
    ref = oracle.decode_unit(k[0, 0], v[0, 0], q[0], W, wl.K, wl.L)
    res = _run_gpu(wl, k, v, q, W)
    mp = res["mp"]
    canon = _bf(ref["codes"][None, None].view(np.uint16))  # raw 16-bit payload
    mp.buf.codes.zero_()
    pkg.binding.import_codes(mp.cfg, canon.view(torch.int16), 1, 1, wl.n, mp.buf.codes)
    s_count = torch.zeros((1, 4), dtype=torch.int32, device=_dev())
    out = mp.decode(res["tq"], res["tk"], res["tv"], s_count=s_count)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(s_count.cpu().numpy()[0], ref["s_count"])
    for g in range(4):
        assert _rel_err(out.cpu().numpy()[0, g], ref["out"][g]) <= TOL


def test_g1_golden_padded_to_d128():
    """Worked example G1 (tests/golden) embedded in d = 128 by zero padding."""
    pkg = _pkg()
    with open(os.path.join(os.path.dirname(__file__), "golden", "g1_worked_example.json")) as f:
        g = json.load(f)
    d = 128
    k = np.zeros((1, 1, 4, d), np.float32)
    v = np.zeros((1, 1, 4, d), np.float32)
    k[0, 0, :, :2] = g["keys"]
    v[0, 0, :, :2] = g["values"]
    q = np.zeros((1, 1, d), np.float32)
    q[0, 0, :2] = g["q"]
    W = np.zeros((d, 3), np.float32)
    W[:2, :] = np.array(g["W_columns"], np.float32).T
    bf = synth.bf16_bits_from_f32
    mp = pkg.MagicPIG(torch.from_numpy(W).to(_dev()), K=1, L=3, center=1, mips=0, min_collisions=2, sink=0,
                      local=0).build(_bf(bf(k)))
    s_count = torch.zeros((1, 1), dtype=torch.int32, device=_dev())
    out = mp.decode(_bf(bf(q)), _bf(bf(k)), _bf(bf(v)), s_count=s_count)
    torch.cuda.synchronize()
    assert int(s_count[0, 0]) == len(g["mips0"]["S"])
    np.testing.assert_allclose(out.cpu().numpy()[0, 0, :2], g["mips0"]["out_padded_d128"], rtol=TOL, atol=1e-6)


def test_tensor_core_accumulation_error_bound():
    """The fix-up filter threshold eps = 2^-19 must dominate the tcgen05 fp32
    accumulation error: measure max |acc - exact| / (|xbar| |W_j|)."""
    pkg = _pkg()
    wl = synth.Workload("acc", 803, B=1, Hq=1, Hkv=1, n=128, K=10, L=150)
    k, v, q = synth.make_batch(wl)
    W = synth.make_projections(wl.K, wl.L, 1)
    res = _run_gpu(wl, k, v, q, W, s_mask=False)
    mp = res["mp"]
    cfg = mp.cfg
    nb = pkg.binding.build_workspace_bytes(cfg, 1, 1, 128) + 4 * pkg.binding.codes_words(cfg, 1, 1, 128) + 1024
    ws = pkg.binding.new_workspace(nb, _dev())
    acc = torch.zeros((128, wl.K * wl.L), dtype=torch.float32, device=_dev())
    pkg.binding.debug_hash_acc(cfg, res["tk"][0, 0].contiguous(), res["tW"], mp.buf.center, mp.buf.r2, acc, ws)
    torch.cuda.synchronize()
    t = oracle.key_transform(k[0, 0], wl.sink, wl.local, 1, 1)
    xb = synth.bf16_bits_to_f32(t["xbar"]).astype(np.float64)
    exact = xb @ W.astype(np.float64)  # products exact; fp64 sum error ~1e-16 relative
    scale = np.linalg.norm(xb, axis=1)[:, None] * np.linalg.norm(W.astype(np.float64), axis=0)[None, :]
    rel = np.abs(acc.cpu().numpy().astype(np.float64) - exact) / np.maximum(scale, 1e-30)
    worst = float(rel.max())
    print(f"tcgen05 bf16 accumulation: max |acc-exact|/(|x||w|) = {worst:.3e} (2^{np.log2(max(worst, 1e-300)):.1f})")
    assert worst < 2.0 ** -22, worst  # eps / 8


def test_sequence_sharding_emulated(decode_kernel):
    """Shard emulator on one GPU: P contiguous key shards, exact statistic
    reductions, per-shard partial decode, fixed-order merge == unsharded (P12)."""
    pkg = _pkg()
    Bd = pkg.binding
    wl = synth.Workload("shard", 804, B=1, Hq=4, Hkv=2, n=5000, K=10, L=150)
    k, v, q = synth.make_batch(wl)
    W = synth.make_projections(wl.K, wl.L, 1)
    full = _run_gpu(wl, k, v, q, W)
    cfg = full["mp"].cfg
    tW = full["tW"]
    cuts = [0, 1024 + 300, 2900, 5000]
    P = len(cuts) - 1
    dev = _dev()
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
        wsd = Bd.new_workspace(Bd.decode_workspace_bytes(cfg, 1, 4, 2, b - a), dev)
        sm = torch.zeros((1, 4, (b - a + 31) // 32), dtype=torch.int32, device=dev)
        Bd.decode(cfg, full["tq"], codes, center, knorm, tk, tv, a, wl.n, tW, wsd, partial=parts[p], s_mask=sm)
        masks.append((a, b, sm))
    out = torch.zeros((1, 4, 128), dtype=torch.float32, device=dev)
    Bd.merge_partials(parts, out)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(center.cpu().numpy(), full["center"])
    np.testing.assert_array_equal(r2.cpu().numpy(), full["r2"])
    for a, b, sm in masks:
        mk = sm.cpu().numpy().view(np.uint32)
        for row in range(4):
            got = np.unpackbits(mk[0, row].view(np.uint8), bitorder="little")[: b - a]
            want = np.unpackbits(full["s_mask"][0, row].view(np.uint8), bitorder="little")[a:b]
            np.testing.assert_array_equal(got, want)
    # the merged shard estimates against the oracle (Alg. 1 on the unsharded unit + the LSE merge; R18)
    for h in range(2):
        ref = oracle.decode_unit(k[0, h], v[0, h], q[0, 2 * h:2 * h + 2], W, wl.K, wl.L, 1, 1, 2, 4, 64)
        for g in range(2):
            assert _rel_err(out.cpu().numpy()[0, 2 * h + g], ref["out"][g]) <= TOL
    # and against the unsharded GPU run: same S and u; kernels 6-8 weight in fp32 (hi + lo bf16 parts), kernel 5
    # rounds the weights to tf32 (relative 2^-11) against a different running maximum per shard
    tol = 2e-4 if decode_kernel == 5 else 2e-5
    for row in range(4):
        assert _rel_err(out.cpu().numpy()[0, row], full["out"][0, row]) <= tol


_C2_CACHE = {}


def _c2_reference():
    """Inputs and oracle results of all 8 units of C2 (computed once, units on parallel host threads)."""
    if not _C2_CACHE:
        from concurrent.futures import ThreadPoolExecutor
        wl = synth.CONFIGS["C2"]
        k, v, q = synth.make_batch(wl, threads=8)
        W = synth.make_projections(wl.K, wl.L, wl.mips)
        with ThreadPoolExecutor(8) as ex:
            refs = list(ex.map(lambda h: oracle.decode_unit(k[0, h], v[0, h], q[0, h * wl.G:(h + 1) * wl.G], W, wl.K,
                                                            wl.L, wl.center, wl.mips, wl.min_collisions, wl.sink,
                                                            wl.local), range(wl.Hkv)))
        _C2_CACHE.update(wl=wl, k=k, v=v, q=q, W=W, refs=refs)
    return _C2_CACHE


def test_c2_full_size_all_units():
    """BASELINE config C2 (Llama-3.1-8B layer, 16K, B=1, (10,150)) at full size in
    the bench's launch configuration; all 8 (sequence, kv head) units checked
    against the oracle end to end (codes, S, |S_g|, outputs)."""
    c = _c2_reference()
    wl = c["wl"]
    res = _run_gpu(wl, c["k"], c["v"], c["q"], c["W"])
    assert res["status_build"] == 0 and res["status_decode"] == 0
    for h in range(wl.Hkv):
        _check_unit(wl, res, c["refs"][h], 0, h, wl.n)


def test_query_codes_near_zero_dots():
    """Query-code signs where the fp32 certificate fails: exact zeros (sign(0)=0,
    R6) and dots cancelling to ~2^-20 of their terms go through the fp64 and
    exact-integer fallbacks; every bit must equal the oracle's."""
    pkg = _pkg()
    rng = np.random.default_rng(77)
    K, L = 4, 40
    KL = K * L
    bf = synth.bf16_bits_from_f32
    q = synth.bf16_bits_to_f32(bf(rng.standard_normal((1, 3, 128), dtype=np.float32)))
    W = synth.bf16_bits_to_f32(bf(rng.standard_normal((128, KL), dtype=np.float32)))
    q[0, 0, :] = 0.0
    q[0, 0, 0], q[0, 0, 1], q[0, 0, 2] = 1.0, -1.0, 2.0 ** -20
    for j in range(0, KL, 3):  # columns with an exact zero or a tiny dot against head 0
        W[:, j] = 0.0
        W[0, j] = W[1, j] = np.float32(rng.choice([0.5, 1.0, 3.0]))
        W[2, j] = np.float32(rng.choice([0.0, 1.0, -1.0]))
    q[0, 1] = q[0, 0] * -1
    cfg = pkg.binding.make_config(K=K, L=L, mips=0)
    tq = _bf(bf(q))
    tW = torch.from_numpy(np.ascontiguousarray(W)).to(_dev())
    qc = torch.zeros((1, 3, L), dtype=torch.int16, device=_dev())
    ws = pkg.binding.new_workspace(pkg.binding.decode_workspace_bytes(cfg, 1, 3, 1, 0) + 4096, _dev())
    pkg.binding.query_codes(cfg, tq, tW, qc, ws)
    torch.cuda.synchronize()
    got = qc.cpu().numpy().view(np.uint16)
    assert pkg.binding.workspace_status(ws) == 0
    for h in range(3):
        np.testing.assert_array_equal(got[0, h], oracle.encode_query(bf(q[0, h]), W, K, L, 0))


def test_decode_session_graph_matches_decode():
    """The serving API (one CUDA graph: H2D q, encode, decode, D2H out) returns the same bits as the
    eager decode, for two different queries replayed through the same graph."""
    pkg = _pkg()
    wl = synth.Workload("session", 950, B=1, Hq=8, Hkv=2, n=3000, K=10, L=150)
    k, v, q = synth.make_batch(wl)
    W = synth.make_projections(wl.K, wl.L, wl.mips)
    tk, tv = _bf(k), _bf(v)
    mp = pkg.MagicPIG(torch.from_numpy(W).to(_dev()), K=wl.K, L=wl.L).build(tk)
    sess = pkg.session(mp, tk, tv, wl.Hq)
    for qq in (q, q[:, ::-1].copy()):
        tq = _bf(qq)
        ref = mp.decode(tq, tk, tv).cpu()
        sess.q_host.copy_(tq.cpu())
        got = sess.step()
        torch.cuda.synchronize()
        assert torch.equal(got, ref)


@pytest.mark.parametrize("G,buckets", [(4, False), (4, True), (8, False), (1, True)])
def test_weighted_set_is_s_union_t(G, buckets, decode_kernel):
    """The compacted list the estimator gathers, exported as the (head, key) pairs that received a
    finite weight: it must equal S_g u T exactly (oracle), and S_g restricted to D must equal the
    oracle's S_g (Alg. 1)."""
    if decode_kernel < 6:
        pytest.skip("weighted-set export exists on the v6 / v7 paths")
    pkg = _pkg()
    n = 5000
    wl = synth.Workload("wset", 960 + G + 10 * buckets, B=2, Hq=2 * G, Hkv=2, n=n, K=8, L=40, sink=4, local=64)
    k, v, q = synth.make_batch(wl)
    W = synth.make_projections(wl.K, wl.L, wl.mips)
    tk, tv, tq = _bf(k), _bf(v), _bf(q)
    tW = torch.from_numpy(W).to(_dev())
    mp = pkg.MagicPIG(tW, K=wl.K, L=wl.L, buckets=buckets).build(tk)
    nw = (n + 31) // 32
    sm = torch.zeros((2, wl.Hq, nw), dtype=torch.int32, device=_dev())
    wt = torch.zeros((2, wl.Hq, nw), dtype=torch.int32, device=_dev())
    out = torch.zeros((2, wl.Hq, 128), dtype=torch.float32, device=_dev())
    ws = mp.decode_workspace(2, wl.Hq, 2, n, _dev())
    pkg.binding.debug_decode_sets(mp.cfg, tq, None if buckets else mp.buf.codes, mp.buf.tables if buckets else None,
                                  mp.buf.center, mp.buf.key_norm, tk, tv, 0, n, tW, ws, out, sm, wt)
    torch.cuda.synchronize()
    smn = sm.cpu().numpy().view(np.uint32)
    wtn = wt.cpu().numpy().view(np.uint32)
    refs = oracle.decode_batch(k, v, q, W, wl.K, wl.L, 1, 1, 2, 4, 64)
    for b in range(2):
        for h in range(2):
            ref = refs[b][h]
            for g in range(G):
                row = h * G + g
                s_bits = np.unpackbits(smn[b, row].view(np.uint8), bitorder="little")[:n]
                w_bits = np.unpackbits(wtn[b, row].view(np.uint8), bitorder="little")[:n]
                np.testing.assert_array_equal(s_bits, (ref["in_s"][g] == 1).astype(np.uint8))
                np.testing.assert_array_equal(w_bits, (ref["in_s"][g] >= 1).astype(np.uint8))
                assert _rel_err(out.cpu().numpy()[b, row], ref["out"][g]) <= TOL


@pytest.mark.gpu
def test_value_cancellation():
    """Heavy cancellation in P.V (|o| << |v|): keys come in pairs (row 2j+1 = row 2j with dimension 0 moved by
    one bf16 ulp, so the pair's weights differ by ~1e-4 relative and its hash codes almost always agree) whose
    values are +64 and -64 (plus small noise).  The R18 tolerance relative to max|o| then needs the weights at
    about fp32 accuracy inside the P.V products (kernel 5: tf32 hi + lo parts; kernels 7-9: bf16 hi + lo);
    weights rounded once to tf32 would lose the pairs' difference."""
    wl = synth.Workload("cancel", 777, B=1, Hq=4, Hkv=1, n=3000, K=10, L=150)
    k, v, q = synth.make_batch(wl)
    k = k.copy()
    k[:, :, 1::2] = k[:, :, 0::2]
    k[:, :, 1::2, 0] = np.where(k[:, :, 1::2, 0] == 0xFFFF, 0xFFFE, k[:, :, 1::2, 0] + 1).astype(np.uint16)
    rng = np.random.default_rng(4242)
    sgn = np.where(np.arange(wl.n) % 2 == 0, 1.0, -1.0).reshape(1, 1, wl.n, 1)
    vf = 64.0 * sgn + 0.25 * rng.standard_normal((1, 1, wl.n, 128))
    v = synth.bf16_bits_from_f32(vf)
    W = synth.make_projections(wl.K, wl.L, wl.mips)
    res = _run_gpu(wl, k, v, q, W)
    assert res["status_build"] == 0 and res["status_decode"] == 0
    ref = oracle.decode_batch(k, v, q, W, wl.K, wl.L, wl.center, wl.mips, wl.min_collisions, wl.sink, wl.local)[0][0]
    vmax = float(np.max(np.abs(synth.bf16_bits_to_f32(v))))
    for g in range(wl.G):
        assert np.max(np.abs(ref["out"][g])) < vmax / 16, "the case must cancel"
        err = _rel_err(res["out"][0, g], ref["out"][g])
        assert err <= TOL, (g, err)
