"""GPU parity at BASELINE sizes and adversarial hashing inputs (-m gpu).

* C3 (B=8, 64K, (10,150)), C4 (70B shape: 64 q / 8 kv heads, 96K) and C5 (128K, sequence-sharded over 4
  emulated shards with the exact statistic reductions and the fixed-order LSE merge): >= 8 randomly
  chosen (sequence, kv head) units each, compared with the oracle (codes / S / |S_g| bit-exact, outputs
  within 2e-3, R18) in the bench's launch configuration (default kernel choice; C3 also on kernel 8).
* Key-side sign exactness (C-2 contract, P:83-84 SimHash sign with sign(0)=0): keys whose dot with some
  projection cancels to 0 or to a value far below the fp32 resolution of its terms; the tensor-core
  accumulator gets some of these signs wrong, the filter + exact fix-up must correct every one of them.
The oracle units run on parallel host threads (ctypes releases the GIL)."""
from __future__ import annotations

from concurrent.futures import ThreadPoolExecutor

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


def _oracle_units(wl, k, v, q, W, units):
    def one(bh):
        b, h = bh
        return oracle.decode_unit(k[b, h], v[b, h], q[b, h * wl.G:(h + 1) * wl.G], W, wl.K, wl.L, wl.center,
                                  wl.mips, wl.min_collisions, wl.sink, wl.local)
    with ThreadPoolExecutor(8) as ex:
        return list(ex.map(one, units))


def _pick_units(wl, count, seed):
    rng = np.random.default_rng(seed)
    all_units = [(b, h) for b in range(wl.B) for h in range(wl.Hkv)]
    idx = rng.choice(len(all_units), size=min(count, len(all_units)), replace=False)
    return [all_units[i] for i in sorted(idx)]


def _check(wl, out, s_count, s_mask, refs, units, n):
    for (b, h), ref in zip(units, refs):
        assert ref["status"] in (0, oracle.OR_EDEGENERATE)
        for g in range(wl.G):
            row = h * wl.G + g
            assert int(s_count[b, row]) == int(ref["s_count"][g]), (b, row)
            if s_mask is not None:
                bits = np.unpackbits(s_mask[b, row].view(np.uint8), bitorder="little")[:n]
                np.testing.assert_array_equal(bits, (ref["in_s"][g] == 1).astype(np.uint8), err_msg=f"S {b},{row}")
            assert _rel_err(out[b, row], ref["out"][g]) <= TOL, (b, row)


@pytest.mark.parametrize("name,kernel,buckets", [("C3", 0, True), ("C3", 0, False), ("C3", 8, True), ("C3", 9, True), ("C4", 9, False), ("C4", 0, False)])
def test_baseline_config_sampled_units(name, kernel, buckets):
    pkg = _pkg()
    wl = synth.CONFIGS[name]
    k, v, q = synth.make_batch(wl, threads=8)
    W = synth.make_projections(wl.K, wl.L, wl.mips)
    units = _pick_units(wl, 8, 3 + (name == "C4"))
    refs = _oracle_units(wl, k, v, q, W, units)
    tk, tv, tq = _bf(k), _bf(v), _bf(q)
    del k, v
    tW = torch.from_numpy(W).to(_dev())
    pkg.binding.set_decode_kernel(kernel)
    try:
        mp = pkg.MagicPIG(tW, K=wl.K, L=wl.L, buckets=buckets).build(tk)
        s_count = torch.zeros((wl.B, wl.Hq), dtype=torch.int32, device=_dev())
        nw = (wl.n + 31) // 32
        s_mask = torch.zeros((wl.B, wl.Hq, nw), dtype=torch.int32, device=_dev())
        out = mp.decode(tq, tk, tv, s_count=s_count, s_mask=s_mask)
        torch.cuda.synchronize()
        assert mp.status() == 0 and mp.status("build") == 0
        canon = torch.zeros((1, 1, wl.n, wl.L), dtype=torch.int16, device=_dev())
        b0, h0 = units[0]
        u0 = b0 * wl.Hkv + h0
        words = pkg.binding.codes_words(mp.cfg, 1, 1, wl.n)
        pkg.binding.export_codes(mp.cfg, mp.buf.codes[u0 * words:(u0 + 1) * words], 1, 1, wl.n, canon)
        np.testing.assert_array_equal(canon.cpu().numpy().view(np.uint16)[0, 0], refs[0]["codes"])
        _check(wl, out.cpu().numpy(), s_count.cpu().numpy(), s_mask.cpu().numpy().view(np.uint32), refs, units, wl.n)
    finally:
        pkg.binding.set_decode_kernel(0)


def test_c5_sequence_sharded_units():
    """C5: 128K keys per (sequence, kv head), split over 4 emulated sequence shards (each a separate index
    with the global centering vector and MIPS radius from the exact reductions), partial states merged in
    shard order; 8 units (all kv heads of the sequence) against the unsharded oracle."""
    pkg = _pkg()
    Bd = pkg.binding
    from paper_2410_16179_b200.sharding import sequence_shard
    wl = synth.CONFIGS["C5"]
    k, v, q = synth.make_batch(wl, threads=8)
    W = synth.make_projections(wl.K, wl.L, wl.mips)
    units = [(0, h) for h in range(wl.Hkv)]
    refs = _oracle_units(wl, k, v, q, W, units)
    dev = _dev()
    tW = torch.from_numpy(W).to(dev)
    tq = _bf(q)
    P = 4
    cfg = Bd.make_config(wl.K, wl.L, wl.center, wl.mips, wl.min_collisions, wl.sink, wl.local)
    shards = []
    ks_all = torch.zeros((P, 1, wl.Hkv, 128, 2), dtype=torch.int64, device=dev)
    cnt_all = torch.zeros((P, 1, wl.Hkv), dtype=torch.int64, device=dev)
    for p in range(P):
        lo, ln = sequence_shard(wl.n, P, p)
        tk, tv = _bf(k[:, :, lo:lo + ln]), _bf(v[:, :, lo:lo + ln])
        ws = Bd.new_workspace(Bd.build_workspace_bytes(cfg, 1, wl.Hkv, ln), dev)
        Bd.key_stats(cfg, tk, lo, wl.n, ks_all[p], cnt_all[p], ws)
        shards.append((lo, ln, tk, tv, ws))
    key_sum = torch.zeros((1, wl.Hkv, 128, 2), dtype=torch.int64, device=dev)
    count = torch.zeros((1, wl.Hkv), dtype=torch.int64, device=dev)
    Bd.reduce_stats(0, ks_all, cnt_all, P, 1, wl.Hkv, key_sum, count)
    center = torch.zeros((1, wl.Hkv, 128), dtype=torch.float32, device=dev)
    r2_all = torch.zeros((P, 1, wl.Hkv, 2), dtype=torch.int64, device=dev)
    for p, (lo, ln, tk, tv, ws) in enumerate(shards):
        Bd.key_norms(cfg, tk, lo, wl.n, key_sum, count, center, r2_all[p], ws)
    r2 = torch.zeros((1, wl.Hkv, 2), dtype=torch.int64, device=dev)
    Bd.reduce_stats(1, r2_all, None, P, 1, wl.Hkv, r2, None)
    parts = torch.zeros((P, wl.Hq, Bd.PART), dtype=torch.float32, device=dev)
    counts = []
    for p, (lo, ln, tk, tv, ws) in enumerate(shards):
        codes = torch.zeros((Bd.codes_words(cfg, 1, wl.Hkv, ln),), dtype=torch.int32, device=dev)
        knorm = torch.zeros((1, wl.Hkv, ln), dtype=torch.float32, device=dev)
        Bd.build_tables(cfg, tk, lo, wl.n, tW, center, r2, codes, knorm, ws)
        wsd = Bd.new_workspace(Bd.decode_workspace_bytes(cfg, 1, wl.Hq, wl.Hkv, ln), dev)
        sc = torch.zeros((1, wl.Hq), dtype=torch.int32, device=dev)
        Bd.decode(cfg, tq, codes, center, knorm, tk, tv, lo, wl.n, tW, wsd, partial=parts[p], s_count=sc)
        counts.append(sc)
    out = torch.zeros((1, wl.Hq, 128), dtype=torch.float32, device=dev)
    Bd.merge_partials(parts, out)
    torch.cuda.synchronize()
    s_count = sum(c.cpu().numpy() for c in counts)
    for h, ref in enumerate(refs):
        np.testing.assert_array_equal(center.cpu().numpy()[0, h], ref["c"])
    _check(wl, out.cpu().numpy(), s_count, None, refs, units, wl.n)


def test_key_side_cancellation_fixup():
    """Keys x with x . W_j = delta exactly, where delta is 0 or far below the fp32 resolution of the cancelling
    terms (+-2^10): the tcgen05 accumulator loses delta for some (key, column) pairs (a wrong or zero sign before
    the fix-up); after the filter + exact fix-up every code bit must equal the oracle's sign of the exact dot
    (sign(0) = 0, R6).  center = mips = 0, so x = k (C-2 contract)."""
    pkg = _pkg()
    Bd = pkg.binding
    rng = np.random.default_rng(17)
    n, K, L = 128, 8, 16
    KL = K * L
    Wf = np.zeros((128, KL), np.float32)
    Wf[0, :] = 1.0
    Wf[1, :] = 1.0  # every column: x0 * 1 + x1 * 1 cancels when x1 = -x0
    Wf[2:, :] = rng.choice([-1.0, -0.5, 0.5, 1.0], size=(126, KL)).astype(np.float32)
    kf = np.zeros((n, 128), np.float32)
    kf[:, 0] = 1024.0
    kf[:, 1] = -1024.0
    # tiny tails: x_d in {0, +-2^-20}, so x . W_j = sum of tails = 0 or a few 2^-21 .. 2^-18 (exact)
    kf[:, 2:] = (rng.integers(-1, 2, (n, 126)) * 2.0 ** -20 * (rng.random((n, 126)) < 0.05)).astype(np.float32)
    k = synth.bf16_bits_from_f32(kf)
    W = synth.bf16_bits_to_f32(synth.bf16_bits_from_f32(Wf))
    dev = _dev()
    tk = _bf(k[None, None])
    tW = torch.from_numpy(W).to(dev)
    mp = pkg.MagicPIG(tW, K=K, L=L, center=0, mips=0, sink=0, local=0).build(tk)
    canon = torch.zeros((1, 1, n, L), dtype=torch.int16, device=dev)
    Bd.export_codes(mp.cfg, mp.buf.codes, 1, 1, n, canon)
    nb = Bd.build_workspace_bytes(mp.cfg, 1, 1, n) + 4 * Bd.codes_words(mp.cfg, 1, 1, n) + 1024
    ws = Bd.new_workspace(nb, dev)
    acc = torch.zeros((n, KL), dtype=torch.float32, device=dev)
    Bd.debug_hash_acc(mp.cfg, tk[0, 0].contiguous(), tW, mp.buf.center, mp.buf.r2, acc, ws)
    torch.cuda.synchronize()
    assert mp.status("build") == 0
    ref = oracle.build_unit(k, W, K, L, 0, 0, 0, 0)
    got = canon.cpu().numpy().view(np.uint16)[0, 0]
    np.testing.assert_array_equal(got, ref["codes"])  # every bit = sign of the exact dot after the fix-up
    # raw tensor-core signs vs the final bits: the fix-up must have changed some of them
    raw = (acc.cpu().numpy() > 0).astype(np.uint16)
    final = np.zeros((n, KL), np.uint16)
    for t in range(L):
        for b in range(K):
            final[:, t * K + b] = (got[:, t] >> b) & 1
    exact = synth.bf16_bits_to_f32(k).astype(np.float64) @ W.astype(np.float64)
    flips = int(np.count_nonzero(raw != final))
    print(f"tensor-core signs corrected by the fix-up: {flips}; exact zero dots: {int(np.sum(exact == 0))}, "
          f"positive {int(np.sum(exact > 0))}")
    assert flips > 0
