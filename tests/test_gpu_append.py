"""Decode-time append + local-window rollover on the GPU against the
oracle (-m gpu): a multi-step decode loop that appends one key (and value) per kv head per step, crossing a
1024-key chunk boundary and rolling tokens out of the 64-token local window into the sampled set D.  At every
step the GPU index (codes of the new key hashed with the frozen centering vector and MIPS radius, reading R3)
and the oracle's incremental index (oracle.append_keys) must give the same S_g (bit-exact, incl. the rolled
tokens), the same |S_g|, and outputs within 2e-3 (R18)."""
from __future__ import annotations

import numpy as np
import pytest

import oracle
import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def _bf(a):
    if not torch.cuda.is_available():
        pytest.fail("GPU tests need a CUDA device (no fallback)")
    return torch.from_numpy(np.ascontiguousarray(a).view(np.int16)).view(torch.bfloat16).to("cuda:0")


@pytest.mark.parametrize("buckets,kernel", [(False, 0), (True, 0), (False, 7), (False, 8), (True, 9)])
def test_append_decode_loop(buckets, kernel):
    import paper_2410_16179_b200 as pkg
    steps, n0 = 20, 2040
    wl = synth.Workload("append", 970, B=1, Hq=4, Hkv=2, n=n0 + steps, K=8, L=40)
    k, v, q = synth.make_batch(wl)
    W = synth.make_projections(wl.K, wl.L, wl.mips)
    tk, tv, tq = _bf(k), _bf(v), _bf(q)
    tW = torch.from_numpy(W).to("cuda:0")
    pkg.binding.set_decode_kernel(kernel)
    try:
        mp = pkg.MagicPIG(tW, K=wl.K, L=wl.L, buckets=buckets).build(tk[:, :, :n0].contiguous())
        idx = [oracle.build_unit_q(k[0, h, :n0], W, wl.K, wl.L, wl.center, wl.mips, wl.sink, wl.local)
               for h in range(wl.Hkv)]
        for t in range(steps):
            n = n0 + t
            mp.append(tk[:, :, n:n + 1].contiguous())
            idx = [oracle.append_keys(idx[h], k[0, h, n:n + 1]) for h in range(wl.Hkv)]
            n1 = n + 1
            kk, vv = tk[:, :, :n1].contiguous(), tv[:, :, :n1].contiguous()
            nw = (n1 + 31) // 32
            s_mask = torch.zeros((1, wl.Hq, nw), dtype=torch.int32, device="cuda:0")
            s_count = torch.zeros((1, wl.Hq), dtype=torch.int32, device="cuda:0")
            out = mp.decode(tq, kk, vv, s_count=s_count, s_mask=s_mask)
            torch.cuda.synchronize()
            assert mp.status() == 0
            sm = s_mask.cpu().numpy().view(np.uint32)
            for h in range(wl.Hkv):
                ref = oracle.decode_indexed(idx[h], k[0, h, :n1], v[0, h, :n1], q[0, h * wl.G:(h + 1) * wl.G])
                assert idx[h]["status"] == 0 and ref["status"] in (0, oracle.OR_EDEGENERATE)
                for g in range(wl.G):
                    row = h * wl.G + g
                    bits = np.unpackbits(sm[0, row].view(np.uint8), bitorder="little")[:n1]
                    np.testing.assert_array_equal(bits, (ref["in_s"][g] == 1).astype(np.uint8),
                                                  err_msg=f"step {t} row {row}")
                    assert int(s_count.cpu()[0, row]) == int(ref["s_count"][g])
                    o, r = out.cpu().numpy()[0, row], ref["out"][g]
                    assert np.max(np.abs(o - r)) / np.max(np.abs(r)) <= 2e-3, (t, row)
        # the codes of every appended key equal the oracle's
        canon = torch.zeros((1, wl.Hkv, n0 + steps, wl.L), dtype=torch.int16, device="cuda:0")
        pkg.binding.export_codes(mp.cfg, mp.buf.codes, 1, wl.Hkv, n0 + steps, canon)
        for h in range(wl.Hkv):
            np.testing.assert_array_equal(canon.cpu().numpy().view(np.uint16)[0, h], idx[h]["codes"])
    finally:
        pkg.binding.set_decode_kernel(0)
