"""Seeded synthetic inputs shared by the oracle tests, the GPU tests and bench.py.

This module holds NONE of the method's arithmetic (no centering, hashing,
collision test, probability or estimator): it only draws random numbers and
rounds them to bf16, the storage type of the KV cache ("bf16").
It imports neither ``oracle`` nor the CUDA package.

Workload recipe:

* keys / values: iid N(0, 1) rounded to bf16, layout ``[B][Hkv][n][d]``;
* queries: GQA group of G heads per kv head (query head ``h*G + g``);
  ``q_g = sigma * (rho * z0 + sqrt(1 - rho^2) * z_g)`` with sigma = 1.5 (logit
  std ~1.5) and rho = 0.8 (heads of one group look at similar tokens);
* an attention sink at position 0 whose logit against the group-mean query is
  ``sink_logit`` ("sink tokens ... high similarity");
* a planted fraction ``planted`` of the dynamic keys whose cosine with the
  group-mean query is ``planted_cos`` (the relevant "needle" tokens that make the
  sampled fraction approach the paper's empirical budget);
* projections ``W``: iid N(0, 1) rounded to bf16 (the paper stores 2-byte
  projectors), returned as fp32, shape ``[(d + mips)][K*L]``,
  one matrix shared by all heads.

Seeds: ``SeedSequence([20241021, cfg_id, b, h])`` per (sequence, kv head) and
``SeedSequence([20241021, 999, K, L, mips, d])`` for W, so any single unit of a
large configuration can be regenerated on its own.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import Dict, Tuple

import numpy as np

ROOT_SEED = 20241021


# ----------------------------------------------------------------------------
# bf16 storage helpers (format conversion only)

def bf16_bits_from_f32(x: np.ndarray) -> np.ndarray:
    """Round float32 values to bf16 (round to nearest, ties to even); uint16 bits."""
    x = np.ascontiguousarray(x, dtype=np.float32)
    u = x.view(np.uint32).astype(np.uint64)
    lsb = (u >> 16) & 1
    r = (u + 0x7FFF + lsb) >> 16
    return r.astype(np.uint16)


def bf16_bits_to_f32(h: np.ndarray) -> np.ndarray:
    h = np.ascontiguousarray(h, dtype=np.uint16)
    return (h.astype(np.uint32) << 16).view(np.float32)


# ----------------------------------------------------------------------------
# configurations (BASELINE.json "configs", restated in SURVEY.md 8(d))

@dataclass(frozen=True)
class Workload:
    name: str
    cfg_id: int
    B: int
    Hq: int
    Hkv: int
    n: int
    d: int = 128
    K: int = 10
    L: int = 150
    center: int = 1
    mips: int = 1
    min_collisions: int = 2
    sink: int = 4
    local: int = 64
    planted: float = 0.01
    planted_cos: float = 0.4
    sink_logit: float = 8.0
    sigma: float = 1.5
    rho: float = 0.8

    @property
    def G(self) -> int:
        return self.Hq // self.Hkv

    def with_(self, **kw) -> "Workload":
        d = dict(self.__dict__)
        d.update(kw)
        return Workload(**d)


CONFIGS: Dict[str, Workload] = {
    # configs[0]: single head d=128, n=1024 keys, K=10 L=150, one query
    "C1": Workload("C1", 1, B=1, Hq=1, Hkv=1, n=1024),
    # configs[1]: Llama-3.1-8B layer (32 q / 8 kv heads), 16K context, batch 1
    "C2": Workload("C2", 2, B=1, Hq=32, Hkv=8, n=16384),
    # configs[2]: Llama-3.1-8B, 64K context, batch 8, (K,L) sweep
    "C3_8_75": Workload("C3_8_75", 3, B=8, Hq=32, Hkv=8, n=65536, K=8, L=75),
    "C3": Workload("C3", 3, B=8, Hq=32, Hkv=8, n=65536, K=10, L=150),
    "C3_11_300": Workload("C3_11_300", 3, B=8, Hq=32, Hkv=8, n=65536, K=11, L=300),
    # configs[3]: Llama-3.1-70B (64 q / 8 kv heads), 96K context, heads sharded
    "C4": Workload("C4", 4, B=1, Hq=64, Hkv=8, n=98304),
    # configs[4]: 128K context, sequence sharded
    "C5": Workload("C5", 5, B=1, Hq=32, Hkv=8, n=131072),
}


# ----------------------------------------------------------------------------
# generators

def unit_rng(cfg_id: int, b: int, h: int) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(np.random.SeedSequence([ROOT_SEED, cfg_id, b, h])))


def make_projections(K: int, L: int, mips: int, d: int = 128) -> np.ndarray:
    """W: [(d + mips)][K*L] float32, every value exactly bf16-representable."""
    rng = np.random.Generator(np.random.PCG64(np.random.SeedSequence([ROOT_SEED, 999, K, L, mips, d])))
    w = rng.standard_normal((d + (1 if mips else 0), K * L), dtype=np.float32)
    return bf16_bits_to_f32(bf16_bits_from_f32(w))


def make_unit(wl: Workload, b: int, h: int, n: int | None = None) -> Tuple[np.ndarray, np.ndarray, np.ndarray]:
    """One (sequence b, kv head h): k, v uint16 [n][d] (bf16 bits), q uint16 [G][d]."""
    n = wl.n if n is None else n
    d, G = wl.d, wl.G
    rng = unit_rng(wl.cfg_id, b, h)
    z0 = rng.standard_normal(d)
    zg = rng.standard_normal((G, d))
    q = wl.sigma * (wl.rho * z0[None, :] + np.sqrt(1.0 - wl.rho ** 2) * zg)
    k = rng.standard_normal((n, d), dtype=np.float32)
    v = rng.standard_normal((n, d), dtype=np.float32)
    qm = q.mean(axis=0)
    qhat = qm / np.linalg.norm(qm)
    if n > 0 and wl.sink > 0:
        k[0] = (wl.sink_logit * np.sqrt(d) / np.linalg.norm(qm)) * qhat
    lo, hi = wl.sink, n - wl.local
    if wl.planted > 0 and hi > lo:
        cnt = int(round(wl.planted * (hi - lo)))
        if cnt > 0:
            pos = lo + rng.choice(hi - lo, size=cnt, replace=False)
            xi = rng.standard_normal((cnt, d))
            xi -= (xi @ qhat)[:, None] * qhat[None, :]
            xi /= np.linalg.norm(xi, axis=1, keepdims=True)
            c = wl.planted_cos
            direction = c * qhat[None, :] + np.sqrt(1.0 - c * c) * xi
            k[pos] = (np.sqrt(d) * direction).astype(np.float32)
    return bf16_bits_from_f32(k), bf16_bits_from_f32(v), bf16_bits_from_f32(q.astype(np.float32))


def make_batch(wl: Workload, n: int | None = None, threads: int = 1,
               b0: int = 0) -> Tuple[np.ndarray, np.ndarray, np.ndarray]:
    """Whole workload: k, v uint16 [B][Hkv][n][d]; q uint16 [B][Hq][d] (sequences b0 .. b0+B-1).
    Units are independent streams, so threads > 1 gives identical arrays."""
    n = wl.n if n is None else n
    k = np.empty((wl.B, wl.Hkv, n, wl.d), dtype=np.uint16)
    v = np.empty_like(k)
    q = np.empty((wl.B, wl.Hq, wl.d), dtype=np.uint16)

    def one(bh):
        b, h = bh
        ku, vu, qu = make_unit(wl, b0 + b, h, n)
        k[b, h], v[b, h] = ku, vu
        q[b, h * wl.G:(h + 1) * wl.G] = qu

    units = [(b, h) for b in range(wl.B) for h in range(wl.Hkv)]
    if threads > 1:
        from concurrent.futures import ThreadPoolExecutor
        with ThreadPoolExecutor(threads) as ex:
            list(ex.map(one, units))
    else:
        for bh in units:
            one(bh)
    return k, v, q


def make_random_case(seed: int, n: int, d: int, G: int, K: int, L: int, mips: int,
                     scale: float = 1.0) -> Dict[str, np.ndarray]:
    """Small iid case for property tests: k, v, q (bf16 bits) and W."""
    rng = np.random.Generator(np.random.PCG64(np.random.SeedSequence([ROOT_SEED, 4242, seed])))
    k = rng.standard_normal((n, d), dtype=np.float32) * np.float32(scale)
    v = rng.standard_normal((n, d), dtype=np.float32)
    q = rng.standard_normal((G, d), dtype=np.float32) * np.float32(1.5)
    w = rng.standard_normal((d + (1 if mips else 0), K * L), dtype=np.float32)
    return {
        "k": bf16_bits_from_f32(k), "v": bf16_bits_from_f32(v), "q": bf16_bits_from_f32(q),
        "W": bf16_bits_to_f32(bf16_bits_from_f32(w)),
    }
