"""Python access to the double-precision CPU oracle (oracle/magicpig_oracle.c).

TEST INFRASTRUCTURE ONLY: only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import this
package.  The product path (``paper_2410_16179_b200``) never imports it, and
this package never imports the product path; they share no code.

The C library is plain fp64 loops following PAPER.md step by step (see the
citations in the C source).  This wrapper only marshals numpy arrays.
bf16 arrays are passed as ``uint16`` bit patterns.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from concurrent.futures import ThreadPoolExecutor
from typing import Dict, Optional

import numpy as np

_DIR = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_DIR, "magicpig_oracle.c")
_LIB = os.path.join(_DIR, "liboracle.so")

OR_OK, OR_EINVAL, OR_EINEXACT, OR_ENOTREPR, OR_EDEGENERATE = 0, -1, -2, -3, -4

CFLAGS = ["-O2", "-ffp-contract=off", "-std=c11", "-fPIC", "-shared"]


def build(force: bool = False) -> str:
    """Compile the oracle with gcc (plain C, no SIMD intrinsics, no FMA contraction)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", *CFLAGS, "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


_lib = None

_p = C.c_void_p
_i = C.c_int
_i64 = C.c_int64
_d = C.c_double


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(_LIB)
        L.oracle_bf16_to_double.argtypes = [C.c_uint16]
        L.oracle_bf16_to_double.restype = _d
        L.oracle_bf16_from_double.argtypes = [_d]
        L.oracle_bf16_from_double.restype = C.c_uint16
        L.oracle_exact_dot_sign.argtypes = [_p, _p, _i]
        L.oracle_exact_dot_sign.restype = _i
        L.oracle_is_static.argtypes = [_i64, _i64, _i, _i]
        L.oracle_is_static.restype = _i
        L.oracle_key_transform.argtypes = [_i, _i, _p, _i, _i, _i, _i, _p, _p, _p, _p, _p, _p, _p]
        L.oracle_key_transform.restype = _i
        L.oracle_check_w.argtypes = [_p, _i64]
        L.oracle_check_w.restype = _i
        L.oracle_encode_vec.argtypes = [_p, _i, _p, _i, _i, _p]
        L.oracle_encode_vec.restype = None
        L.oracle_encode_keys.argtypes = [_i, _i, _p, _p, _i, _i, _p]
        L.oracle_encode_keys.restype = None
        L.oracle_encode_query.argtypes = [_i, _i, _p, _p, _i, _i, _p]
        L.oracle_encode_query.restype = None
        L.oracle_collision_counts.argtypes = [_i, _i, _p, _p, _p]
        L.oracle_collision_counts.restype = None
        L.oracle_bucket_query.argtypes = [_i, _i, _i, _p, _p, _p]
        L.oracle_bucket_query.restype = None
        L.oracle_collision_prob.argtypes = [_d]
        L.oracle_collision_prob.restype = _d
        L.oracle_sampling_prob.argtypes = [_d, _i, _i, _i]
        L.oracle_sampling_prob.restype = _d
        L.oracle_sampling_prob_naive.argtypes = [_d, _i, _i]
        L.oracle_sampling_prob_naive.restype = _d
        L.oracle_expected_budget.argtypes = [_i, _i, _i]
        L.oracle_expected_budget.restype = _d
        L.oracle_exact_attention.argtypes = [_i, _i, _p, _p, _p, _p]
        L.oracle_exact_attention.restype = None
        L.oracle_exact_attention_f64.argtypes = [_i, _i, _p, _p, _p, _p]
        L.oracle_exact_attention_f64.restype = None
        L.oracle_estimate.argtypes = [_i, _i, _p, _p, _p, _p, _p, _p, _p, _p, _p]
        L.oracle_estimate.restype = _i
        L.oracle_decode_unit.argtypes = [_i, _i, _i, _i, _i, _i, _i, _i, _i, _i,
                                         _p, _p, _p, _p, _p, _p, _p, _p, _p, _p, _p, _p, _p, _p]
        L.oracle_decode_unit.restype = _i
        L.oracle_build_unit.argtypes = [_i, _i, _i, _i, _i, _i, _i, _i, _p, _p, _p, _p, _p, _p, _p]
        L.oracle_build_unit.restype = _i
        L.oracle_decode_indexed.argtypes = [_i, _i, _i, _i, _i, _i, _i, _i, _i, _p, _p, _p, _p, _p, _p, _p,
                                            _p, _p, _p, _p, _p, _p, _p]
        L.oracle_decode_indexed.restype = _i
        L.oracle_merge_partials.argtypes = [_i, _i, _p, _p]
        L.oracle_merge_partials.restype = _i
        L.oracle_softmax_f64.argtypes = [_i, _p, _p]
        L.oracle_softmax_f64.restype = None
        L.oracle_expectation.argtypes = [_i, _i, _p, _p, _p]
        L.oracle_expectation.restype = None
        L.oracle_topk_estimate.argtypes = [_i, _i, _p, _p, _i, _p]
        L.oracle_topk_estimate.restype = _i
        L.oracle_oracle_sampling.argtypes = [_i, _i, _p, _p, _i, _p, _p]
        L.oracle_oracle_sampling.restype = _i
        L.oracle_oracle_sampling_std.argtypes = [_i, _i, _p, _p, _i, _p]
        L.oracle_oracle_sampling_std.restype = None
        L.oracle_expected_unique.argtypes = [_i, _p, _i]
        L.oracle_expected_unique.restype = _d
        L.oracle_append_keys.argtypes = [_i, _i, _i, _i, _i, _p, _p, _p, _p, _p, _p, _p]
        L.oracle_append_keys.restype = _i
        _lib = L
    return _lib


def _ptr(a: Optional[np.ndarray]):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def _c(a, dt):
    return np.ascontiguousarray(a, dtype=dt)


# ----------------------------------------------------------------------------
# scalar helpers

def bf16_to_double(h: int) -> float:
    return lib().oracle_bf16_to_double(int(h))


def bf16_from_double(x: float) -> int:
    return int(lib().oracle_bf16_from_double(float(x)))


def collision_prob(cos: float) -> float:
    """p = 1 - arccos(cos)/pi."""
    return lib().oracle_collision_prob(float(cos))


def sampling_prob(p: float, K: int, L: int, min_collisions: int = 2) -> float:
    """u(p) of Eq. (LSH sampling probability) P:86-91 (stable form, reading R11)."""
    return lib().oracle_sampling_prob(float(p), int(K), int(L), int(min_collisions))


def sampling_prob_naive(p: float, K: int, L: int) -> float:
    return lib().oracle_sampling_prob_naive(float(p), int(K), int(L))


def expected_budget(K: int, L: int, min_collisions: int = 2) -> float:
    """Eq. (budget) P:472-476."""
    return lib().oracle_expected_budget(int(K), int(L), int(min_collisions))


def exact_dot_sign(a: np.ndarray, b: np.ndarray) -> int:
    a = _c(a, np.float64)
    b = _c(b, np.float64)
    return lib().oracle_exact_dot_sign(_ptr(a), _ptr(b), int(a.size))


def is_static(pos: int, n: int, sink: int, local: int) -> bool:
    return bool(lib().oracle_is_static(int(pos), int(n), int(sink), int(local)))


# ----------------------------------------------------------------------------
# array-level steps

def key_transform(k: np.ndarray, sink: int, local: int, center: int = 1, mips: int = 1):
    """Centering + MIPS transform for one unit. k: uint16 [n][d].
    Returns dict(c f32[d], xbar u16[n][d+mips], n2 f64[n], r2, status,
    ksum_q / r2_q / n2_q: the exact fixed-point integers (units of 2^-64) as
    Python ints)."""
    k = _c(k, np.uint16)
    n, d = k.shape
    dp = d + (1 if mips else 0)
    c = np.zeros(d, np.float32)
    xbar = np.zeros((n, dp), np.uint16)
    n2 = np.zeros(n, np.float64)
    r2 = C.c_double(0.0)
    ksum = np.zeros((d, 2), np.uint64)
    r2q = np.zeros(2, np.uint64)
    n2q = np.zeros((n, 2), np.uint64)
    st = lib().oracle_key_transform(n, d, _ptr(k), sink, local, center, mips, _ptr(c), _ptr(xbar),
                                    _ptr(n2), C.byref(r2), _ptr(ksum), _ptr(r2q), _ptr(n2q))
    return {"c": c, "xbar": xbar, "n2": n2, "r2": r2.value, "status": st,
            "ksum_q": [i128(x) for x in ksum], "r2_q": i128(r2q), "n2_q": [i128(x) for x in n2q]}


def i128(pair) -> int:
    """(lo, hi) uint64 pair -> Python int (two's complement)."""
    v = int(pair[0]) | (int(pair[1]) << 64)
    return v - (1 << 128) if v >= (1 << 127) else v


def encode_vec(vec: np.ndarray, W: np.ndarray, K: int, L: int) -> np.ndarray:
    vec = _c(vec, np.float64)
    W = _c(W, np.float32)
    out = np.zeros(L, np.uint16)
    lib().oracle_encode_vec(_ptr(vec), int(vec.size), _ptr(W), K, L, _ptr(out))
    return out


def encode_keys(xbar: np.ndarray, W: np.ndarray, K: int, L: int) -> np.ndarray:
    xbar = _c(xbar, np.uint16)
    W = _c(W, np.float32)
    n, dp = xbar.shape
    assert W.shape == (dp, K * L)
    out = np.zeros((n, L), np.uint16)
    lib().oracle_encode_keys(n, dp, _ptr(xbar), _ptr(W), K, L, _ptr(out))
    return out


def encode_query(q: np.ndarray, W: np.ndarray, K: int, L: int, mips: int) -> np.ndarray:
    q = _c(q, np.uint16)
    W = _c(W, np.float32)
    out = np.zeros(L, np.uint16)
    lib().oracle_encode_query(int(q.size), mips, _ptr(q), _ptr(W), K, L, _ptr(out))
    return out


def collision_counts(codes: np.ndarray, qcode: np.ndarray) -> np.ndarray:
    codes = _c(codes, np.uint16)
    qcode = _c(qcode, np.uint16)
    n, L = codes.shape
    cnt = np.zeros(n, np.int32)
    lib().oracle_collision_counts(n, L, _ptr(codes), _ptr(qcode), _ptr(cnt))
    return cnt


def bucket_query(codes: np.ndarray, qcode: np.ndarray, K: int) -> np.ndarray:
    codes = _c(codes, np.uint16)
    qcode = _c(qcode, np.uint16)
    n, L = codes.shape
    cnt = np.zeros(n, np.int32)
    lib().oracle_bucket_query(n, K, L, _ptr(codes), _ptr(qcode), _ptr(cnt))
    return cnt


def exact_attention(q: np.ndarray, k: np.ndarray, v: np.ndarray) -> np.ndarray:
    q, k, v = _c(q, np.uint16), _c(k, np.uint16), _c(v, np.uint16)
    n, d = k.shape
    out = np.zeros(d, np.float64)
    lib().oracle_exact_attention(n, d, _ptr(q), _ptr(k), _ptr(v), _ptr(out))
    return out


def exact_attention_f64(q: np.ndarray, k: np.ndarray, v: np.ndarray) -> np.ndarray:
    q, k, v = _c(q, np.float64), _c(k, np.float64), _c(v, np.float64)
    n, d = k.shape
    out = np.zeros(d, np.float64)
    lib().oracle_exact_attention_f64(n, d, _ptr(q), _ptr(k), _ptr(v), _ptr(out))
    return out


def estimate(q, k, v, sel, logu):
    """Eq. (close form) for a fixed candidate set; sel 0/1(S)/2(T)."""
    q, k, v = _c(q, np.uint16), _c(k, np.uint16), _c(v, np.uint16)
    sel = _c(sel, np.uint8)
    logu = _c(logu, np.float64)
    n, d = k.shape
    out = np.zeros(d, np.float64)
    a = np.zeros(d, np.float64)
    m = C.c_double(0.0)
    s = C.c_double(0.0)
    any_ = lib().oracle_estimate(n, d, _ptr(q), _ptr(k), _ptr(v), _ptr(sel), _ptr(logu), _ptr(out),
                                 C.byref(m), C.byref(s), _ptr(a))
    return {"out": out, "m": m.value, "s": s.value, "a": a, "any": bool(any_)}


# ---------------------------------------------------------------- estimator-quality harness (NEXT-3)
def softmax_f64(x: np.ndarray) -> np.ndarray:
    x = _c(x, np.float64)
    w = np.zeros_like(x)
    lib().oracle_softmax_f64(int(x.size), _ptr(x), _ptr(w))
    return w


def expectation(w: np.ndarray, v: np.ndarray) -> np.ndarray:
    """o = wV; v [n][d] (or [n] for scalars)."""
    w, v = _c(w, np.float64), _c(v.reshape(len(w), -1), np.float64)
    n, d = v.shape
    out = np.zeros(d, np.float64)
    lib().oracle_expectation(n, d, _ptr(w), _ptr(v), _ptr(out))
    return out


def topk_estimate(w: np.ndarray, v: np.ndarray, m: int) -> np.ndarray:
    """TopK attention, renormalized over the m largest weights."""
    w, v = _c(w, np.float64), _c(v.reshape(len(w), -1), np.float64)
    n, d = v.shape
    out = np.zeros(d, np.float64)
    lib().oracle_topk_estimate(n, d, _ptr(w), _ptr(v), int(m), _ptr(out))
    return out


def oracle_sampling(w: np.ndarray, v: np.ndarray, uniforms: np.ndarray):
    """Oracle sampling estimation with the caller's uniform variates -> (estimate, |S|)."""
    w, v, u = _c(w, np.float64), _c(v.reshape(len(w), -1), np.float64), _c(uniforms, np.float64)
    n, d = v.shape
    out = np.zeros(d, np.float64)
    uniq = lib().oracle_oracle_sampling(n, d, _ptr(w), _ptr(v), int(u.size), _ptr(u), _ptr(out))
    return out, int(uniq)


def oracle_sampling_std(w: np.ndarray, v: np.ndarray, B: int) -> np.ndarray:
    """Theorem 1: per-coordinate standard deviation of the oracle-sampling estimate with budget B."""
    w, v = _c(w, np.float64), _c(v.reshape(len(w), -1), np.float64)
    n, d = v.shape
    out = np.zeros(d, np.float64)
    lib().oracle_oracle_sampling_std(n, d, _ptr(w), _ptr(v), int(B), _ptr(out))
    return out


def expected_unique(w: np.ndarray, B: int) -> float:
    """Theorem 2: E|S| = sum_i (1 - (1 - w_i)^B)."""
    w = _c(w, np.float64)
    return float(lib().oracle_expected_unique(int(w.size), _ptr(w), int(B)))


def merge_partials(parts: np.ndarray) -> np.ndarray:
    parts = _c(parts, np.float64)
    P, dd = parts.shape
    out = np.zeros(dd - 2, np.float64)
    lib().oracle_merge_partials(P, dd - 2, _ptr(parts), _ptr(out))
    return out


def decode_unit(k, v, q, W, K: int, L: int, center: int = 1, mips: int = 1,
                min_collisions: int = 2, sink: int = 4, local: int = 64) -> Dict[str, np.ndarray]:
    """Algorithm 1 for one (sequence, kv head) with G query heads.
    k, v: uint16 [n][d]; q: uint16 [G][d]; W: f32 [(d+mips)][K*L]."""
    k, v = _c(k, np.uint16), _c(v, np.uint16)
    q = _c(q, np.uint16)
    if q.ndim == 1:
        q = q[None, :]
    W = _c(W, np.float32)
    n, d = k.shape
    G = q.shape[0]
    assert W.shape == (d + (1 if mips else 0), K * L), W.shape
    out = np.zeros((G, d), np.float64)
    partial = np.zeros((G, d + 2), np.float64)
    s_count = np.zeros(G, np.int32)
    counts = np.zeros((G, n), np.int32)
    in_s = np.zeros((G, n), np.uint8)
    codes = np.zeros((n, L), np.uint16)
    qcodes = np.zeros((G, L), np.uint16)
    c = np.zeros(d, np.float32)
    r2 = C.c_double(0.0)
    logu = np.zeros((G, n), np.float64)
    st = lib().oracle_decode_unit(n, d, G, K, L, center, mips, min_collisions, sink, local,
                                  _ptr(k), _ptr(v), _ptr(q), _ptr(W), _ptr(out), _ptr(partial),
                                  _ptr(s_count), _ptr(counts), _ptr(in_s), _ptr(codes), _ptr(qcodes),
                                  _ptr(c), C.byref(r2), _ptr(logu))
    return {"out": out, "partial": partial, "s_count": s_count, "counts": counts, "in_s": in_s,
            "codes": codes, "qcodes": qcodes, "c": c, "r2": r2.value, "logu": logu, "status": st}


def build_unit(k, W, K: int, L: int, center: int = 1, mips: int = 1, sink: int = 4, local: int = 64):
    """Build half of Alg. 1 for one unit: dict(xbar, n2, codes, c, r2, status)."""
    k = _c(k, np.uint16)
    W = _c(W, np.float32)
    n, d = k.shape
    dp = d + (1 if mips else 0)
    xbar = np.zeros((n, dp), np.uint16)
    n2 = np.zeros(n, np.float64)
    codes = np.zeros((n, L), np.uint16)
    c = np.zeros(d, np.float32)
    r2 = C.c_double(0.0)
    st = lib().oracle_build_unit(n, d, K, L, center, mips, sink, local, _ptr(k), _ptr(W), _ptr(xbar), _ptr(n2),
                                 _ptr(codes), _ptr(c), C.byref(r2))
    return {"xbar": xbar, "n2": n2, "codes": codes, "c": c, "r2": r2.value, "status": st, "K": K, "L": L,
            "mips": mips, "sink": sink, "local": local, "W": W}


def build_unit_q(k, W, K: int, L: int, center: int = 1, mips: int = 1, sink: int = 4, local: int = 64):
    """build_unit plus the exact fixed-point MIPS radius r2_q (a Python int), needed to append keys."""
    idx = build_unit(k, W, K, L, center, mips, sink, local)
    idx["r2_q"] = key_transform(k, sink, local, center, mips)["r2_q"]
    return idx


def append_keys(index, k_new):
    """Decode-time append (NEXT-2): hash k_new [m][d] with the index's frozen c and r^2 and return a new index
    for n + m keys (the local window rolls by position at decode time)."""
    k_new = _c(k_new, np.uint16)
    m, d = k_new.shape
    K, L, mips = index["K"], index["L"], index["mips"]
    dp = d + (1 if mips else 0)
    xbar = np.zeros((m, dp), np.uint16)
    n2 = np.zeros(m, np.float64)
    codes = np.zeros((m, L), np.uint16)
    r2q = index["r2_q"] & ((1 << 128) - 1)
    pair = np.array([r2q & ((1 << 64) - 1), r2q >> 64], np.uint64)
    st = lib().oracle_append_keys(m, d, K, L, mips, _ptr(k_new), _ptr(index["W"]), _ptr(_c(index["c"], np.float32)),
                                  _ptr(pair), _ptr(xbar), _ptr(n2), _ptr(codes))
    out = dict(index)
    out.update(xbar=np.vstack([index["xbar"], xbar]), n2=np.concatenate([index["n2"], n2]),
               codes=np.vstack([index["codes"], codes]), status=st)
    return out


def decode_indexed(index, k, v, q, min_collisions: int = 2):
    """Decode half of Alg. 1 for one unit given oracle.build_unit(...) output."""
    k, v = _c(k, np.uint16), _c(v, np.uint16)
    q = _c(q, np.uint16)
    if q.ndim == 1:
        q = q[None, :]
    n, d = k.shape
    G = q.shape[0]
    out = np.zeros((G, d), np.float64)
    s_count = np.zeros(G, np.int32)
    in_s = np.zeros((G, n), np.uint8)
    st = lib().oracle_decode_indexed(n, d, G, index["K"], index["L"], index["mips"], min_collisions,
                                     index["sink"], index["local"], _ptr(k), _ptr(v), _ptr(q), _ptr(index["W"]),
                                     _ptr(index["xbar"]), _ptr(index["n2"]), _ptr(index["codes"]), _ptr(out),
                                     None, _ptr(s_count), None, _ptr(in_s), None, None)
    return {"out": out, "s_count": s_count, "in_s": in_s, "status": st}


def decode_batch(k, v, q, W, K, L, center=1, mips=1, min_collisions=2, sink=4, local=64,
                 threads: Optional[int] = None):
    """All units of k [B][Hkv][n][d], q [B][Hq][d]; units run on parallel threads
    (the C call releases the GIL).  Returns a list indexed [b][h] of decode_unit dicts."""
    B, Hkv = k.shape[:2]
    G = q.shape[1] // Hkv
    jobs = [(b, h) for b in range(B) for h in range(Hkv)]
    threads = threads or min(len(jobs), os.cpu_count() or 1)

    def run(bh):
        b, h = bh
        return decode_unit(k[b, h], v[b, h], q[b, h * G:(h + 1) * G], W, K, L, center, mips,
                           min_collisions, sink, local)

    with ThreadPoolExecutor(max_workers=threads) as ex:
        res = list(ex.map(run, jobs))
    return [[res[b * Hkv + h] for h in range(Hkv)] for b in range(B)]
