"""Thin ctypes binding of libmagicpig.so (include/magicpig.h).

Argument marshalling only: every step of the method runs in the CUDA kernels
behind the C ABI.  Tensors are torch CUDA tensors (bf16 data as
torch.bfloat16); they are passed as raw device pointers on the current torch
stream.  There is no CPU fallback: if the shared library or a GPU is missing,
loading raises.
"""
from __future__ import annotations

import ctypes as C
import os
from typing import Optional

import torch

from . import build as _build

_p = C.c_void_p
_i = C.c_int
_i64 = C.c_int64
_sz = C.c_size_t

OK, EINVAL, ENOTREPR, EDEGENERATE, ECUDA, EWORKSPACE, EINEXACT, EOVERFLOW = 0, -1, -2, -3, -4, -5, -6, -7
STATUS_INEXACT, STATUS_OVERFLOW, STATUS_DEGENERATE, STATUS_NOTREPR = 1, 2, 4, 8
PART = 130
HEAD_DIM = 128


class magicpig_config(C.Structure):
    _fields_ = [("K", C.c_int32), ("L", C.c_int32), ("head_dim", C.c_int32), ("center", C.c_int32),
                ("mips", C.c_int32), ("min_collisions", C.c_int32), ("sink", C.c_int32), ("local", C.c_int32)]


def make_config(K=10, L=150, center=1, mips=1, min_collisions=2, sink=4, local=64) -> magicpig_config:
    return magicpig_config(K, L, HEAD_DIM, center, mips, min_collisions, sink, local)


_SIGS = {
    "magicpig_validate_config": ([_p], _i),
    "magicpig_codes_words": ([_p, _i64, _i64, _i64], _sz),
    "magicpig_build_workspace_bytes": ([_p, _i64, _i64, _i64], _sz),
    "magicpig_decode_workspace_bytes": ([_p, _i64, _i64, _i64, _i64], _sz),
    "magicpig_workspace_init": ([_p, _sz, _p], _i),
    "magicpig_workspace_status": ([_p, _p, _p], _i),
    "magicpig_key_stats": ([_p, _p, _i64, _i64, _i64, _i64, _i64, _p, _p, _p, _sz, _p], _i),
    "magicpig_key_norms": ([_p, _p, _i64, _i64, _i64, _i64, _i64, _p, _p, _p, _p, _p, _sz, _p], _i),
    "magicpig_reduce_stats": ([_i, _p, _p, _i, _i64, _i64, _p, _p, _p], _i),
    "magicpig_build_tables": ([_p, _p, _i64, _i64, _i64, _i64, _i64, _p, _p, _p, _p, _p, _p, _sz, _p], _i),
    "magicpig_build_index": ([_p, _p, _i64, _i64, _i64, _p, _p, _p, _p, _p, _p, _p, _p, _sz, _p], _i),
    "magicpig_decode": ([_p, _p, _i64, _p, _p, _p, _p, _p, _i64, _i64, _i64, _i64, _i64, _p, _p, _p, _p, _p,
                         _p, _sz, _p], _i),
    "magicpig_encode_queries": ([_p, _p, _i64, _i64, _p, _p, _sz, _p], _i),
    "magicpig_decode_encoded": ([_p, _p, _i64, _p, _p, _p, _p, _p, _i64, _i64, _i64, _i64, _i64, _p, _p, _p, _p,
                                 _p, _sz, _p], _i),
    "magicpig_merge_partials": ([_p, _i, _i64, _p, _p], _i),
    "magicpig_bucket_tables_words": ([_p, _i64, _i64, _i64], _sz),
    "magicpig_build_buckets": ([_p, _p, _i64, _i64, _i64, _p, _p], _i),
    "magicpig_decode_buckets": ([_p, _p, _i64, _p, _p, _p, _p, _p, _i64, _i64, _i64, _i64, _i64, _p, _p, _p, _p,
                                 _p, _p, _sz, _p], _i),
    "magicpig_decode_buckets_encoded": ([_p, _p, _i64, _p, _p, _p, _p, _p, _i64, _i64, _i64, _i64, _i64, _p, _p,
                                         _p, _p, _p, _sz, _p], _i),
    "magicpig_debug_set_decode_kernel": ([_i], _i),
    "magicpig_debug_decode_kernel_choice": ([_p, _i64, _i64, _i64, _i64, _i], _i),
    "magicpig_debug_decode_sets": ([_p, _p, _i64, _p, _p, _p, _p, _p, _p, _i64, _i64, _i64, _i64, _i64, _p, _p, _p,
                                    _p, _p, _sz, _p], _i),
    "magicpig_export_codes": ([_p, _p, _i64, _i64, _i64, _p, _p], _i),
    "magicpig_import_codes": ([_p, _p, _i64, _i64, _i64, _p, _p], _i),
    "magicpig_query_codes": ([_p, _p, _i64, _i64, _p, _p, _p, _sz, _p], _i),
    "magicpig_collision_counts": ([_p, _p, _i64, _p, _i64, _i64, _i64, _p, _p, _p, _sz, _p], _i),
    "magicpig_debug_hash_acc": ([_p, _p, _i64, _p, _p, _p, _p, _p, _sz, _p], _i),
    "magicpig_debug_decode_timeline": ([_p, _p, _i64, _p, _p, _p, _p, _p, _i64, _i64, _i64, _p, _p, _p, _i64, _p,
                                        _sz, _p], _i64),
    "magicpig_append_keys": ([_p, _p, _i64, _i64, _i64, _i64, _p, _p, _p, _p, _p, _p, _sz, _p], _i),
    "magicpig_decode_host": ([_p, _p, _i64, _p, _p, _p, _p, _p, _p, _i64, _i64, _i64, _p, _p, _p, _sz, _p], _i),
    "magicpig_debug_decode_stage": ([_p, _i, _p, _i64, _p, _p, _p, _p, _p, _p, _i64, _i64, _i64, _p, _p, _sz, _p],
                                    _i),
    "magicpig_debug_build_phases": ([_p, _p, _i64, _i64, _i64, _p, _p, _p, _p, _p, _p, _p, _p, _sz, _p, _p], _i),
    "magicpig_debug_decode_timeline_buckets": ([_p, _p, _i64, _p, _p, _p, _p, _p, _i64, _i64, _i64, _p, _p, _p,
                                                _i64, _p, _sz, _p], _i64),
    "magicpig_strerror": ([_i], C.c_char_p),
    "magicpig_version": ([], C.c_char_p),
    "magicpig_launch_count": ([], C.c_uint64),
}

_lib = None


def lib():
    """Load the in-tree shared library, (re)building it first if it is missing
    or older than its sources (so a kernel edit is never validated or timed
    against a stale binary)."""
    global _lib
    if _lib is None:
        path = _build.LIB
        alt = os.environ.get("MAGICPIG_LIB")  # debug: A/B against another build of the library
        if alt:
            path = alt
        elif _build._stale():
            path = _build.build()
        L = C.CDLL(path)
        for name, (args, res) in _SIGS.items():
            if alt and not hasattr(L, name):
                continue
            f = getattr(L, name)
            f.argtypes = args
            f.restype = res
        _lib = L
    return _lib


def exported_symbols():
    return list(_SIGS)


class MagicPIGError(RuntimeError):
    pass


def _check(rc: int, what: str):
    if rc != OK:
        raise MagicPIGError(f"{what}: {lib().magicpig_strerror(rc).decode()} ({rc})")


def _ptr(t: Optional[torch.Tensor]):
    if t is None:
        return None
    if not t.is_cuda:
        raise MagicPIGError("expected a CUDA tensor (no CPU fallback)")
    if not t.is_contiguous():
        raise MagicPIGError("expected a contiguous tensor")
    return C.c_void_p(t.data_ptr())


def _stream():
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


def _cfg(cfg):
    return C.byref(cfg)


# ---------------------------------------------------------------- sizes
def codes_words(cfg, B, Hkv, n):
    return int(lib().magicpig_codes_words(_cfg(cfg), B, Hkv, n))


def build_workspace_bytes(cfg, B, Hkv, n):
    return int(lib().magicpig_build_workspace_bytes(_cfg(cfg), B, Hkv, n))


def decode_workspace_bytes(cfg, B, Hq, Hkv, n):
    return int(lib().magicpig_decode_workspace_bytes(_cfg(cfg), B, Hq, Hkv, n))


def new_workspace(nbytes: int, device="cuda") -> torch.Tensor:
    ws = torch.empty(max(nbytes, 256), dtype=torch.uint8, device=device)
    workspace_init(ws)
    return ws


def workspace_init(ws):
    _check(lib().magicpig_workspace_init(_ptr(ws), ws.numel(), _stream()), "workspace_init")


def workspace_status(ws) -> int:
    st = C.c_uint32(0)
    _check(lib().magicpig_workspace_status(_ptr(ws), C.byref(st), _stream()), "workspace_status")
    return int(st.value)


# ---------------------------------------------------------------- build
def key_stats(cfg, k, seq_offset, n_global, key_sum, count, ws):
    B, Hkv, n, _ = k.shape
    _check(lib().magicpig_key_stats(_cfg(cfg), _ptr(k), B, Hkv, n, seq_offset, n_global, _ptr(key_sum),
                                    _ptr(count), _ptr(ws), ws.numel(), _stream()), "key_stats")


def key_norms(cfg, k, seq_offset, n_global, key_sum, count, center, r2, ws):
    B, Hkv, n, _ = k.shape
    _check(lib().magicpig_key_norms(_cfg(cfg), _ptr(k), B, Hkv, n, seq_offset, n_global, _ptr(key_sum),
                                    _ptr(count), _ptr(center), _ptr(r2), _ptr(ws), ws.numel(), _stream()),
           "key_norms")


def reduce_stats(mode, parts_sum, parts_cnt, P, B, Hkv, out_sum, out_cnt):
    _check(lib().magicpig_reduce_stats(mode, _ptr(parts_sum), _ptr(parts_cnt), P, B, Hkv, _ptr(out_sum),
                                       _ptr(out_cnt), _stream()), "reduce_stats")


def build_tables(cfg, k, seq_offset, n_global, W, center, r2, codes, key_norm, ws):
    B, Hkv, n, _ = k.shape
    _check(lib().magicpig_build_tables(_cfg(cfg), _ptr(k), B, Hkv, n, seq_offset, n_global, _ptr(W),
                                       _ptr(center), _ptr(r2), _ptr(codes), _ptr(key_norm), _ptr(ws), ws.numel(),
                                       _stream()), "build_tables")


def build_index(cfg, k, W, center, r2, codes, key_norm, key_sum, count, ws):
    B, Hkv, n, _ = k.shape
    _check(lib().magicpig_build_index(_cfg(cfg), _ptr(k), B, Hkv, n, _ptr(W), _ptr(center), _ptr(r2),
                                      _ptr(codes), _ptr(key_norm), _ptr(key_sum), _ptr(count), _ptr(ws), ws.numel(),
                                      _stream()), "build_index")


# ---------------------------------------------------------------- decode
def decode(cfg, q, codes, center, key_norm, k, v, seq_offset, n_global, W, ws, out=None, partial=None,
           s_count=None, s_mask=None):
    B, Hkv, n, _ = k.shape
    Hq = q.shape[1]
    _check(lib().magicpig_decode(_cfg(cfg), _ptr(q), Hq, _ptr(codes), _ptr(center), _ptr(key_norm), _ptr(k), _ptr(v),
                                 B, Hkv, n, seq_offset, n_global, _ptr(W), _ptr(out), _ptr(partial),
                                 _ptr(s_count), _ptr(s_mask), _ptr(ws), ws.numel(), _stream()), "decode")


def bucket_tables_words(cfg, B, Hkv, n) -> int:
    return int(lib().magicpig_bucket_tables_words(_cfg(cfg), B, Hkv, n))


def build_buckets(cfg, codes, B, Hkv, n, tables):
    _check(lib().magicpig_build_buckets(_cfg(cfg), _ptr(codes), B, Hkv, n, _ptr(tables), _stream()), "build_buckets")


def decode_buckets(cfg, q, tables, center, key_norm, k, v, seq_offset, n_global, W, ws, out=None, partial=None,
                   s_count=None, s_mask=None):
    B, Hkv, n, _ = k.shape
    Hq = q.shape[1]
    _check(lib().magicpig_decode_buckets(_cfg(cfg), _ptr(q), Hq, _ptr(tables), _ptr(center), _ptr(key_norm), _ptr(k),
                                         _ptr(v), B, Hkv, n, seq_offset, n_global, _ptr(W), _ptr(out), _ptr(partial),
                                         _ptr(s_count), _ptr(s_mask), _ptr(ws), ws.numel(), _stream()),
           "decode_buckets")


def decode_buckets_encoded(cfg, q, tables, center, key_norm, k, v, seq_offset, n_global, ws, out=None,
                           partial=None, s_count=None, s_mask=None):
    B, Hkv, n, _ = k.shape
    Hq = q.shape[1]
    _check(lib().magicpig_decode_buckets_encoded(_cfg(cfg), _ptr(q), Hq, _ptr(tables), _ptr(center), _ptr(key_norm),
                                                 _ptr(k), _ptr(v), B, Hkv, n, seq_offset, n_global, _ptr(out),
                                                 _ptr(partial), _ptr(s_count), _ptr(s_mask), _ptr(ws), ws.numel(),
                                                 _stream()), "decode_buckets_encoded")


def encode_queries(cfg, q, W, ws):
    Bn, Hq, _ = q.shape
    _check(lib().magicpig_encode_queries(_cfg(cfg), _ptr(q), Bn, Hq, _ptr(W), _ptr(ws), ws.numel(), _stream()),
           "encode_queries")


def decode_encoded(cfg, q, codes, center, key_norm, k, v, seq_offset, n_global, ws, out=None, partial=None,
                   s_count=None, s_mask=None):
    Bn, Hkv, n, _ = k.shape
    Hq = q.shape[1]
    _check(lib().magicpig_decode_encoded(_cfg(cfg), _ptr(q), Hq, _ptr(codes), _ptr(center), _ptr(key_norm), _ptr(k),
                                         _ptr(v), Bn, Hkv, n, seq_offset, n_global, _ptr(out), _ptr(partial),
                                         _ptr(s_count), _ptr(s_mask), _ptr(ws), ws.numel(), _stream()),
           "decode_encoded")


def decode_host(cfg, q_host, codes, tables, center, key_norm, k, v, W, out_host, ws):
    """One decode step from host memory: q_host [B][Hq][128] bf16 and out_host [B][Hq][128] fp32 are CPU
    tensors (pinned for asynchronous copies); returns after out_host holds the result."""
    B, Hkv, n, _ = k.shape
    Hq = q_host.shape[1]
    if q_host.is_cuda or out_host.is_cuda or q_host.dtype != torch.bfloat16 or out_host.dtype != torch.float32:
        raise MagicPIGError("decode_host takes CPU tensors: q_host bf16, out_host float32")
    if not (q_host.is_contiguous() and out_host.is_contiguous()) or tuple(out_host.shape) != (B, Hq, 128):
        raise MagicPIGError("decode_host: contiguous q_host [B][Hq][128] and out_host [B][Hq][128]")
    _check(lib().magicpig_decode_host(_cfg(cfg), C.c_void_p(q_host.data_ptr()), Hq, _ptr(codes), _ptr(tables),
                                      _ptr(center), _ptr(key_norm), _ptr(k), _ptr(v), B, Hkv, n, _ptr(W),
                                      C.c_void_p(out_host.data_ptr()), _ptr(ws), ws.numel(), _stream()), "decode_host")


def append_keys(cfg, k_new, n_old, W, center, r2, codes, key_norm, ws):
    """Hash the new keys k_new [B][Hkv][m][128] (positions n_old ..) with the frozen c, r^2 into codes /
    key_norm already laid out for n_old + m keys."""
    B, Hkv, m, _ = k_new.shape
    _check(lib().magicpig_append_keys(_cfg(cfg), _ptr(k_new), m, B, Hkv, n_old, _ptr(W), _ptr(center), _ptr(r2),
                                      _ptr(codes), _ptr(key_norm), _ptr(ws), ws.numel(), _stream()), "append_keys")


def merge_partials(parts, out):
    P, BH, _ = parts.shape
    _check(lib().magicpig_merge_partials(_ptr(parts), P, BH, _ptr(out), _stream()), "merge_partials")


# ---------------------------------------------------------------- debug
def export_codes(cfg, codes, B, Hkv, n, canonical):
    _check(lib().magicpig_export_codes(_cfg(cfg), _ptr(codes), B, Hkv, n, _ptr(canonical), _stream()),
           "export_codes")


def import_codes(cfg, canonical, B, Hkv, n, codes):
    _check(lib().magicpig_import_codes(_cfg(cfg), _ptr(canonical), B, Hkv, n, _ptr(codes), _stream()),
           "import_codes")


def query_codes(cfg, q, W, qcodes, ws):
    B, Hq, _ = q.shape
    _check(lib().magicpig_query_codes(_cfg(cfg), _ptr(q), B, Hq, _ptr(W), _ptr(qcodes), _ptr(ws), ws.numel(),
                                      _stream()), "query_codes")


def collision_counts(cfg, q, codes, k_shape, W, counts, ws):
    B, Hkv, n = k_shape[:3]
    Hq = q.shape[1]
    _check(lib().magicpig_collision_counts(_cfg(cfg), _ptr(q), Hq, _ptr(codes), B, Hkv, n, _ptr(W), _ptr(counts),
                                           _ptr(ws), ws.numel(), _stream()), "collision_counts")


def debug_hash_acc(cfg, k_unit, W, center, r2, acc, ws):
    n = k_unit.shape[0]
    _check(lib().magicpig_debug_hash_acc(_cfg(cfg), _ptr(k_unit), n, _ptr(W), _ptr(center), _ptr(r2), _ptr(acc),
                                         _ptr(ws), ws.numel(), _stream()), "debug_hash_acc")


def debug_decode_timeline(cfg, q, codes, center, key_norm, k, v, W, out, timeline, ws, buckets=False) -> int:
    """Kernel 5: per-CTA stamps [grid][32]; kernel 7: per-warp stamps [rows][16] (returns rows).  With
    buckets=True, `codes` is the bucketed tables."""
    Bn, Hkv, n, _ = k.shape
    if buckets:
        rc = lib().magicpig_debug_decode_timeline_buckets(_cfg(cfg), _ptr(q), q.shape[1], _ptr(codes), _ptr(center),
                                                          _ptr(key_norm), _ptr(k), _ptr(v), Bn, Hkv, n, _ptr(W),
                                                          _ptr(out), _ptr(timeline), timeline.numel(), _ptr(ws),
                                                          ws.numel(), _stream())
        if rc < 0:
            _check(int(rc), "debug_decode_timeline")
        return int(rc)
    Hq = q.shape[1]
    rc = lib().magicpig_debug_decode_timeline(_cfg(cfg), _ptr(q), Hq, _ptr(codes), _ptr(center), _ptr(key_norm),
                                              _ptr(k), _ptr(v), Bn, Hkv, n, _ptr(W), _ptr(out), _ptr(timeline),
                                              timeline.numel(), _ptr(ws), ws.numel(), _stream())
    if rc < 0:
        _check(int(rc), "debug_decode_timeline")
    return int(rc)


def debug_decode_sets(cfg, q, codes, tables, center, key_norm, k, v, seq_offset, n_global, W, ws, out, s_mask,
                      weighted):
    """One decode step that also exports S_g (restricted to D) and the (head, key) pairs that received a
    weight in the estimator's gather (S_g u T), as [B][Hq][ceil(n/32)] uint32 bitmaps."""
    B, Hkv, n, _ = k.shape
    Hq = q.shape[1]
    _check(lib().magicpig_debug_decode_sets(_cfg(cfg), _ptr(q), Hq, _ptr(codes), _ptr(tables), _ptr(center),
                                            _ptr(key_norm), _ptr(k), _ptr(v), B, Hkv, n, seq_offset, n_global, _ptr(W),
                                            _ptr(out), _ptr(s_mask), _ptr(weighted), _ptr(ws), ws.numel(), _stream()),
           "debug_decode_sets")


def debug_decode_stage(cfg, stage, q, codes, tables, center, key_norm, k, v, ws, out=None):
    """Debug: stage 1 = the Query kernel alone (S bitmaps into ws), stage 2 = the estimator kernel alone."""
    B, Hkv, n, _ = k.shape
    Hq = q.shape[1]
    _check(lib().magicpig_debug_decode_stage(_cfg(cfg), int(stage), _ptr(q), Hq, _ptr(codes), _ptr(tables),
                                             _ptr(center), _ptr(key_norm), _ptr(k), _ptr(v), B, Hkv, n, _ptr(out),
                                             _ptr(ws), ws.numel(), _stream()), "debug_decode_stage")


def debug_build_phases(cfg, k, W, center, r2, codes, key_norm, key_sum, count, ws, events):
    """build_index with torch.cuda.Event objects (5, enable_timing) recorded at the phase boundaries:
    stats | norms | prep | hash GEMM + fix-up."""
    B, Hkv, n, _ = k.shape
    for e in events:  # torch creates the CUDA event lazily, on its first record
        e.record()
    arr = (C.c_void_p * 5)(*[C.c_void_p(e.cuda_event) for e in events])
    _check(lib().magicpig_debug_build_phases(_cfg(cfg), _ptr(k), B, Hkv, n, _ptr(W), _ptr(center), _ptr(r2),
                                             _ptr(codes), _ptr(key_norm), _ptr(key_sum), _ptr(count), _ptr(ws),
                                             ws.numel(), _stream(), arr), "debug_build_phases")


def set_decode_kernel(version: int):
    """Debug knob (magicpig.h): 0 = automatic (default), 4..8 = a specific decode kernel generation."""
    _check(lib().magicpig_debug_set_decode_kernel(int(version)), "set_decode_kernel")


def decode_kernel_choice(cfg, B, Hq, Hkv, n, buckets=False) -> int:
    """The decode kernel generation the next decode with these shapes runs (resolves the automatic choice)."""
    rc = int(lib().magicpig_debug_decode_kernel_choice(_cfg(cfg), B, Hq, Hkv, n, int(bool(buckets))))
    if rc < 0:
        _check(rc, "decode_kernel_choice")
    return rc


def launch_count() -> int:
    return int(lib().magicpig_launch_count())


def version() -> str:
    return lib().magicpig_version().decode()
