"""MagicPIG index: device buffers + the build / decode sequence over the C ABI,
including multi-GPU sharding with torch.distributed (NCCL on GPUs).

Sharding:
  * heads / batch: each rank owns whole (sequence, kv head) units -> no
    collective on the data path (weak scaling);
  * sequence: each rank owns a contiguous key range.  Build: all-gather of the
    exact fixed-point centering sums (summed exactly on device), then of the
    per-shard MIPS radius (max on device) -> every rank hashes with the global
    c and r, so the union of the shards' S is the unsharded S.  Decode: each
    rank emits (m, s, a) partial states; one all-gather; the same fixed-order
    log-sum-exp merge on every rank ("recursive attention").
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Optional

import torch

from . import binding as B_
from .sharding import all_gather_stacked


@dataclass
class IndexBuffers:
    center: torch.Tensor   # [B][Hkv][128] f32
    r2: torch.Tensor       # [B][Hkv][2] int64 (q64)
    codes: torch.Tensor    # [codes_words] int32 (uint32 bit planes)
    key_norm: torch.Tensor  # [B][Hkv][n] f32 |xbar_i|
    key_sum: torch.Tensor  # [B][Hkv][128][2] int64 (q64)
    count: torch.Tensor    # [B][Hkv] int64
    tables: Optional[torch.Tensor] = None  # bucketed hash tables (int32 words), when buckets=True


class MagicPIG:
    """One attention layer's LSH index over a KV cache k, v [B][Hkv][n][128] bf16."""

    def __init__(self, W: torch.Tensor, K=10, L=150, center=1, mips=1, min_collisions=2, sink=4, local=64,
                 buckets=False):
        """buckets=True also builds the paper's hash tables as inverted lists (per table, key ids sorted by
        code) and decodes by reading only the query's buckets (same S as the dense code scan)."""
        self.cfg = B_.make_config(K, L, center, mips, min_collisions, sink, local)
        self.buckets = bool(buckets)
        rc = B_.lib().magicpig_validate_config(B_.C.byref(self.cfg))
        if rc != 0:
            raise B_.MagicPIGError("unsupported configuration")
        if W.dtype != torch.float32 or not W.is_cuda:
            raise B_.MagicPIGError("W must be a CUDA float32 tensor [(128+mips)][K*L]")
        if tuple(W.shape) != (128 + (1 if mips else 0), K * L):
            raise B_.MagicPIGError(f"W shape {tuple(W.shape)} != {(128 + mips, K * L)}")
        self.W = W.contiguous()
        self.buf: Optional[IndexBuffers] = None
        self._ws_build = None
        self._ws_dec = None
        self.seq_offset = 0
        self.n_global = 0
        self.shape = None

    # ------------------------------------------------------------ helpers
    def _alloc(self, Bn, Hkv, n, dev):
        words = B_.codes_words(self.cfg, Bn, Hkv, n)
        self.buf = IndexBuffers(
            center=torch.empty((Bn, Hkv, 128), dtype=torch.float32, device=dev),
            r2=torch.empty((Bn, Hkv, 2), dtype=torch.int64, device=dev),
            codes=torch.empty((max(words, 1),), dtype=torch.int32, device=dev),
            key_norm=torch.empty((Bn, Hkv, max(n, 1)), dtype=torch.float32, device=dev),
            key_sum=torch.empty((Bn, Hkv, 128, 2), dtype=torch.int64, device=dev),
            count=torch.empty((Bn, Hkv), dtype=torch.int64, device=dev))
        nb = B_.build_workspace_bytes(self.cfg, Bn, Hkv, n)
        if self._ws_build is None or self._ws_build.numel() < nb:
            self._ws_build = B_.new_workspace(nb, dev)

    def decode_workspace(self, Bn, Hq, Hkv, n, dev):
        nb = B_.decode_workspace_bytes(self.cfg, Bn, Hq, Hkv, n)
        if self._ws_dec is None or self._ws_dec.numel() < nb:
            self._ws_dec = B_.new_workspace(nb, dev)
        return self._ws_dec

    def release_build_workspace(self):
        self._ws_build = None

    # ------------------------------------------------------------ build
    def build(self, k: torch.Tensor):
        """Unsharded build over k [B][Hkv][n][128] bf16."""
        Bn, Hkv, n, d = k.shape
        self._alloc(Bn, Hkv, n, k.device)
        b = self.buf
        B_.build_index(self.cfg, k, self.W, b.center, b.r2, b.codes, b.key_norm, b.key_sum, b.count, self._ws_build)
        self.seq_offset, self.n_global, self.shape = 0, n, (Bn, Hkv, n)
        self._build_buckets()
        return self

    def _build_buckets(self):
        if not self.buckets:
            return
        Bn, Hkv, n = self.shape
        words = B_.bucket_tables_words(self.cfg, Bn, Hkv, n)
        if words == 0:
            raise B_.MagicPIGError("bucketed tables unsupported for this configuration (K <= 14, n <= 819200)")
        self.buf.tables = torch.empty((words,), dtype=torch.int32, device=self.buf.codes.device)
        B_.build_buckets(self.cfg, self.buf.codes, Bn, Hkv, n, self.buf.tables)

    def append(self, k_new: torch.Tensor):
        """Decode-time append: the new keys k_new [B][Hkv][m][128] bf16 become positions
        n .. n+m-1, hashed with the frozen centering vector and MIPS radius of the build; the local window of
        the static set rolls with n at the next decode.  The index buffers are re-laid out for n + m keys
        (plumbing); the bucketed tables, when present, are rebuilt from the codes."""
        if self.buf is None or self.seq_offset != 0:
            raise B_.MagicPIGError("append needs an unsharded built index")
        Bn, Hkv, n = self.shape
        if k_new.dtype != torch.bfloat16 or k_new.dim() != 4 or tuple(k_new.shape[:2]) != (Bn, Hkv) or \
                k_new.shape[3] != 128:
            raise B_.MagicPIGError(f"k_new must be bfloat16 [{Bn}][{Hkv}][m][128]")
        m = k_new.shape[2]
        n_new = n + m
        b = self.buf
        units = Bn * Hkv
        w_old, w_new = B_.codes_words(self.cfg, Bn, Hkv, n), B_.codes_words(self.cfg, Bn, Hkv, n_new)
        if w_new != w_old:  # a new 1024-key chunk per unit: move each unit's chunks to the wider layout
            codes = torch.zeros((w_new,), dtype=torch.int32, device=b.codes.device)
            codes.view(units, -1)[:, :w_old // units].copy_(b.codes[:w_old].view(units, -1))
            b.codes = codes
        key_norm = torch.empty((Bn, Hkv, n_new), dtype=torch.float32, device=b.key_norm.device)
        key_norm[:, :, :n].copy_(b.key_norm[:, :, :n])
        b.key_norm = key_norm
        ws = self._ws_dec if self._ws_dec is not None else B_.new_workspace(256, k_new.device)
        B_.append_keys(self.cfg, k_new.contiguous(), n, self.W, b.center, b.r2, b.codes, b.key_norm, ws)
        self.shape, self.n_global = (Bn, Hkv, n_new), n_new
        self._build_buckets()
        return self

    def build_sharded(self, k_local: torch.Tensor, seq_offset: int, n_global: int, group=None):
        """Sequence-sharded build: this rank holds keys [seq_offset, seq_offset + n_local)."""
        import torch.distributed as dist
        Bn, Hkv, n, d = k_local.shape
        self._alloc(Bn, Hkv, n, k_local.device)
        b = self.buf
        ws = self._ws_build
        P = dist.get_world_size(group)
        ks = torch.empty_like(b.key_sum)
        cnt = torch.empty_like(b.count)
        B_.key_stats(self.cfg, k_local, seq_offset, n_global, ks, cnt, ws)
        all_ks = all_gather_stacked(ks, group)
        all_cnt = all_gather_stacked(cnt, group)
        B_.reduce_stats(0, all_ks, all_cnt, P, Bn, Hkv, b.key_sum, b.count)
        r2_local = torch.empty_like(b.r2)
        B_.key_norms(self.cfg, k_local, seq_offset, n_global, b.key_sum, b.count, b.center, r2_local, ws)
        all_r2 = all_gather_stacked(r2_local, group)
        B_.reduce_stats(1, all_r2, None, P, Bn, Hkv, b.r2, None)
        B_.build_tables(self.cfg, k_local, seq_offset, n_global, self.W, b.center, b.r2, b.codes, b.key_norm, ws)
        self.seq_offset, self.n_global, self.shape = seq_offset, n_global, (Bn, Hkv, n)
        self._build_buckets()
        return self

    # ------------------------------------------------------------ decode
    def _check_decode_args(self, q, k, v, out=None, partial=None, s_count=None, s_mask=None):
        """Shapes and dtypes against the built index: a mismatch would be an out-of-bounds device access."""
        if self.buf is None:
            raise B_.MagicPIGError("build the index first")
        if k.dtype != torch.bfloat16 or v.dtype != torch.bfloat16:
            raise B_.MagicPIGError("k and v must be bfloat16")
        if k.dim() != 4 or tuple(k.shape[:3]) != tuple(self.shape) or k.shape[3] != 128 or v.shape != k.shape:
            raise B_.MagicPIGError(f"k, v must be [B][Hkv][n][128] = {tuple(self.shape)} + (128,) (the built index); "
                                   f"got {tuple(k.shape)}, {tuple(v.shape)}")
        Bn, Hkv, n = self.shape
        if q.dim() != 3 or q.shape[0] != Bn or q.shape[2] != 128 or q.shape[1] % Hkv:
            raise B_.MagicPIGError(f"q must be [B={Bn}][G*{Hkv}][128]; got {tuple(q.shape)}")
        if not q.is_cuda and q.dtype == torch.bfloat16:
            return
        if q.dtype != torch.bfloat16:
            raise B_.MagicPIGError("q must be bfloat16")
        Hq = q.shape[1]
        if out is not None and (out.dtype != torch.float32 or tuple(out.shape) != (Bn, Hq, 128)):
            raise B_.MagicPIGError(f"out must be float32 [{Bn}][{Hq}][128]")
        if partial is not None and (partial.dtype != torch.float32 or partial.numel() != Bn * Hq * B_.PART):
            raise B_.MagicPIGError(f"partial must be float32 [{Bn * Hq}][{B_.PART}]")
        if s_count is not None and (s_count.dtype != torch.int32 or s_count.numel() != Bn * Hq):
            raise B_.MagicPIGError(f"s_count must be int32 [{Bn}][{Hq}]")
        if s_mask is not None and (s_mask.dtype != torch.int32 or s_mask.numel() != Bn * Hq * ((n + 31) // 32)):
            raise B_.MagicPIGError(f"s_mask must be int32 [{Bn}][{Hq}][{(n + 31) // 32}]")

    def decode(self, q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, out=None, partial=None,
               s_count=None, s_mask=None):
        """One decode step for q [B][Hq][128] bf16 over this rank's keys."""
        self._check_decode_args(q, k, v, out, partial, s_count, s_mask)
        Bn, Hkv, n, _ = k.shape
        Hq = q.shape[1]
        ws = self.decode_workspace(Bn, Hq, Hkv, n, q.device)
        if out is None and partial is None:
            out = torch.empty((Bn, Hq, 128), dtype=torch.float32, device=q.device)
        b = self.buf
        if self.buckets:
            B_.decode_buckets(self.cfg, q, b.tables, b.center, b.key_norm, k, v, self.seq_offset, self.n_global,
                              self.W, ws, out=out, partial=partial, s_count=s_count, s_mask=s_mask)
        else:
            B_.decode(self.cfg, q, b.codes, b.center, b.key_norm, k, v, self.seq_offset, self.n_global, self.W, ws,
                      out=out, partial=partial, s_count=s_count, s_mask=s_mask)
        return out if out is not None else partial

    def decode_host(self, q_host: torch.Tensor, k: torch.Tensor, v: torch.Tensor, out_host=None):
        """One serving step from host memory through the C ABI (magicpig_decode_host): q_host [B][Hq][128]
        bf16 on the CPU (pinned for an asynchronous copy) -> out_host [B][Hq][128] float32 on the CPU,
        valid on return.  Unsharded indexes only."""
        self._check_decode_args(q_host, k, v)
        if self.seq_offset != 0 or self.n_global != self.shape[2]:
            raise B_.MagicPIGError("decode_host is for unsharded indexes")
        Bn, Hkv, n, _ = k.shape
        Hq = q_host.shape[1]
        if out_host is None:
            out_host = torch.empty((Bn, Hq, 128), dtype=torch.float32).pin_memory()
        ws = self.decode_workspace(Bn, Hq, Hkv, n, k.device)
        b = self.buf
        B_.decode_host(self.cfg, q_host, None if self.buckets else b.codes, b.tables if self.buckets else None,
                       b.center, b.key_norm, k, v, self.W, out_host, ws)
        return out_host

    def decode_sharded(self, q, k_local, v_local, group=None, out=None, s_count=None):
        """Sequence-sharded decode: partial states, one all-gather, fixed-order merge."""
        Bn, Hkv, n, _ = k_local.shape
        Hq = q.shape[1]
        part = torch.empty((Bn * Hq, B_.PART), dtype=torch.float32, device=q.device)
        self.decode(q, k_local, v_local, partial=part, s_count=s_count)
        allp = all_gather_stacked(part, group)
        if out is None:
            out = torch.empty((Bn, Hq, 128), dtype=torch.float32, device=q.device)
        B_.merge_partials(allp, out)
        return out

    def status(self, which="decode") -> int:
        ws = self._ws_dec if which == "decode" else self._ws_build
        return B_.workspace_status(ws) if ws is not None else 0


class DecodeSession:
    """A serving step as ONE CUDA graph (CUDA graphs instead of a tracing compiler): the H2D copy of
    q from a pinned host buffer, the query encode, the decode kernel and the D2H copy of the output
    into a pinned host buffer.  ``step()`` replays it asynchronously on the current stream; write the
    next query into ``q_host`` and read the result from ``out_host`` after synchronising.  The graph
    binds this index, k and v: rebuild the session if they change."""

    def __init__(self, mp: MagicPIG, k: torch.Tensor, v: torch.Tensor, Hq: int):
        Bn, Hkv, n, _ = k.shape
        dev = k.device
        self.q_host = torch.zeros((Bn, Hq, 128), dtype=torch.bfloat16).pin_memory()
        self.out_host = torch.zeros((Bn, Hq, 128), dtype=torch.float32).pin_memory()
        self.q_dev = torch.zeros((Bn, Hq, 128), dtype=torch.bfloat16, device=dev)
        self.out_dev = torch.zeros((Bn, Hq, 128), dtype=torch.float32, device=dev)
        mp.decode_workspace(Bn, Hq, Hkv, n, dev)
        self._mp, self._k, self._v = mp, k, v
        # the graph holds raw pointers: keep every buffer it captured alive, and refuse to replay
        # once the index was rebuilt or the workspace replaced
        self._held = (mp.buf, mp._ws_dec, mp.W)
        side = torch.cuda.Stream(device=dev)
        side.wait_stream(torch.cuda.current_stream(dev))
        with torch.cuda.stream(side):  # warm-up outside the capture (library attributes, allocations)
            self._body()
        torch.cuda.current_stream(dev).wait_stream(side)
        torch.cuda.synchronize(dev)
        self.graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.graph):
            self._body()
        torch.cuda.synchronize(dev)

    def _body(self):
        self.q_dev.copy_(self.q_host, non_blocking=True)
        self._mp.decode(self.q_dev, self._k, self._v, out=self.out_dev)
        self.out_host.copy_(self.out_dev, non_blocking=True)

    def step(self):
        if self._mp.buf is not self._held[0] or self._mp._ws_dec is not self._held[1]:
            raise B_.MagicPIGError("the index or its workspace changed since this session was captured; "
                                   "create a new session")
        self.graph.replay()
        return self.out_host


def session(mp: MagicPIG, k: torch.Tensor, v: torch.Tensor, Hq: int) -> DecodeSession:
    """Graph-captured decode step for serving (see DecodeSession)."""
    return DecodeSession(mp, k, v, Hq)
