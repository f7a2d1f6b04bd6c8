#!/usr/bin/env python
"""Benchmark of the MagicPIG decode hot path on B200.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config C3] [--path buckets|dense]
                  [--impl ours|reference] [--sweep SPEC,...]

One step = one MagicPIG decode step of one attention layer for the whole batch:
query Encode + Query(HT, q_code) + sampling / estimator
(P:109-116), all heads, with the KV cache and its index already resident in
HBM (the index build is reported separately under "build").

Workloads (BASELINE.json configs, synth.CONFIGS):
  C3 (default)  Llama-3.1-8B layer, B=8, 64K context, (K,L)=(10,150); batch
                sharded: every rank decodes its own 8 sequences (weak scaling,
                no collective on the data path).
  C2            the same layer at B=1, 16K.
  C4            Llama-3.1-70B layer (64 q / 8 kv heads), 96K, kv heads sharded
                over the ranks (strong scaling, no collective on the data path).
  C5            128K context, sequence sharded over the ranks: exact NCCL
                all-gathers of the centering / radius statistics at build, and
                per step one all-gather of the partial (m, s, a) states + a
                fixed-order log-sum-exp merge (strong scaling).
--path buckets (default) queries the paper's bucketed hash tables (inverted
lists); --path dense streams the packed codes of every key.

--gpus N > 1 without torchrun re-launches this script under
torch.distributed.run with N ranks on 127.0.0.1.  Time = CUDA events on the
launching stream around K steps, max over ranks.  L2: every timed step rotates
through R input replicas so the bytes a step touches were last touched R-1
steps earlier (R from the replica size; >= 2).
"""
from __future__ import annotations

import argparse
import dataclasses
import json
import os
import socket
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

import synth  # noqa: E402

METRIC = "decode attention tokens/s and HBM GB/s (% roofline) vs context len, 1/2/4/8 B200"
MODES = {"C1": "batch", "C2": "batch", "C3": "batch", "C3_8_75": "batch", "C3_11_300": "batch", "C4": "heads",
         "C5": "sequence"}
DEFAULT_SWEEP = ("C3_8_75:buckets,C3_11_300:buckets,C3:dense,C3_8_75:dense,C3_11_300:dense,"
                 "C2:buckets,C2:dense,C2:4096:buckets,C2:65536:buckets,C2:131072:buckets")


def _peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return ({"hbm": float(d["hbm_gbs"]), "bf16": float(d["bf16_tflops"]),
                 "bf16_sustained": float(d.get("bf16_tflops_sustained", d["bf16_tflops"]))},
                "measured (MEASURED_PEAKS.json)")
    return {"hbm": 6650.0, "bf16": 1650.0, "bf16_sustained": 1400.0}, "fallback (B200_PROFILING.md)"


def _traffic(kernel_key):
    """DRAM bytes per launch of a kernel (dram__bytes_read.sum + dram__bytes_write.sum) from the committed
    ncu --set full summary (tools/ncu_summary2.py), captured at the same workload, as (bytes, source), or
    None."""
    p = os.path.join(ROOT, "profiles", "ncu_summary.json")
    if os.path.exists(p):
        try:
            with open(p) as f:
                d = json.load(f)
            e = d.get(kernel_key)
            return (e["dram_bytes_per_launch"], f"profiles/ncu_summary.json ({d.get('tag')}, "
                    f"{e.get('capture')})") if e else None
        except Exception:
            return None
    return None


class ClockSampler:
    """NVML sampling of SM clock and throttle reasons during the timed region."""

    NAMES = {"gpu_idle": 0x1, "applications_clocks_setting": 0x2, "sw_power_cap": 0x4, "hw_slowdown": 0x8,
             "sync_boost": 0x10, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
             "hw_power_brake_slowdown": 0x80}

    def __init__(self, index=0, period=0.002):
        self.period = period
        self.samples = []
        self.reasons = set()
        self.max_mhz = None
        self._stop = threading.Event()
        self._t = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None

    def _run(self):
        nv = self.nv
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for k, bit in self.NAMES.items():
                    if r & bit:
                        self.reasons.add(k)
            except Exception:
                pass
            time.sleep(self.period)

    def __enter__(self):
        if self.nv:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons), "samples": 0}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons - {"gpu_idle"}), "samples": len(self.samples)}


# ----------------------------------------------------------------------------- launch / distribution
def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _relaunch(n):
    """Re-exec this script under torch.distributed.run with n ranks (one process per GPU)."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={_free_port()}", os.path.abspath(__file__)] + sys.argv[1:]
    os.execv(sys.executable, cmd)


def _dist(expect_world):
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    if ws != expect_world:
        raise SystemExit(f"bench.py --gpus {expect_world} but WORLD_SIZE={ws}")
    if ws > 1:
        import torch
        import torch.distributed as dist
        backend = os.environ.get("MAGICPIG_BENCH_BACKEND", "nccl")  # gloo: multi-rank check on one GPU
        if not dist.is_initialized():
            if backend == "nccl":
                torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")))
            dist.init_process_group(backend)
        return dist, dist.get_rank(), ws
    return None, 0, 1


def _dist_on():
    import torch.distributed as dist
    return dist.is_available() and dist.is_initialized()


def _gather_parts(part, group=None):
    """[P][rows][130] partial states of every rank (one rank: no collective)."""
    if not _dist_on():
        return part[None]
    from paper_2410_16179_b200.sharding import all_gather_stacked
    return all_gather_stacked(part, group)


def _device(local_rank):
    import torch
    n = torch.cuda.device_count()
    if n < 1:
        raise SystemExit("bench.py needs a CUDA device (there is no CPU fallback)")
    return torch.device("cuda", local_rank % n)


def _max_over_ranks(dist, dev, x):
    if not dist:
        return x
    import torch
    t = torch.tensor([x], dtype=torch.float64, device=dev if dist.get_backend() == "nccl" else "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


# ----------------------------------------------------------------------------- workload per rank
@dataclasses.dataclass
class RankWork:
    wl: synth.Workload       # the full workload
    mode: str
    B: int                   # sequences on this rank
    Hkv: int                 # kv heads on this rank
    Hq: int
    n: int                   # keys on this rank (per unit)
    seq_offset: int
    b0: int                  # first global sequence index
    h0: int                  # first global kv head
    units_total: int         # units of the whole job (for tokens/s)


def rank_work(wl, mode, rank, world):
    from paper_2410_16179_b200.sharding import head_shard, sequence_shard
    if mode == "batch":
        return RankWork(wl, mode, wl.B, wl.Hkv, wl.Hq, wl.n, 0, rank * wl.B, 0, world * wl.B * wl.Hkv)
    if mode == "heads":
        h0, h1 = head_shard(wl.Hkv, world, rank)
        if h1 <= h0:
            raise SystemExit(f"{wl.name}: {world} ranks > {wl.Hkv} kv heads")
        return RankWork(wl, mode, wl.B, h1 - h0, (h1 - h0) * wl.G, wl.n, 0, 0, h0, wl.B * wl.Hkv)
    lo, nl = sequence_shard(wl.n, world, rank)
    return RankWork(wl, mode, wl.B, wl.Hkv, wl.Hq, nl, lo, 0, 0, wl.B * wl.Hkv)


def make_rank_inputs(rw, threads):
    """k, v [B][Hkv_r][n_r][128], q [B][Hq_r][128] (bf16 bits) of this rank: the same seeded units as
    the unsharded workload (synth.make_unit), sliced by batch, kv head or key range."""
    wl = rw.wl
    k = np.empty((rw.B, rw.Hkv, rw.n, wl.d), np.uint16)
    v = np.empty_like(k)
    q = np.empty((rw.B, rw.Hq, wl.d), np.uint16)

    def one(bh):
        b, h = bh
        ku, vu, qu = synth.make_unit(wl, rw.b0 + b, rw.h0 + h)
        k[b, h], v[b, h] = ku[rw.seq_offset:rw.seq_offset + rw.n], vu[rw.seq_offset:rw.seq_offset + rw.n]
        q[b, h * wl.G:(h + 1) * wl.G] = qu

    from concurrent.futures import ThreadPoolExecutor
    with ThreadPoolExecutor(max(1, threads)) as ex:
        list(ex.map(one, [(b, h) for b in range(rw.B) for h in range(rw.Hkv)]))
    return k, v, q


# ----------------------------------------------------------------------------- algorithmic bytes
def alg_bytes(cfg_wl, B, Hq, Hkv, n, n_union, nT, path, ids_read=0, id_bytes=4):
    """Per step: query (codes of D, or bucket ids + offsets; + S bitmaps written), select (S bitmaps read,
    lists written), estimator (K/V rows + |xbar| of union_g S_g u T, lists read, q, c)."""
    KL = cfg_wl.K * cfg_wl.L
    nD = max(n - nT, 0)
    sbits = B * Hq * ((n + 31) // 32) * 4
    if path == "dense":
        q_read = B * Hkv * nD * KL / 8 + B * Hq * KL / 8
    else:
        q_read = ids_read * id_bytes + B * Hq * cfg_wl.L * 8 + B * Hq * KL / 8
    query = q_read + sbits
    select = sbits + n_union * 4 + B * Hkv * 4 + B * Hq * 4
    rows = (n_union + B * Hkv * nT)
    estimate = rows * 512 + rows * 4 + n_union * 4 + B * Hq * 256 + B * Hkv * 512 + B * Hq * 512
    # SURVEY 8(d) per-step formula (what the method must move): codes | bucket ids, rows, q/qcodes, c
    step = q_read + rows * 512 + n_union * 4 + B * Hq * 256 + B * Hkv * 512
    return {"query": query, "select": select, "estimate": estimate, "step": step}


def _graph_time(fn, R, launches, reps=5):
    """Median per-call time (us) of `launches` calls fn(i % R) captured in one CUDA graph."""
    import torch
    for i in range(R):
        fn(i)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for i in range(launches):
            fn(i % R)
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(reps):
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3 / launches)
    return float(np.median(ts))


class Replicas:
    """R copies (distinct addresses) of everything a decode step reads: KV cache, index, queries."""

    def __init__(self, rw, path, dev, R, tW, k, v, q, group=None):
        import torch
        import paper_2410_16179_b200 as pkg
        wl = rw.wl
        bf = lambda a: torch.from_numpy(np.ascontiguousarray(a).view(np.int16)).view(torch.bfloat16).to(dev)
        tk, tv, tq = bf(k), bf(v), bf(q)
        self.mps, self.ks, self.vs, self.qs = [], [], [], []
        for r in range(R):
            kr = tk if r == 0 else tk.clone()
            vr = tv if r == 0 else tv.clone()
            mp = pkg.MagicPIG(tW, K=wl.K, L=wl.L, center=wl.center, mips=wl.mips, min_collisions=wl.min_collisions,
                              sink=wl.sink, local=wl.local, buckets=(path == "buckets"))
            if rw.mode == "sequence" and _dist_on():
                mp.build_sharded(kr, rw.seq_offset, wl.n, group)
            else:
                mp.build(kr)
            mp.release_build_workspace()
            self.mps.append(mp), self.ks.append(kr), self.vs.append(vr), self.qs.append(tq.clone())
        torch.cuda.synchronize()
        self.R = R
        self.path = path
        self.cfg = self.mps[0].cfg
        self.ws = self.mps[0].decode_workspace(rw.B, rw.Hq, rw.Hkv, rw.n, dev)
        for mp in self.mps[1:]:
            mp._ws_dec = self.ws
        self.tW = tW

    def codes(self, r):
        return None if self.path == "buckets" else self.mps[r].buf.codes

    def tables(self, r):
        return self.mps[r].buf.tables if self.path == "buckets" else None


def measure_decode(rw, path, dev, tW, peaks, k, v, q, graph_steps=64, group=None, partial=False):
    """Build R replicas of this rank's index and time, in CUDA graphs: the whole step (encode + decode),
    and each kernel stage of the decode alone (Query, select, estimator).  Returns the measurements and
    the replicas (for the timed loop / e2e)."""
    import torch
    from paper_2410_16179_b200 import binding as B_
    wl = rw.wl
    per_rep = rw.B * rw.Hkv * rw.n * (512 + wl.K * wl.L / 8 + (wl.L * 4 if path == "buckets" else 0))
    R = int(min(16, max(2, -(-400e6 // per_rep))))
    reps = Replicas(rw, path, dev, R, tW, k, v, q, group)
    Bn, Hq, Hkv, n = rw.B, rw.Hq, rw.Hkv, rw.n
    cfg, ws = reps.cfg, reps.ws
    nw = (n + 31) // 32
    out = torch.empty((Bn, Hq, 128), dtype=torch.float32, device=dev)
    part = torch.empty((Bn * Hq, B_.PART), dtype=torch.float32, device=dev)
    smask = torch.zeros((Bn, Hq, nw), dtype=torch.int32, device=dev)
    scount = torch.zeros((Bn, Hq), dtype=torch.int32, device=dev)
    reps.mps[0].decode(reps.qs[0], reps.ks[0], reps.vs[0], out=out, s_count=scount, s_mask=smask)
    torch.cuda.synchronize()
    status = B_.workspace_status(ws)
    sm = smask.cpu().numpy().view(np.uint32).reshape(Bn, Hkv, wl.G, nw)
    union = np.bitwise_or.reduce(sm, axis=2)
    n_union = int(np.unpackbits(union.view(np.uint8)).sum())
    off, ng = reps.mps[0].seq_offset, reps.mps[0].n_global
    lo1, hi1 = max(0, -off), min(n, wl.sink - off)
    lo2, hi2 = max(0, ng - wl.local - off), min(n, ng - off)
    if hi1 > lo1 and lo2 < hi1:
        lo2 = hi1
    nT = max(0, hi1 - lo1) + max(0, hi2 - lo2)
    ids_read = 0
    if path == "buckets":
        qc = torch.zeros((Bn, Hq, wl.L), dtype=torch.int16, device=dev)
        B_.query_codes(cfg, reps.qs[0], tW, qc, ws)
        qc = qc.cpu().numpy().view(np.uint16).astype(np.int64)
        nb = 1 << wl.K
        per = B_.bucket_tables_words(cfg, 1, 1, n)  # words per unit (16-bit ids when n <= 65536)
        tabs = reps.mps[0].buf.tables
        for b in range(Bn):
            for hq in range(Hq):
                u = b * Hkv + hq // wl.G
                offs = tabs[u * per:u * per + wl.L * (nb + 1)].view(wl.L, nb + 1).cpu().numpy()
                c = qc[b, hq]
                ids_read += int((offs[np.arange(wl.L), c + 1] - offs[np.arange(wl.L), c]).sum())
    ab = alg_bytes(wl, Bn, Hq, Hkv, n, n_union, nT, path, ids_read, 2 if n <= 65536 else 4)

    if partial:
        def step(r):
            B_.encode_queries(cfg, reps.qs[r], tW, ws)
            dec = B_.decode_buckets_encoded if path == "buckets" else B_.decode_encoded
            dec(cfg, reps.qs[r], reps.tables(r) if path == "buckets" else reps.codes(r), reps.mps[r].buf.center,
                reps.mps[r].buf.key_norm, reps.ks[r], reps.vs[r], reps.mps[r].seq_offset, reps.mps[r].n_global, ws,
                partial=part)
    else:
        def step(r):
            B_.encode_queries(cfg, reps.qs[r], tW, ws)
            dec = B_.decode_buckets_encoded if path == "buckets" else B_.decode_encoded
            dec(cfg, reps.qs[r], reps.tables(r) if path == "buckets" else reps.codes(r), reps.mps[r].buf.center,
                reps.mps[r].buf.key_norm, reps.ks[r], reps.vs[r], 0, n, ws, out=out)

    def stage(bits):
        def fn(r):
            B_.debug_decode_stage(cfg, bits, reps.qs[r], reps.codes(r), reps.tables(r), reps.mps[r].buf.center,
                                  reps.mps[r].buf.key_norm, reps.ks[r], reps.vs[r], ws, out=out)
        return fn

    res = {"step_us": _graph_time(step, R, graph_steps)}
    choice = B_.decode_kernel_choice(cfg, Bn, Hq, Hkv, n, path == "buckets")
    res["decode_kernel"] = choice
    if rw.mode != "sequence":
        B_.encode_queries(cfg, reps.qs[0], tW, ws)
        kern = {}
        if choice == 5:  # one fused kernel (scan or bitmap Query + estimator + unit merge)
            def dec(r):
                d = B_.decode_buckets_encoded if path == "buckets" else B_.decode_encoded
                d(cfg, reps.qs[r], reps.tables(r) if path == "buckets" else reps.codes(r), reps.mps[r].buf.center,
                  reps.mps[r].buf.key_norm, reps.ks[r], reps.vs[r], 0, n, ws, out=out)
            us = _graph_time(dec, R, graph_steps)
            names = {"decode": "decode5_kernel" + (" (+ bucket_mark3_kernel)" if path == "buckets" else "")}
            ab["decode"] = ab["step"] - Bn * Hq * 256
            kern["decode"] = {"us": us, "alg_MB": ab["decode"] / 1e6}
        else:
            # stages 2 and 4 re-use replica 0's lists for every replica's K/V: the same bytes are moved
            kern["query"] = {"us": _graph_time(stage(1), R, graph_steps)}
            if path == "buckets":
                kern["select"] = {"us": _graph_time(stage(2), R, graph_steps)}
            else:  # the select step is fused into the dense scan
                ab["query"] += ab["select"]
            kern["estimate"] = {"us": _graph_time(stage(4), R, graph_steps), "note": "estimate + merge kernels"}
            names = {"query": "bucket_mark3_kernel" if path == "buckets" else "scan6_kernel (select fused)",
                     "select": "select_kernel", "estimate": {7: "estimate_kernel", 8: "estimate8_kernel", 9: "estimate9_kernel"}[choice]}
            for nm in kern:
                kern[nm]["alg_MB"] = ab[nm] / 1e6
        for nm, kd in kern.items():
            kd["GBs"] = kd["alg_MB"] * 1e6 / kd["us"] / 1e3
            kd["frac"] = kd["GBs"] / peaks["hbm"]
            kd["kernel"] = names[nm]
        res["kernels"] = kern
    res.update(n=n, B=Bn, Hq=Hq, Hkv=Hkv, K=wl.K, L=wl.L, path=path, replicas=R, union_rows=n_union, static_rows=nT,
               alg_bytes=ab, sampled_fraction=float(scount.float().mean()) / max(n - nT, 1), status=status,
               step_GBs=ab["step"] / res["step_us"] / 1e3, step_frac=ab["step"] / res["step_us"] / 1e3 / peaks["hbm"])
    if path == "buckets":
        res["ids_read"] = ids_read
    res["_reps"] = reps
    res["_step"] = step
    res["_out"] = out
    res["_part"] = part
    return res


def measure_build(rw, dev, tW, peaks, k):
    """Index build phases (events between the phases of one build): key statistics, norms / centering /
    MIPS radius, operand preparation, hash GEMM on tcgen05 + exact fix-up."""
    import torch
    import paper_2410_16179_b200 as pkg
    from paper_2410_16179_b200 import binding as B_
    wl = rw.wl
    tk = torch.from_numpy(np.ascontiguousarray(k).view(np.int16)).view(torch.bfloat16).to(dev)
    mp = pkg.MagicPIG(tW, K=wl.K, L=wl.L, center=wl.center, mips=wl.mips, min_collisions=wl.min_collisions,
                      sink=wl.sink, local=wl.local)
    mp.build(tk)  # warm (allocations, attributes)
    b = mp.buf
    ts = []
    for _ in range(3):
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(5)]
        B_.debug_build_phases(mp.cfg, tk, tW, b.center, b.r2, b.codes, b.key_norm, b.key_sum, b.count,
                              mp._ws_build, ev)
        torch.cuda.synchronize()
        ts.append([ev[i].elapsed_time(ev[i + 1]) * 1e3 for i in range(4)])
    st = mp.status("build")
    t = np.median(np.array(ts), axis=0)
    units = rw.B * rw.Hkv
    flops = 2.0 * units * rw.n * (128 + wl.mips) * wl.K * wl.L
    kbytes = units * rw.n * 256
    tf = flops / (t[3] * 1e-6) / 1e12
    return {"stats_us": t[0], "norms_us": t[1], "prep_us": t[2], "hash_gemm_us": t[3], "total_us": float(t.sum()),
            "hash_gflop": flops / 1e9, "hash_tflops": tf, "tensor_peak_tflops": peaks["bf16"],
            "tensor_frac": tf / peaks["bf16"], "stats_GBs": kbytes / t[0] / 1e3, "norms_GBs": kbytes / t[1] / 1e3,
            "prep_GBs": kbytes * 2.125 / t[2] / 1e3, "status": st,
            "note": "hash_gemm_us includes the exact fix-up kernel; prep writes the xbar tiles (256 B read + "
                    "288 B written per key)"}


# ----------------------------------------------------------------------------- CPU oracle (baseline / reference arm)
def cpu_oracle_unit(wl, steps_cap=None, target_s=10.0):
    """The oracle as it stands, on the host: build unit (b=0, h=0) once (untimed), then time decode steps
    of that unit single-threaded.  The whole-job step is extrapolated as units / cores unit-decodes
    (units are independent, one per host thread)."""
    import oracle
    k, v, q = synth.make_unit(wl, 0, 0)
    W = synth.make_projections(wl.K, wl.L, wl.mips)
    t0 = time.perf_counter()
    idx = oracle.build_unit(k, W, wl.K, wl.L, wl.center, wl.mips, wl.sink, wl.local)
    t_build = time.perf_counter() - t0
    oracle.decode_indexed(idx, k, v, q, wl.min_collisions)  # warm
    times = []
    t_start = time.perf_counter()
    while True:
        t = time.perf_counter()
        oracle.decode_indexed(idx, k, v, q, wl.min_collisions)
        times.append(time.perf_counter() - t)
        if (steps_cap and len(times) >= steps_cap) or (not steps_cap and time.perf_counter() - t_start > target_s):
            break
    cores = os.cpu_count() or 1
    units = wl.B * wl.Hkv
    t_unit = statistics.mean(times)
    step_s = t_unit * -(-units // cores)
    return {"value": wl.B / step_s, "step_s": step_s, "t_unit_s": t_unit, "steps": len(times), "cores": cores,
            "build_s": t_build,
            "sample": f"{wl.name} unit (b=0, kv head 0: n={wl.n}, G={wl.G}) decoded {len(times)} times "
                      f"single-threaded ({t_unit * 1e3:.1f} ms each; oracle build {t_build:.1f} s untimed); "
                      f"step = {units} independent units over {cores} host threads = "
                      f"{-(-units // cores)} unit-decodes per thread"}


# ----------------------------------------------------------------------------- ours
def run_ours(args):
    import torch
    from paper_2410_16179_b200 import binding as B_

    dist, rank, world = _dist(args.gpus)
    if args.kernel:
        B_.set_decode_kernel(args.kernel)
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    dev = _device(local_rank)
    torch.cuda.set_device(dev)
    group = None
    wl = synth.CONFIGS[args.config]
    mode = MODES[args.config]
    rw = rank_work(wl, mode, rank, world)
    path = args.path
    peaks, peak_src = _peaks()
    k, v, q = make_rank_inputs(rw, os.cpu_count() or 1)
    W = synth.make_projections(wl.K, wl.L, wl.mips)
    tW = torch.from_numpy(W).to(dev)

    m = measure_decode(rw, path, dev, tW, peaks, k, v, q, group=group, partial=(mode == "sequence"))
    reps, step = m.pop("_reps"), m.pop("_step")
    out, part = m.pop("_out"), m.pop("_part")
    R = reps.R

    merge_us = None
    if mode == "sequence":
        from paper_2410_16179_b200.sharding import all_gather_stacked
        out_m = torch.empty((rw.B, rw.Hq, 128), dtype=torch.float32, device=dev)

        g1 = torch.cuda.CUDAGraph()
        for i in range(R):
            step(i)
        torch.cuda.synchronize()
        graphs = []
        for r in range(R):
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                step(r)
            graphs.append(g)
        del g1

        def full_step(i):
            graphs[i % R].replay()
            B_.merge_partials(_gather_parts(part, group), out_m)

        def merge_only(i):
            B_.merge_partials(_gather_parts(part, group), out_m)
        timed = full_step
    else:
        GS = min(args.steps, 64)

        def capture(nsteps, offset=0):
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                for i in range(nsteps):
                    step((offset + i) % R)
            return g
        l0 = B_.launch_count()
        g_main = capture(GS)
        launches_per_graph = B_.launch_count() - l0
        rem = args.steps % GS
        g_rem = capture(rem) if rem else None
        reps_n = args.steps // GS

        def timed(i):
            raise AssertionError

    stream = torch.cuda.current_stream()
    # ---- warm-up (>= W steps), then exactly K timed steps between barriers + synchronize
    if mode == "sequence":
        for i in range(args.warmup):
            full_step(i)
    else:
        for _ in range(max(1, -(-args.warmup // GS))):
            g_main.replay()
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    l0 = B_.launch_count()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(dev.index) as clk:
        e0.record(stream)
        if mode == "sequence":
            for i in range(args.steps):
                full_step(i)
        else:
            for _ in range(reps_n):
                g_main.replay()
            if g_rem is not None:
                g_rem.replay()
        e1.record(stream)
        torch.cuda.synchronize()
        t_extra = time.perf_counter()  # keep sampling under load briefly if the region was short
        while time.perf_counter() - t_extra < 0.2:
            if mode == "sequence":
                full_step(0)
            else:
                g_main.replay()
            torch.cuda.synchronize()
    gpu_launches = (B_.launch_count() - l0 if mode == "sequence" else
                    reps_n * launches_per_graph + (launches_per_graph // GS) * rem)
    if dist:
        dist.barrier()
    ms = _max_over_ranks(dist, dev, e0.elapsed_time(e1))
    ms_step = ms / args.steps
    tokens_per_step = world * rw.B if mode == "batch" else rw.B
    value = tokens_per_step / (ms_step / 1e3)
    if mode == "sequence":
        torch.cuda.synchronize()
        f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        f0.record(stream)
        for i in range(args.steps):
            merge_only(i)
        f1.record(stream)
        torch.cuda.synchronize()
        merge_us = _max_over_ranks(dist, dev, f0.elapsed_time(f1) * 1e3 / args.steps)

    # ---- roofline of the dominant kernel (time measured alone, in its own graph, on this stream)
    roof = None
    if "kernels" in m:
        dom = max(m["kernels"], key=lambda kn: m["kernels"][kn]["us"])
        kd = m["kernels"][dom]
        kname = kd["kernel"].split(" ")[0]
        tr = _traffic(kname)
        roof = {"bound": "hbm", "achieved": kd["GBs"], "peak": peaks["hbm"], "unit": "GB/s", "frac": kd["frac"],
                "traffic": tr[0] if tr else None, "traffic_source": tr[1] if tr else None,
                "kernel": kd["kernel"], "kernel_us": kd["us"],
                "alg_bytes_per_launch": kd["alg_MB"] * 1e6, "peak_source": peak_src,
                "step": {"alg_bytes": m["alg_bytes"]["step"], "us": m["step_us"], "GBs": m["step_GBs"],
                         "frac": m["step_frac"]}}

    # ---- end to end through the C ABI from host buffers (magicpig_decode_host): per step the H2D copy of
    # q from pinned memory, encode, decode, the D2H copy of the output, and a stream synchronize (the host
    # has the step's output before it issues the next one).  Sequence mode: host q -> partial decode ->
    # NCCL all-gather -> merge -> host out.
    q_host = torch.from_numpy(np.ascontiguousarray(q).view(np.int16)).view(torch.bfloat16).pin_memory()
    out_host = torch.empty((rw.B, rw.Hq, 128), dtype=torch.float32).pin_memory()
    E = min(args.steps, args.e2e_steps)
    if mode == "sequence":
        from paper_2410_16179_b200.sharding import all_gather_stacked
        qd = torch.empty_like(reps.qs[0])

        def e2e_step(i):
            r = i % R
            qd.copy_(q_host, non_blocking=True)
            reps.mps[r].decode(qd, reps.ks[r], reps.vs[r], partial=part)
            B_.merge_partials(_gather_parts(part, group), out_m)
            out_host.copy_(out_m, non_blocking=True)
            torch.cuda.current_stream().synchronize()
    else:
        def e2e_step(i):
            r = i % R
            reps.mps[r].decode_host(q_host, reps.ks[r], reps.vs[r], out_host)
    for i in range(max(args.warmup, R)):
        e2e_step(i)
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    f0.record(stream)
    for i in range(E):
        e2e_step(i)
    f1.record(stream)
    torch.cuda.synchronize()
    e2e_ms = _max_over_ranks(dist, dev, f0.elapsed_time(f1) / E)
    e2e_value = tokens_per_step / (e2e_ms / 1e3)
    # correctness guard: the host output of the last e2e step equals the device path's output
    if mode != "sequence":
        reps.mps[(E - 1) % R].decode(reps.qs[0], reps.ks[(E - 1) % R], reps.vs[(E - 1) % R], out=out)
        torch.cuda.synchronize()
        assert torch.isfinite(out).all().item(), "non-finite output"
        assert torch.equal(out_host, out.cpu()), "host-path output differs from the device path"

    build = measure_build(rw, dev, tW, peaks, k) if rank == 0 and not args.no_build else None

    sweep = None
    if rank == 0 and args.sweep and world == 1:
        sweep = []
        for spec in args.sweep.split(","):
            parts = spec.split(":")
            name, pth, nn = parts[0], "buckets", None
            for p_ in parts[1:]:
                if p_ in ("buckets", "dense"):
                    pth = p_
                elif p_:
                    nn = int(p_)
            wl_s = synth.CONFIGS[name] if nn is None else dataclasses.replace(synth.CONFIGS[name], n=nn)
            if (wl_s, pth) == (wl, path):
                continue
            rw_s = rank_work(wl_s, "batch", 0, 1)
            ks, vs_, qs = make_rank_inputs(rw_s, os.cpu_count() or 1)
            tWs = tW if (wl_s.K, wl_s.L, wl_s.mips) == (wl.K, wl.L, wl.mips) else \
                torch.from_numpy(synth.make_projections(wl_s.K, wl_s.L, wl_s.mips)).to(dev)
            pt = measure_decode(rw_s, pth, dev, tWs, peaks, ks, vs_, qs)
            for key in ("_reps", "_step", "_out", "_part"):
                pt.pop(key)
            pt["config"] = name
            pt["tokens_per_s"] = wl_s.B / pt["step_us"] * 1e6
            sweep.append(pt)
            del ks, vs_, qs
            torch.cuda.empty_cache()

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        c = cpu_oracle_unit(wl, target_s=args.cpu_seconds)
        cpu = {"value": c["value"], "unit": "tokens/s", "cores": c["cores"], "kind": "oracle", "sample": c["sample"]}

    if rank == 0:
        par = {"batch": f"batch x{world} (each rank its own {rw.B} sequences; no collective)",
               "heads": f"kv heads / {world} ranks ({rw.Hkv} kv + {rw.Hq} q heads per rank; no collective)",
               "sequence": f"sequence / {world} ranks ({rw.n} keys per rank; NCCL all-gather of partial states "
                           f"+ fixed-order LSE merge per step)"}[mode]
        line = {
            "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
            "scaling": "weak" if mode == "batch" else "strong", "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic (seeded Llama-shaped KV cache, synth/)",
            "config": {"workload": f"{args.config}: B={wl.B}{' per GPU' if mode == 'batch' else ''}, Hq={wl.Hq}, "
                                   f"Hkv={wl.Hkv}, d=128, n={wl.n}, K={wl.K}, L={wl.L}, mips={wl.mips}, "
                                   f"center={wl.center}, sink={wl.sink}, local={wl.local}; path={path}",
                       "global_batch": tokens_per_step, "seq_len": wl.n, "parallelism": par,
                       "l2": f"{R} rotating input replicas (each step's bytes last touched {R - 1} steps earlier)",
                       "sampled_fraction": m["sampled_fraction"], "union_rows": m["union_rows"],
                       "alg_bytes_per_step": m["alg_bytes"]["step"], "status": m["status"]},
            "roofline": roof,
            "kernels": m.get("kernels"),
            "decode_kernel": m.get("decode_kernel"),
            "cpu_baseline": cpu,
            "e2e": {"value": e2e_value, "unit": "tokens/s", "h2d_bytes_per_step": int(q_host.numel() * 2),
                    "d2h_bytes_per_step": int(out_host.numel() * 4), "ms_per_step": e2e_ms,
                    "api": "magicpig_decode_host (C ABI, host buffers, synchronous)" if mode != "sequence" else
                           "host q -> decode(partial) -> NCCL all-gather -> merge -> host out, synchronous"},
            "gpu_launches": int(gpu_launches),
            "clocks": clk.summary(),
            "build": build,
            "context_sweep": sweep,
        }
        if merge_us is not None:
            line["merge_us"] = merge_us
            line["local_step_us"] = m["step_us"]
        print(json.dumps(line), flush=True)
    if dist:
        dist.barrier()
        dist.destroy_process_group()


# ----------------------------------------------------------------------------- reference arm
def run_reference(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    wl = synth.CONFIGS[args.config]
    c = cpu_oracle_unit(wl, steps_cap=max(1, min(args.steps, args.ref_steps_cap)))
    line = {
        "impl": "reference", "metric": METRIC, "value": c["value"], "unit": "tokens/s", "n_gpus": world,
        "steps": c["steps"], "warmup": args.warmup, "ms_per_step": c["step_s"] * 1e3, "higher_is_better": True,
        "scaling": "weak" if MODES[args.config] == "batch" else "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded Llama-shaped KV cache, synth/)",
        "config": {"workload": f"{args.config} (CPU oracle, double precision, plain C)", "global_batch": wl.B,
                   "seq_len": wl.n},
        "cpu_baseline": {"value": c["value"], "unit": "tokens/s", "cores": c["cores"], "kind": "oracle",
                         "sample": c["sample"]},
        "e2e": {"value": c["value"], "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=1000)
    ap.add_argument("--warmup", type=int, default=64)
    ap.add_argument("--config", default="C3", choices=sorted(MODES))
    ap.add_argument("--path", default="buckets", choices=["buckets", "dense"])
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--kernel", type=int, default=0, help="decode kernel (0 = the library's automatic choice)")
    ap.add_argument("--e2e-steps", type=int, default=300)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-build", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--ref-steps-cap", type=int, default=150)
    ap.add_argument("--sweep", default=DEFAULT_SWEEP,
                    help="extra points: comma list of CONFIG[:n][:buckets|dense] ('' = off)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.impl == "reference":
        run_reference(args)
        return
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        _relaunch(args.gpus)
    run_ours(args)


if __name__ == "__main__":
    main()
