#!/usr/bin/env python
"""Benchmark of the MagicPIG decode hot path on B200.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config C2] [--impl ours|reference]

One step = one MagicPIG decode step of one attention layer for the whole batch:
query Encode + Query / sampling / estimator, all heads, with
the KV cache and its index already resident in HBM.  Default workload: BASELINE
config[1] (C2, Llama-3.1-8B layer, 32 q / 8 kv heads, d=128, 16K context, B=1,
K=10, L=150).  Under torchrun each rank decodes its own sequence(s) (heads/batch
sharding: no collective on the data path -> weak scaling); time = max over ranks.

L2: every timed step rotates through R input replicas (codes + K/V + index), so
the bytes a step touches were last touched R-1 steps earlier (> L2 capacity).
"""
from __future__ import annotations

import argparse
import json
import os
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


def _peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md)"


def _traffic(kernel_key="decode"):
    p = os.path.join(ROOT, "profiles", "ncu_summary.json")
    if os.path.exists(p):
        try:
            with open(p) as f:
                d = json.load(f)
            return d.get(kernel_key, {}).get("dram_bytes_per_launch")
        except Exception:
            return None
    return None


class ClockSampler:
    """NVML sampling of SM clock and throttle reasons during the timed region."""

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
        names = {
            "gpu_idle": 0x1, "applications_clocks_setting": 0x2, "sw_power_cap": 0x4, "hw_slowdown": 0x8,
            "sync_boost": 0x10, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
            "hw_power_brake_slowdown": 0x80,
        }
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for k, bit in names.items():
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


def _dist():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    if ws > 1:
        import torch.distributed as dist
        if not dist.is_initialized():
            dist.init_process_group("nccl")
        return dist, dist.get_rank(), ws
    return None, 0, 1


def _workload(name):
    return synth.CONFIGS[name]


def _make_inputs(wl, rank):
    """This rank's batch: sequence indices rank*B .. rank*B + B - 1 (weak scaling)."""
    k = np.empty((wl.B, wl.Hkv, wl.n, wl.d), np.uint16)
    v = np.empty_like(k)
    q = np.empty((wl.B, wl.Hq, wl.d), np.uint16)
    for b in range(wl.B):
        for h in range(wl.Hkv):
            ku, vu, qu = synth.make_unit(wl, rank * wl.B + b, h)
            k[b, h], v[b, h] = ku, vu
            q[b, h * wl.G:(h + 1) * wl.G] = qu
    return k, v, q


# ----------------------------------------------------------------------------- CPU oracle
def cpu_oracle_timing(wl, k, v, q, W, steps_cap=None, target_s=10.0):
    """Times the oracle (as it stands) on the host cores: build every unit once
    (setup, untimed), then decode steps (all units on parallel threads)."""
    import oracle
    from concurrent.futures import ThreadPoolExecutor
    units = [(b, h) for b in range(wl.B) for h in range(wl.Hkv)]
    threads = max(1, min(len(units), os.cpu_count() or 1))
    t0 = time.perf_counter()
    with ThreadPoolExecutor(threads) as ex:
        idx = list(ex.map(lambda bh: oracle.build_unit(k[bh[0], bh[1]], W, wl.K, wl.L, wl.center, wl.mips, wl.sink,
                                                        wl.local), units))
    t_build = time.perf_counter() - t0

    def one_step():
        with ThreadPoolExecutor(threads) as ex:
            list(ex.map(lambda j: oracle.decode_indexed(idx[j], k[units[j][0], units[j][1]],
                                                        v[units[j][0], units[j][1]],
                                                        q[units[j][0], units[j][1] * wl.G:(units[j][1] + 1) * wl.G],
                                                        wl.min_collisions), range(len(units))))

    one_step()  # warm
    times = []
    t_start = time.perf_counter()
    while True:
        t = time.perf_counter()
        one_step()
        times.append(time.perf_counter() - t)
        if (steps_cap and len(times) >= steps_cap) or (not steps_cap and time.perf_counter() - t_start > target_s):
            break
    return {"step_s": statistics.mean(times), "steps": len(times), "threads": threads, "build_s": t_build}


# ----------------------------------------------------------------------------- context sweep
def sweep_point(wl, dev, tW, peak, graph_launches=64, buckets=False):
    """Decode kernel alone (the roofline kernel) at one workload: inputs rotated over R
    replicas so that a launch's bytes were last touched R-1 launches earlier (> L2).
    buckets=True: the bucketed hash-table path (bucket query kernel + decode kernel in bitmap
    mode); its algorithmic bytes replace the code stream by the ids of the query's buckets,
    the bucket offsets and the S bitmaps (written and read)."""
    import torch
    import paper_2410_16179_b200 as pkg
    from paper_2410_16179_b200 import binding as B_

    k, v, q = synth.make_batch(wl, threads=os.cpu_count() or 1)
    bf = lambda a: torch.from_numpy(np.ascontiguousarray(a).view(np.int16)).view(torch.bfloat16).to(dev)
    tk, tv, tq = bf(k), bf(v), bf(q)
    del k, v
    per_rep = wl.B * wl.Hkv * wl.n * (512 + wl.K * wl.L / 8)
    R = int(min(16, max(2, -(-300e6 // per_rep))))
    mps, ks, vs = [], [], []
    for r in range(R):
        kr = tk if r == 0 else tk.clone()
        vr = tv if r == 0 else tv.clone()
        mp = pkg.MagicPIG(tW, K=wl.K, L=wl.L, center=wl.center, mips=wl.mips, min_collisions=wl.min_collisions,
                          sink=wl.sink, local=wl.local, buckets=buckets).build(kr)
        mp.release_build_workspace()
        mps.append(mp), ks.append(kr), vs.append(vr)
    cfg = mps[0].cfg
    n, Bn, Hq, Hkv = wl.n, wl.B, wl.Hq, wl.Hkv
    ws = B_.new_workspace(B_.decode_workspace_bytes(cfg, Bn, Hq, Hkv, n), dev)
    out = torch.empty((Bn, Hq, 128), dtype=torch.float32, device=dev)
    nw = (n + 31) // 32
    smask = torch.zeros((Bn, Hq, nw), dtype=torch.int32, device=dev)
    scount = torch.zeros((Bn, Hq), dtype=torch.int32, device=dev)
    mps[0]._ws_dec = ws
    mps[0].decode(tq, ks[0], vs[0], out=out, s_count=scount, s_mask=smask)
    torch.cuda.synchronize()
    sm = smask.cpu().numpy().view(np.uint32).reshape(Bn, Hkv, wl.G, nw)
    n_union = int(np.unpackbits(np.bitwise_or.reduce(sm, axis=2).view(np.uint8)).sum())
    nT = min(n, wl.sink + wl.local)
    KL = wl.K * wl.L
    alg = (Bn * Hkv * (n - nT) * KL / 8 + (n_union + Bn * Hkv * nT) * 512 + n_union * 4 + Bn * Hq * (256 + KL / 8)
           + Bn * Hkv * 512)

    ids_read = None
    if buckets:
        qc = torch.zeros((Bn, Hq, wl.L), dtype=torch.int16, device=dev)
        B_.query_codes(cfg, tq, tW, qc, ws)
        qc = qc.cpu().numpy().view(np.uint16).astype(np.int64)
        nb = 1 << wl.K
        per = wl.L * (nb + 1 + n)
        tabs = mps[0].buf.tables
        ids_read = 0
        for b in range(Bn):
            for hq in range(Hq):
                u = b * Hkv + hq // wl.G
                offs = tabs[u * per:u * per + wl.L * (nb + 1)].view(wl.L, nb + 1).cpu().numpy()
                c = qc[b, hq]
                ids_read += int((offs[np.arange(wl.L), c + 1] - offs[np.arange(wl.L), c]).sum())
        alg = (alg - Bn * Hkv * (n - nT) * KL / 8 + ids_read * 4 + Bn * Hq * wl.L * 8
               + 2 * Bn * Hq * ((n + 31) // 32) * 4)

    def kern(r):
        if buckets:
            B_.decode_buckets_encoded(cfg, tq, mps[r].buf.tables, mps[r].buf.center, mps[r].buf.key_norm, ks[r],
                                      vs[r], 0, n, ws, out=out)
        else:
            B_.decode_encoded(cfg, tq, mps[r].buf.codes, mps[r].buf.center, mps[r].buf.key_norm, ks[r], vs[r], 0, n,
                              ws, out=out)

    for r in range(R):
        kern(r)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for i in range(graph_launches):
            kern(i % R)
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(5):
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3 / graph_launches)
    us = float(np.median(ts))
    gbs = alg / us / 1e3
    res = {"n": n, "B": Bn, "Hq": Hq, "Hkv": Hkv, "K": wl.K, "L": wl.L, "kernel_us": us, "tokens_per_s": Bn / us * 1e6,
           "alg_MB": alg / 1e6, "GBs": gbs, "frac": gbs / peak, "sampled_fraction": float(scount.float().mean()) /
           max(n - nT, 1), "replicas": R}
    if buckets:
        res.update(buckets=True, ids_read=ids_read, kernels="bucket_mark + decode5 (bitmap mode)")
    del mps, ks, vs, tk, tv
    torch.cuda.empty_cache()
    return res


# ----------------------------------------------------------------------------- ours
def run_ours(args):
    import torch
    import paper_2410_16179_b200 as pkg
    from paper_2410_16179_b200 import binding as B_

    dist, rank, world = _dist()
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    wl = _workload(args.config)
    k, v, q = _make_inputs(wl, rank)
    W = synth.make_projections(wl.K, wl.L, wl.mips)

    def bf(a):
        return torch.from_numpy(np.ascontiguousarray(a).view(np.int16)).view(torch.bfloat16).to(dev)

    tW = torch.from_numpy(W).to(dev)
    tk, tv, tq = bf(k), bf(v), bf(q)
    R = args.replicas
    # replicas (distinct addresses) of everything a step reads
    mps, ks, vs, qs = [], [], [], []
    for r in range(R):
        kr = tk if r == 0 else tk.clone()
        vr = tv if r == 0 else tv.clone()
        mp = pkg.MagicPIG(tW, K=wl.K, L=wl.L, center=wl.center, mips=wl.mips, min_collisions=wl.min_collisions,
                          sink=wl.sink, local=wl.local).build(kr)
        mp.release_build_workspace()
        mps.append(mp)
        ks.append(kr)
        vs.append(vr)
        qs.append(tq.clone())
    torch.cuda.synchronize()
    cfg = mps[0].cfg
    Bn, Hkv, n = wl.B, wl.Hkv, wl.n
    Hq = wl.Hq
    ws = B_.new_workspace(B_.decode_workspace_bytes(cfg, Bn, Hq, Hkv, n), dev)
    outs = [torch.empty((Bn, Hq, 128), dtype=torch.float32, device=dev) for _ in range(R)]

    # ---- algorithmic bytes: codes of D + K/V rows of (union_g S_g) U T + q/qcodes + c
    nw = (n + 31) // 32
    smask = torch.zeros((Bn, Hq, nw), dtype=torch.int32, device=dev)
    scount = torch.zeros((Bn, Hq), dtype=torch.int32, device=dev)
    B_.decode(cfg, qs[0], mps[0].buf.codes, mps[0].buf.center, mps[0].buf.key_norm, ks[0], vs[0], 0, n, tW, ws,
              out=outs[0], s_count=scount, s_mask=smask)
    torch.cuda.synchronize()
    status = B_.workspace_status(ws)
    sm = smask.cpu().numpy().view(np.uint32).reshape(Bn, Hkv, wl.G, nw)
    union = np.bitwise_or.reduce(sm, axis=2)
    n_union = int(sum(int(np.unpackbits(union[b, h].view(np.uint8)).sum()) for b in range(Bn) for h in range(Hkv)))
    nT = min(n, wl.sink + wl.local)
    nD = n - nT
    KL = wl.K * wl.L
    bytes_codes = Bn * Hkv * nD * KL / 8
    bytes_rows = (n_union + Bn * Hkv * nT) * 512 + n_union * 4  # K/V rows + |xbar_i| of sampled keys
    bytes_misc = Bn * Hq * (256 + KL / 8) + Bn * Hkv * 512
    alg_bytes = bytes_codes + bytes_rows + bytes_misc
    sampled_frac = float(scount.float().mean().item()) / max(nD, 1)

    stream = torch.cuda.current_stream()

    def step(r):
        B_.encode_queries(cfg, qs[r], tW, ws)
        B_.decode_encoded(cfg, qs[r], mps[r].buf.codes, mps[r].buf.center, mps[r].buf.key_norm, ks[r], vs[r], 0, n, ws,
                          out=outs[r])

    def kernel_only(r):
        B_.decode_encoded(cfg, qs[r], mps[r].buf.codes, mps[r].buf.center, mps[r].buf.key_norm, ks[r], vs[r], 0, n, ws,
                          out=outs[r])

    def capture(fn, nsteps, offset=0):
        g = torch.cuda.CUDAGraph()
        for i in range(R):  # warm all replicas outside capture
            fn(i)
        torch.cuda.synchronize()
        l0 = B_.launch_count()
        with torch.cuda.graph(g):
            for i in range(nsteps):
                fn((offset + i) % R)
        return g, B_.launch_count() - l0

    GS = min(args.steps, 64)
    g_main, launches_main = capture(step, GS)
    rem = args.steps % GS
    g_rem, launches_rem = capture(step, rem) if rem else (None, 0)
    reps = args.steps // GS
    gpu_launches = reps * launches_main + launches_rem

    # warm-up: >= W steps
    wreps = max(1, -(-args.warmup // GS))
    for _ in range(wreps):
        g_main.replay()
    torch.cuda.synchronize()

    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local_rank) as clk:
        e0.record(stream)
        for _ in range(reps):
            g_main.replay()
        if g_rem is not None:
            g_rem.replay()
        e1.record(stream)
        torch.cuda.synchronize()
        # keep sampling under the same load for a moment if the region was very short
        t_extra = time.perf_counter()
        while time.perf_counter() - t_extra < 0.2:
            g_main.replay()
            torch.cuda.synchronize()
    if dist:
        dist.barrier()
    ms = e0.elapsed_time(e1)
    if dist:
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    ms_step = ms / args.steps
    value = world * Bn / (ms_step / 1e3)

    # ---- dominant kernel alone (decode_encoded: scan + gather + estimator + merge)
    KG = 256
    g_k, _ = capture(kernel_only, KG)
    g_k.replay()
    torch.cuda.synchronize()
    k0, k1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    k0.record(stream)
    g_k.replay()
    k1.record(stream)
    torch.cuda.synchronize()
    kern_ms = k0.elapsed_time(k1) / KG
    peak, peak_src = _peaks()
    achieved = alg_bytes / (kern_ms / 1e3) / 1e9
    tr = _traffic("decode")

    # ---- end to end through the public serving API (pkg.session: one CUDA graph per step holding the
    # H2D copy of q from pinned host memory, encode, decode and the D2H copy of the output)
    sess = [pkg.session(mps[r], ks[r], vs[r], Hq) for r in range(R)]
    for s_ in sess:
        s_.q_host.copy_(torch.from_numpy(q.view(np.int16)).view(torch.bfloat16))
    E = min(args.steps, args.e2e_steps)

    def e2e_step(i):
        sess[i % R].step()

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
    e2e_ms = f0.elapsed_time(f1) / E
    if dist:
        t = torch.tensor([e2e_ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms = float(t.item())
    e2e_value = world * Bn / (e2e_ms / 1e3)

    # correctness guard on the timed paths: the last outputs are finite and the session's host output
    # equals the device-timed path's output for the same inputs
    assert torch.isfinite(outs[0]).all().item(), "non-finite output"
    assert torch.equal(sess[0].out_host, outs[0].cpu()), "session output differs from decode output"

    sweep = None
    if rank == 0 and args.sweep:
        import dataclasses
        sweep = []
        for spec in args.sweep.split(","):
            name, _, rest = spec.partition(":")
            nn, _, ov = rest.partition(":")  # "C2:16384:mips=0+min_collisions=1": variant flags (NEXT-4)
            bk = name.endswith("b")  # "C2b:16384": the bucketed hash-table path
            name = name[:-1] if bk else name
            wl_s = dataclasses.replace(synth.CONFIGS[name], n=int(nn)) if nn else synth.CONFIGS[name]
            over = {kv.split("=")[0]: int(kv.split("=")[1]) for kv in ov.split("+") if kv}
            if over:
                wl_s = dataclasses.replace(wl_s, **over)
            if wl_s == wl and not bk:
                sweep.append({"n": n, "B": Bn, "Hq": Hq, "Hkv": Hkv, "K": wl.K, "L": wl.L, "kernel_us": kern_ms * 1e3,
                              "tokens_per_s": Bn / kern_ms * 1e3, "alg_MB": alg_bytes / 1e6, "GBs": achieved,
                              "frac": achieved / peak, "sampled_fraction": sampled_frac, "replicas": R})
                continue
            tWs = tW if (wl_s.K, wl_s.L, wl_s.mips) == (wl.K, wl.L, wl.mips) else \
                torch.from_numpy(synth.make_projections(wl_s.K, wl_s.L, wl_s.mips)).to(dev)
            pt = sweep_point(wl_s, dev, tWs, peak, buckets=bk)
            pt["config"] = name
            if over:
                pt["variant"] = over
            sweep.append(pt)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        c = cpu_oracle_timing(wl, k, v, q, W, target_s=args.cpu_seconds)
        cpu = {"value": wl.B / c["step_s"], "unit": "tokens/s", "cores": c["threads"], "kind": "oracle",
               "sample": f"full {args.config} decode step (all {wl.B * wl.Hkv} units x {wl.G} heads, oracle codes "
                         f"built once untimed in {c['build_s']:.1f}s), {c['steps']} steps on {c['threads']} threads"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
            "config": {"workload": f"{args.config}: B={Bn} per GPU, Hq={Hq}, Hkv={Hkv}, d=128, n={n}, K={wl.K}, "
                                   f"L={wl.L}, mips={wl.mips}, center={wl.center}, sink={wl.sink}, local={wl.local}",
                       "global_batch": Bn * world, "seq_len": n, "parallelism": f"heads/batch x{world} (no collective)",
                       "l2": f"{R} rotating input replicas", "sampled_fraction": sampled_frac,
                       "union_rows": n_union, "alg_bytes_per_step": alg_bytes, "status": status},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                         "traffic": tr, "kernel": "decode5_kernel (persistent: scan + gather + estimator + unit merge)",
                         "kernel_us": kern_ms * 1e3, "peak_source": peak_src},
            "cpu_baseline": cpu,
            "e2e": {"value": e2e_value, "unit": "tokens/s", "h2d_bytes_per_step": int(tq.numel() * 2),
                    "d2h_bytes_per_step": int(Bn * Hq * 128 * 4), "ms_per_step": e2e_ms},
            "gpu_launches": int(gpu_launches),
            "clocks": clk.summary(),
            "context_sweep": sweep,
        }
        print(json.dumps(line))
    if dist:
        dist.barrier()
        dist.destroy_process_group()


# ----------------------------------------------------------------------------- reference arm
def run_reference(args):
    dist, rank, world = _dist()
    if rank != 0:
        if dist:
            dist.barrier()
        return
    wl = _workload(args.config)
    k, v, q = _make_inputs(wl, 0)
    W = synth.make_projections(wl.K, wl.L, wl.mips)
    steps = max(1, min(args.steps, args.ref_steps_cap))
    c = cpu_oracle_timing(wl, k, v, q, W, steps_cap=steps)
    value = wl.B / c["step_s"]
    sample = (f"full {args.config} decode step per step (all {wl.B * wl.Hkv} units x {wl.G} heads; oracle codes built "
              f"once untimed in {c['build_s']:.1f}s); {c['steps']} timed steps (cap {args.ref_steps_cap})")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": world,
        "steps": c["steps"], "warmup": args.warmup, "ms_per_step": c["step_s"] * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"{args.config} (CPU oracle, double precision)", "global_batch": wl.B,
                   "seq_len": wl.n},
        "cpu_baseline": {"value": value, "unit": "tokens/s", "cores": c["threads"], "kind": "oracle",
                         "sample": sample},
        "e2e": {"value": value, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))
    if dist:
        dist.barrier()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=2000)
    ap.add_argument("--warmup", type=int, default=64)
    ap.add_argument("--config", default="C2", choices=sorted(synth.CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--replicas", type=int, default=8)
    ap.add_argument("--e2e-steps", type=int, default=500)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--ref-steps-cap", type=int, default=200)
    ap.add_argument("--sweep", default="C2:4096,C2:16384,C2:65536,C2:131072,C2b:16384,C2b:131072",
                    help="decode-kernel roofline vs context length: comma list of CONFIG[:n] ('' = off)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
