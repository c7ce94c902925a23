#!/usr/bin/env python
"""bench.py — RBRP time-to-ID on B200 (BASELINE.json metric), one JSON line.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...      (rows sharded over N GPUs)

A step is one complete RBRP interpolative decomposition (Alg. 2 selection to the
tolerance + Alg. 3 W) of the config's synthetic X, already resident in HBM.  At N = 1
the workload is BASELINE.json configs[1] (c2: fp64 65536 x 1024, exactly rank-128 +
1e-8 noise, b = 32, tau = 1e-12) — the metric's configuration; configs[0] (c1) is the
oracle-sized parity case.  N > 1: the same problem with its rows sharded over the ranks
(strong scaling; NCCL exchange points).  Timing: W warm-up steps, then K
steps between barrier + synchronize, CUDA events on the stream the library launches on,
max over ranks.  X (537 MB) and the residual are larger than the 126 MB L2, so no
explicit flush is needed.

Also reported: the roofline of the dominant projection pass (Alg. 2 l.13/l.16), timed
live inside the timed region by %globaltimer stamps in the kernels (the block loop runs
as one CUDA graph, whose body admits no event nodes); the end-to-end figure through the
public API with host buffers (pinned X -> HBM and W -> pinned host inside the timed
region); the kernel-launch count; the SM clocks seen by nvidia-smi during the timed
region; the CPU oracle timed on this host (N = 1, rank 0).
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = ("RBRP time-to-(r,ε)-ID (s) and projection-pass HBM GB/s / roofline fraction, "
          "1–8 GPU")
FP64_PEAK_TFLOPS = 148 * 64 * 2 * 1.965e9 / 1e12   # FP64 units x max clock
HBM_GBS = 6551.4                                     # MEASURED_PEAKS.json hbm_gbs


def _args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c2")
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--form", default="residual", choices=["residual", "paper"],
                    help="residual: north_star hot path (default); paper: Alg. 2 literally (NEXT-1)")
    ap.add_argument("--no-alt-form", action="store_true", help="skip the side measurement of the other form")
    ap.add_argument("--no-sketch", action="store_true", help="skip the SkLUPP-OSID side measurement (NEXT-4)")
    return ap.parse_args()


class Clocks:
    """nvidia-smi sampler (SM clock + throttle reasons) around the timed region."""
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None
        self.t0 = self.t1 = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.th = threading.Thread(target=self._read, daemon=True)
            self.th.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append((time.time(), line.strip()))

    def stop(self):
        if self.proc:
            time.sleep(0.12)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        import statistics
        sel = [r for (t, r) in self.rows if self.t0 - 0.06 <= t <= self.t1 + 0.06] or \
              [r for (_, r) in self.rows]
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in sel:
            f = [x.strip() for x in r.split(",")]
            if len(f) < 6:
                continue
            try:
                sm.append(float(f[0]))
                mx = float(f[1])
            except ValueError:
                continue
            for nm, v in zip(names, f[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


def _tau(cfg, X, world=1):
    """tau for the config: given, or (1+eps) eta_r with eta_r from the Gram
    eigenvalues (harness code, untimed; R3).  Sharded: the Gram is summed
    over the ranks."""
    import torch
    if cfg.tau is not None:
        return cfg.tau
    G = X.double().T @ X.double()
    if world > 1:
        import torch.distributed as dist
        dist.all_reduce(G)
    ev = torch.linalg.eigvalsh(G).flip(0).clamp_min(0)
    return float((1 + cfg.eps) * ev[cfg.r:].sum() / ev.sum())


def _proj_roofline(cfg, res_list, proj_ms, n_local, form="residual"):
    """Algorithmic flops/bytes of the projection pass, per block:
    residual form: flops = 4 n d b' + 2 n d, bytes = 2 n d w + n b' w + 8 n;
    paper form (NEXT-1, read-only pass): flops = 2 n d b' + 2 n b',
    bytes = n d w + n b' w + 16 n (n = this rank's rows)."""
    n, d = n_local, cfg.d
    w = 8 if cfg.dtype == "f64" else 4
    flops = bytes_ = 0.0
    for res in res_list:
        for bp in res.b_prime:
            if form == "paper":
                flops += 2.0 * n * d * bp + 2.0 * n * bp
                bytes_ += n * d * w + n * bp * w + 16.0 * n
            else:
                flops += 4.0 * n * d * bp + 2.0 * n * d
                bytes_ += 2.0 * n * d * w + n * bp * w + 8.0 * n
    t = proj_ms / 1e3
    return flops / t / 1e12, bytes_ / t / 1e9, flops, bytes_


def _dominant_kernel(cfg, res_list, n_local, form="residual"):
    """Roofline of the DOMINANT projection kernel: the bucket instantiation (b' <= 16, 32,
    64, 128 -> one kernel template each) with the most device time.  Per launch: the
    algorithmic flops/bytes of _proj_roofline, divided by that launch's in-kernel stamp
    time.  Also the mixed-bound fraction over all blocks: sum of per-block roofline floors
    max(flops/F64 peak, bytes/HBM peak) over the summed block times."""
    n, d = n_local, cfg.d
    w = 8 if cfg.dtype == "f64" else 4
    peak = FP64_PEAK_TFLOPS if cfg.dtype == "f64" else FP64_PEAK_TFLOPS * 2
    per = {}
    floor_s = time_s = 0.0
    for res in res_list:
        for bp, ms in zip(res.b_prime, res.proj_ms_blk):
            if bp <= 0 or ms <= 0:
                continue
            bk = 16 if bp <= 16 else 32 if bp <= 32 else 64 if bp <= 64 else 128
            if form == "paper":
                fl, by = 2.0 * n * d * bp + 2.0 * n * bp, n * d * w + n * bp * w + 16.0 * n
            else:
                fl, by = 4.0 * n * d * bp + 2.0 * n * d, 2.0 * n * d * w + n * bp * w + 8.0 * n
            e = per.setdefault(bk, [0.0, 0.0, 0.0, 0])
            e[0] += fl
            e[1] += by
            e[2] += ms / 1e3
            e[3] += 1
            floor_s += max(fl / (peak * 1e12), by / (HBM_GBS * 1e9))
            time_s += ms / 1e3
    if not per:
        return None
    bk, (fl, by, t, cnt) = max(per.items(), key=lambda kv: kv[1][2])
    return {"bucket": bk, "launches": cnt, "avg_launch_ms": t / cnt * 1e3,
            "achieved_tflops": fl / t / 1e12, "frac_fp64": fl / t / 1e12 / peak,
            "achieved_GBs": by / t / 1e9, "frac_hbm": by / t / 1e9 / HBM_GBS,
            "algorithmic_flops_per_launch": fl / cnt, "algorithmic_bytes_per_launch": by / cnt,
            "mixed_bound_frac_all_blocks": floor_s / time_s if time_s > 0 else None}


def _traffic_from_profile(cfg_name):
    """dram bytes per block of the projection kernels from the committed ncu capture."""
    p = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(p):
        try:
            return json.load(open(p)).get(cfg_name, {}).get("proj_dram_bytes_per_block")
        except Exception:
            return None
    return None


def _workload(cfg, tau):
    desc = {"c2": " exactly rank-128 + 1e-8 noise,"}.get(cfg.name, "")
    return f"{cfg.name}: {cfg.dtype} n={cfg.n} d={cfg.d}{desc} b={cfg.b}, tau={tau:.3g}"


def _threads():
    try:
        from threadpoolctl import threadpool_info
        return int(max([i.get("num_threads", 1) for i in threadpool_info()] or [1]))
    except Exception:
        return os.cpu_count()


def _cpu_baseline(cfg, Xnp, tau):
    from oracle import rbrp as O
    t = time.perf_counter()
    ores = O.rbrp(Xnp, tau=tau, b=cfg.b, seed=0)
    O.form_W(ores.L, ores.S, method="trsm")
    dt = time.perf_counter() - t
    return {"value": dt, "unit": "s", "cores": _threads(), "kind": "oracle",
            "sample": f"one full {cfg.name} ID ({cfg.n}x{cfg.d} {cfg.dtype}, b={cfg.b}, k={ores.k}) "
                      f"incl. W, NumPy/BLAS, {len(os.sched_getaffinity(0))} host cores visible"}


def run_reference(a):
    """The reference arm: the CPU oracle (as it stands) on the same workload; rank 0 only."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import numpy as np

    from oracle import rbrp as O
    from workloads import CONFIGS, make
    cfg = CONFIGS[a.config]
    X = make(cfg)
    Xnp = X.numpy()
    tau = _tau(cfg, X)
    for _ in range(a.warmup):
        O.rbrp(Xnp, tau=tau, b=cfg.b, seed=a.seed)
    times = []
    r = None
    for _ in range(a.steps):
        t = time.perf_counter()
        r = O.rbrp(Xnp, tau=tau, b=cfg.b, seed=a.seed)
        O.form_W(r.L, r.S, method="trsm")
        times.append(time.perf_counter() - t)
    v = float(np.mean(times))
    line = {"metric": METRIC, "value": v, "unit": "s", "n_gpus": a.gpus, "steps": a.steps,
            "warmup": a.warmup, "ms_per_step": v * 1e3, "higher_is_better": False,
            "scaling": "weak", "vs_baseline": None, "dtype": cfg.dtype,
            "data": "synthetic", "impl": "reference",
            "config": {"workload": _workload(cfg, tau),
                       "n": cfg.n, "d": cfg.d, "b": cfg.b, "k": r.k},
            "cpu_baseline": {"value": v, "unit": "s", "cores": _threads(), "kind": "oracle",
                             "sample": f"one full {cfg.name} ID per step (CPU oracle as it stands)"},
            "e2e": {"value": v, "unit": "s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    a = _args()
    if a.impl == "reference":
        return run_reference(a)
    import torch
    import torch.distributed as dist

    import paper_2309_16002_b200 as rb
    from paper_2309_16002_b200 import dist as rdist
    from workloads import CONFIGS, make

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)

    def barrier():
        if world > 1:
            dist.barrier()

    cfg = CONFIGS[a.config]
    # rows of X sharded over the ranks (contiguous, 4096-row aligned); every rank holds
    # only its shard; N = 1 is the single-GPU path (CUDA-graph loop)
    r0, n_local = rdist.partition_rows(cfg.n, world, rank)
    X = make(cfg, device=dev, row_offset=r0, n_local=n_local)
    tau = _tau(cfg, X, world)
    comm = rdist.Comm(dev) if world > 1 else None
    dkw = dict(n_global=cfg.n, row_offset=r0, comm=comm.handle) if comm else {}
    ws = torch.empty(rb.workspace_size(X, tol=tau, b=cfg.b, n_global=cfg.n, row_offset=r0),
                     dtype=torch.uint8, device=dev)
    k_cap = min(cfg.n, cfg.d)
    Wbuf = torch.empty((n_local, k_cap), dtype=cfg.torch_dtype, device=dev)
    kw = dict(tol=tau, b=cfg.b, seed=a.seed, workspace=ws, log_blocks=False, W_out=Wbuf, form=a.form, **dkw)
    for _ in range(a.warmup):
        rb.id(X, **kw)
    torch.cuda.synchronize()

    clk = Clocks(local)
    clk.start()
    time.sleep(0.3)
    res_list = []
    stream = torch.cuda.current_stream(dev)
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    barrier()
    torch.cuda.synchronize()
    clk.t0 = time.time()
    e0.record(stream)
    for _ in range(a.steps):
        r = rb.id(X, **kw)
        r.W = None
        res_list.append(r)
    e1.record(stream)
    torch.cuda.synchronize()
    barrier()
    clk.t1 = time.time()
    clk.stop()
    ms = e0.elapsed_time(e1) / a.steps
    if world > 1:
        ms = rdist.max_over_ranks(ms, device=dev)

    # projection-pass device time inside the timed region (in-kernel %globaltimer stamps,
    # first CTA start of L-hat -> last CTA end of the fused update, summed over blocks)
    proj_ms = sum(r.proj_ms for r in res_list)
    tflops, gbs, flops, bytes_ = _proj_roofline(cfg, res_list, proj_ms, n_local, a.form)
    dom = _dominant_kernel(cfg, res_list, n_local, a.form)
    launches = sum(r.launches for r in res_list)
    r0res = res_list[-1]
    # per-phase breakdown from one eager, event-instrumented run (outside the timed region)
    rp = rb.id(X, profile=True, **kw)
    torch.cuda.synchronize()

    e2e = None
    if not a.no_e2e:
        # end to end through the public API with HOST buffers: every step copies X
        # (pinned host -> HBM) and reads W (n x k) back to pinned host memory
        Xh = X.cpu().pin_memory()
        Xd = torch.empty_like(X)
        Wh = torch.empty((n_local, k_cap), dtype=cfg.torch_dtype, pin_memory=True)
        w = 8 if cfg.dtype == "f64" else 4
        rb.id_host(Xh, X_dev=Xd, W_host=Wh, **kw)
        torch.cuda.synchronize()
        barrier()
        f0 = torch.cuda.Event(enable_timing=True)
        f1 = torch.cuda.Event(enable_timing=True)
        f0.record(stream)
        ks = 0
        for _ in range(a.steps):
            rr, _W = rb.id_host(Xh, X_dev=Xd, W_host=Wh, **kw)
            ks = rr.k
        f1.record(stream)
        torch.cuda.synchronize()
        te = f0.elapsed_time(f1) / a.steps
        if world > 1:
            te = rdist.max_over_ranks(te, device=dev)
        e2e = {"value": te / 1e3, "unit": "s", "h2d_bytes_per_step": cfg.n * cfg.d * w,
               "d2h_bytes_per_step": cfg.n * ks * w + ks * 8,
               "note": "per step: X pinned host -> HBM (each rank its shard), ID, W -> pinned host"}

    alt = None
    if not a.no_alt_form:
        # side measurement of the other form of Alg. 2 on the same input (not the headline)
        other = "paper" if a.form == "residual" else "residual"
        kw2 = dict(kw, form=other)
        for _ in range(2):
            rb.id(X, **kw2)
        torch.cuda.synchronize()
        barrier()
        g0 = torch.cuda.Event(enable_timing=True)
        g1 = torch.cuda.Event(enable_timing=True)
        ns = max(1, min(a.steps, 10))
        rl2 = []
        g0.record(stream)
        for _ in range(ns):
            r2 = rb.id(X, **kw2)
            r2.W = None
            rl2.append(r2)
        g1.record(stream)
        torch.cuda.synchronize()
        t2 = g0.elapsed_time(g1) / ns
        if world > 1:
            t2 = rdist.max_over_ranks(t2, device=dev)
        pm2 = sum(r.proj_ms for r in rl2)
        tf2, gb2, _, _ = _proj_roofline(cfg, rl2, pm2, n_local, other)
        alt = {"form": other, "value": t2 / 1e3, "unit": "s", "steps": ns, "k": rl2[-1].k,
               "b_prime": rl2[-1].b_prime, "resid_rel": rl2[-1].resid_rel,
               "proj_tflops": tf2, "proj_frac_fp64": tf2 / FP64_PEAK_TFLOPS,
               "proj_hbm_GBs": gb2, "proj_share": pm2 / ns / t2,
               "note": ("paper: Alg. 2 literally (X read only, CGS2 l.6, downdated norms l.16; "
                        "SURVEY NEXT-1)" if other == "paper" else "residual: north_star form")}

    sk = None
    if not a.no_sketch and world == 1 and cfg.dtype == "f64" and cfg.d % 8 == 0:
        # side measurement of SkLUPP-OSID at the ID's rank, l = 3k
        from paper_2309_16002_b200 import sketch as rbs
        ksk = min(res_list[-1].k, rbs.SK_MAX_K)
        sk_ws = torch.empty(rbs.sketch_workspace_size(X.shape[0], X.shape[1], ksk, 3 * ksk), dtype=torch.uint8,
                            device=dev)
        sk_W = torch.empty((X.shape[0], ksk), dtype=torch.float64, device=dev)
        kws = dict(k=ksk, l=3 * ksk, seed=a.seed, workspace=sk_ws, W_out=sk_W)
        for _ in range(2):
            rbs.sketch_id(X, **kws)
        torch.cuda.synchronize()
        g0 = torch.cuda.Event(enable_timing=True)
        g1 = torch.cuda.Event(enable_timing=True)
        ns = max(1, min(a.steps, 10))
        g0.record(stream)
        for _ in range(ns):
            rs = rbs.sketch_id(X, **kws)
        g1.record(stream)
        torch.cuda.synchronize()
        ts = g0.elapsed_time(g1) / ns
        ph = rbs.sketch_id(X, profile=True, **kws).ms_phase
        lp = (3 * ksk + 7) // 8 * 8
        sk = {"method": "SkLUPP-OSID (Alg. 4, l = 3k)", "value": ts / 1e3, "unit": "s", "steps": ns, "k": rs.k,
              "l": 3 * ksk, "ms_phase": ph, "launches": rs.launches,
              "sketch_gemm_tflops": 2 * cfg.n * cfg.d * lp / (ph["sketch"] * 1e9),
              "note": "SURVEY NEXT-4 (the paper's GPU competitor, Table 3 P:783); not the headline"}

    if rank != 0:
        if comm:
            comm.close()
        if world > 1:
            dist.destroy_process_group()
        return
    cpu = None
    if world == 1 and not a.no_cpu_baseline:
        cpu = _cpu_baseline(cfg, X.cpu().numpy(), tau)
    peak = FP64_PEAK_TFLOPS if cfg.dtype == "f64" else FP64_PEAK_TFLOPS * 2
    nblk = sum(len(r.b_prime) for r in res_list)
    traffic = _traffic_from_profile(cfg.name)
    line = {
        "metric": METRIC, "value": ms / 1e3, "unit": "s", "n_gpus": world, "steps": a.steps,
        "warmup": a.warmup, "ms_per_step": ms, "higher_is_better": False,
        "scaling": "strong" if world > 1 else "weak", "vs_baseline": None,
        "dtype": cfg.dtype, "data": "synthetic",
        "config": {"workload": _workload(cfg, tau),
                   "n": cfg.n, "d": cfg.d, "b": cfg.b, "tau": tau, "k": r0res.k, "blocks": r0res.nblocks,
                   "b_prime": r0res.b_prime, "resid_rel": r0res.resid_rel,
                   "parallelism": "single" if world == 1 else f"rows{world} (NCCL row sharding)",
                   "rows_per_rank": n_local, "graph_loop": r0res.graph,
                   "l2": "inputs larger than L2 (X 537 MB + residual 537 MB vs 126 MB L2); no flush"},
        "roofline": {"kernel": ("projection pass a4, dominant kernel: the b' <= %d instantiation "
                                "(%d launches; residual form: L-hat pass + update pass per 64-row tile, "
                                "Alg. 2 l.13/l.16)" % (dom["bucket"], dom["launches"])) if dom else "projection pass a4",
                     "bound": "tensor", "achieved": dom["achieved_tflops"] if dom else tflops, "peak": peak,
                     "unit": "TFLOP/s", "frac": (dom["frac_fp64"] if dom else tflops / peak), "traffic": traffic,
                     "timing": "in-kernel %globaltimer stamps per launch (first CTA start -> last CTA end), "
                               "K timed steps",
                     "peak_note": "FP64 tensor path (DMMA, mma.sync.m8n8k4.f64; tcgen05 has no f64 kind): "
                                  "measured 37.15 TF (profiles/r01_peak_fp64.json) = 148 SM x 64 FMA/clk x 2 x "
                                  "1.965 GHz (37.2, used); MEASURED_PEAKS.json has no FP64 entry and the guide no "
                                  "FP64 nominal ratio to scale its bf16 peak (DESIGN.md §6)",
                     "dominant": dom,
                     "all_blocks": {"achieved_tflops": tflops, "frac_fp64": tflops / peak,
                                    "algorithmic_GBs": gbs, "hbm_frac_of_measured": gbs / HBM_GBS,
                                    "mixed_bound_frac": dom["mixed_bound_frac_all_blocks"] if dom else None,
                                    "note": "every block incl. the HBM-bound small-b' tail block; mixed_bound_frac "
                                            "= sum of per-block max(flops/F64 peak, bytes/HBM peak) / sum of times"},
                     "algorithmic_flops_per_block": flops / max(nblk, 1),
                     "algorithmic_bytes_per_block": bytes_ / max(nblk, 1),
                     "share_of_step": proj_ms / a.steps / ms},
        "phase_ms_eager_profile": {k: v for k, v in rp.ms_phase.items() if k != "unused"},
        "gpu_launches": launches,
        "alt_form": alt,
        "next4_sklupp_osid": sk,
        "e2e": e2e,
        "cpu_baseline": cpu,
        "clocks": clk.summary(),
    }
    print(json.dumps(line), flush=True)
    if comm:
        comm.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
