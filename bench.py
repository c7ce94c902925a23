#!/usr/bin/env python
"""bench.py — RBRP time-to-(r,ε)-ID on B200 (BASELINE.json metric), one JSON line.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c5] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...      (rows sharded over N GPUs)

A step is one complete RBRP interpolative decomposition (Alg. 2 selection to the
tolerance + Alg. 3 W) of the config's synthetic X, already resident in HBM.  The headline
workload is c5 (BASELINE.json configs[4]): fp64 4194304 x 1024 Gaussian mixture, b = 128,
(r, eps) = (256, 0.1), i.e. tau = 1.1 eta_256 (eta from the Gram spectrum,
harness code, untimed), k_max = 768 -- the largest (r, eps) configuration that fits one
B200 (X 34 GB + residual 34 GB + L 26 GB + W 26 GB).  N > 1: the same problem with its
rows sharded over the ranks (strong scaling; NCCL exchange points).
At N = 1 the other full-size configs are measured after the headline and reported
under "configs" (c4 fp32, c3 adversarial, c2 exact rank), each with its own roofline.

Timing: W warm-up steps, then K steps between barrier + synchronize, CUDA events on the
stream the library launches on, max over ranks.  Every X is larger than the 126 MB L2
(c2/c3: 537 MB; c4: 8.6 GB; c5: 34 GB), so no flush is needed.

Roofline: the dominant projection kernel (Alg. 2 l.13/l.16), timed live
inside the timed region by %globaltimer stamps in the kernels (the block loop runs as one
CUDA graph, whose body admits no event nodes).  Its bound is the larger of the two floors
of the block's algorithmic work: flops / compute peak (FP64 DMMA for fp64 data) and bytes /
HBM peak (MEASURED_PEAKS.json).  Also: the end-to-end figure through the C ABI with host
buffers (rbrp_id_host: pinned X -> HBM and W -> pinned host inside the timed region); the
kernel-launch count; the SM clocks seen by nvidia-smi during the timed region; the CPU
oracle on a bounded sample of the workload (rank 0, N = 1).
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
# FP64 peak: 148 SM x 64 FP64 FMA/clk x 2 x 1.965 GHz; measured DMMA 37.15 TF
# (profiles/r01_peak_fp64.json).  MEASURED_PEAKS.json carries HBM and bf16 only.
FP64_PEAK_TFLOPS = 148 * 64 * 2 * 1.965e9 / 1e12
K_MAX = {"c5": 768}            # L / W capacity (memory), SURVEY §8(d)
EXTRA = ("c4", "c3", "c2")     # per-config measurements after the headline (N = 1)


def _peaks():
    """HBM / bf16 peaks measured on this pool (driver-written MEASURED_PEAKS.json), else the
    profiling guide's fallback."""
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        m = json.load(open(p))
        return {"hbm_gbs": float(m["hbm_gbs"]), "bf16_tflops": float(m["bf16_tflops"]),
                "bf16_tflops_sustained": float(m.get("bf16_tflops_sustained", m["bf16_tflops"])),
                "source": "measured (MEASURED_PEAKS.json)"}
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0,
                "source": "fallback (B200_PROFILING.md)"}


PEAKS = _peaks()


def _args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c5")
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-extra", action="store_true", help="skip the per-config measurements (c4, c3, c2)")
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


def _tau(cfg, X, world=1, chunk=1 << 18):
    """tau for the config: given, or (1+eps) eta_r with eta_r from the eigenvalues of the
    fp64 Gram matrix X^T X (Eq. 1.3; harness code, untimed; R3).  Accumulated in
    row chunks (X itself may be 34 GB); sharded: summed over the ranks."""
    import torch
    if cfg.tau is not None:
        return cfg.tau
    G = torch.zeros((cfg.d, cfg.d), dtype=torch.float64, device=X.device)
    for a in range(0, X.shape[0], chunk):
        Xc = X[a:a + chunk].double()
        G += Xc.T @ Xc
    if world > 1:
        import torch.distributed as dist
        dist.all_reduce(G)
    ev = torch.linalg.eigvalsh(G).flip(0).clamp_min(0)
    return float((1 + cfg.eps) * ev[cfg.r:].sum() / ev.sum())


def _block_work(cfg, n, bp, form):
    """Algorithmic flops / bytes of one block's projection pass:
    residual form: flops = 4 n d b' + 2 n d, bytes = 2 n d w + n b' w + 8 n;
    paper form (NEXT-1, read-only pass): flops = 2 n d b' + 2 n b', bytes = n d w + n b' w + 16 n."""
    d = cfg.d
    w = 8 if cfg.dtype == "f64" else 4
    if form == "paper":
        return 2.0 * n * d * bp + 2.0 * n * bp, n * d * w + n * bp * w + 16.0 * n
    return 4.0 * n * d * bp + 2.0 * n * d, 2.0 * n * d * w + n * bp * w + 8.0 * n


def _compute_peak(cfg):
    """(TFLOP/s, label) of the arithmetic the projection kernel of this dtype runs on."""
    if cfg.dtype == "f64":
        return FP64_PEAK_TFLOPS, "FP64 tensor path (DMMA): 148 SM x 64 FMA/clk x 2 x 1.965 GHz (measured 37.15)"
    # fp32 data: 3xTF32 on the tcgen05 tensor cores (3 TF32 products per fp32 product):
    # measured bf16 burst x 1/2 (TF32 : BF16 nominal ratio 1.1 : 2.25) / 3
    return PEAKS["bf16_tflops"] / 2 / 3, "3xTF32 on tcgen05: measured bf16 / 2 (TF32 ratio) / 3 products"


def _roofline(cfg, res_list, n_local, form):
    """Dominant projection kernel: the bucket instantiation (b' <= 16, 32, 64, 128) with the
    most device time; per launch = per block (a block's projection launches between the
    in-kernel stamps: first CTA start -> last CTA end).  achieved = algorithmic work per
    launch / average launch time, in the unit of the larger floor (HBM bytes or FLOPs)."""
    pk, _ = _compute_peak(cfg)
    per = {}
    floor_s = time_s = 0.0
    for res in res_list:
        for bp, ms in zip(res.b_prime, res.proj_ms_blk):
            if bp <= 0 or ms <= 0:
                continue
            bk = 16 if bp <= 16 else 32 if bp <= 32 else 64 if bp <= 64 else 128
            fl, by = _block_work(cfg, n_local, bp, form)
            e = per.setdefault(bk, [0.0, 0.0, 0.0, 0])
            e[0] += fl
            e[1] += by
            e[2] += ms / 1e3
            e[3] += 1
            floor_s += max(fl / (pk * 1e12), by / (PEAKS["hbm_gbs"] * 1e9))
            time_s += ms / 1e3
    if not per:
        return None
    bk, (fl, by, t, cnt) = max(per.items(), key=lambda kv: kv[1][2])
    t_cmp, t_hbm = fl / (pk * 1e12), by / (PEAKS["hbm_gbs"] * 1e9)
    hbm_bound = t_hbm >= t_cmp
    ach_tf, ach_gb = fl / t / 1e12, by / t / 1e9
    return {"bucket": bk, "launches": cnt, "avg_launch_ms": t / cnt * 1e3,
            "bound": "hbm" if hbm_bound else "tensor",
            "achieved": ach_gb if hbm_bound else ach_tf,
            "peak": PEAKS["hbm_gbs"] if hbm_bound else pk,
            "unit": "GB/s" if hbm_bound else "TFLOP/s",
            "frac": (ach_gb / PEAKS["hbm_gbs"]) if hbm_bound else (ach_tf / pk),
            "achieved_tflops": ach_tf, "frac_compute": ach_tf / pk,
            "achieved_GBs": ach_gb, "frac_hbm": ach_gb / PEAKS["hbm_gbs"],
            "algorithmic_flops_per_launch": fl / cnt, "algorithmic_bytes_per_launch": by / cnt,
            "mixed_bound_frac_all_blocks": floor_s / time_s if time_s > 0 else None}


def _traffic_from_profile(cfg_name):
    """dram bytes per block of the dominant projection kernel from the committed ncu capture
    (profiles/traffic.json), or None."""
    p = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(p):
        try:
            return json.load(open(p)).get(cfg_name, {}).get("proj_dram_bytes_per_block")
        except Exception:
            return None
    return None


def _workload(cfg, tau, k_max):
    desc = {"c2": " exactly rank-128 + 1e-8 noise,", "c3": " 100 heavy dirs x500 duplicates,",
            "c4": " sigma_i = i^-1.5,", "c5": " GMM 256 centres + 0.05 N(0,I),"}.get(cfg.name, "")
    rr = f" (r,eps)=({cfg.r},{cfg.eps}) ->" if cfg.r else ""
    km = f", k_max={k_max}" if k_max else ""
    return f"{cfg.name}: {cfg.dtype} n={cfg.n} d={cfg.d}{desc} b={cfg.b},{rr} tau={tau:.4g}{km}"


def _threads():
    try:
        from threadpoolctl import threadpool_info
        return int(max([i.get("num_threads", 1) for i in threadpool_info()] or [1]))
    except Exception:
        return os.cpu_count()


def _oracle_sample(cfg, n_sample):
    """The bounded CPU sample of a workload: its first n_sample rows (same generator), with
    the sample's own tau (same (r, eps) or tau rule).  Returns (Xnp, tau)."""
    import numpy as np

    from oracle import referee as R
    from workloads import make
    n_s = min(cfg.n, n_sample)
    Xnp = make(cfg, n_local=n_s).numpy()
    if cfg.tau is not None:
        tau = cfg.tau
    else:
        tau = (1 + cfg.eps) * R.eta(np.asarray(Xnp, dtype=np.float64), cfg.r)
    return Xnp, tau, n_s


ORACLE_SAMPLE_ROWS = {"c5": 16384, "c4": 16384, "c3": 131072, "c2": 65536, "c1": 2000, "t3": 100000}


def _cpu_oracle_run(cfg, Xnp, tau, seed):
    from oracle import rbrp as O
    t = time.perf_counter()
    ores = O.rbrp(Xnp, tau=tau, b=cfg.b, seed=seed, k_max=K_MAX.get(cfg.name))
    O.form_W(ores.L, ores.S, method="trsm")
    return time.perf_counter() - t, ores.k


def _cpu_baseline(cfg, seed=0):
    Xnp, tau, n_s = _oracle_sample(cfg, ORACLE_SAMPLE_ROWS.get(cfg.name, 65536))
    dt, k = _cpu_oracle_run(cfg, Xnp, tau, seed)
    scale = cfg.n / n_s
    return {"value": dt * scale, "unit": "s", "cores": _threads(), "kind": "oracle",
            "sample": (f"one {cfg.name} ID of the first {n_s} of {cfg.n} rows ({cfg.dtype}, b={cfg.b}, k={k}) incl. W, "
                       f"NumPy/BLAS, {len(os.sched_getaffinity(0))} host cores visible: {dt:.3f} s measured, x {scale:g} "
                       f"(cost linear in n at fixed k) = the value"),
            "measured_s": dt, "rows": n_s, "scale": scale}


def run_reference(a):
    """The reference arm: the CPU oracle (as it stands) on a bounded sample of the same
    workload per step (the first rows of the config, extrapolated linearly in n to the
    full config, stated in cpu_baseline.sample); rank 0 only."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import numpy as np

    from workloads import CONFIGS
    cfg = CONFIGS[a.config]
    Xnp, tau, n_s = _oracle_sample(cfg, ORACLE_SAMPLE_ROWS.get(cfg.name, 65536))
    for _ in range(a.warmup):
        _cpu_oracle_run(cfg, Xnp, tau, a.seed)
    times, k = [], 0
    for _ in range(a.steps):
        dt, k = _cpu_oracle_run(cfg, Xnp, tau, a.seed)
        times.append(dt)
    scale = cfg.n / n_s
    v = float(np.mean(times)) * scale
    line = {"metric": METRIC, "value": v, "unit": "s", "n_gpus": a.gpus, "steps": a.steps,
            "warmup": a.warmup, "ms_per_step": v * 1e3, "higher_is_better": False,
            "scaling": "weak", "vs_baseline": None, "dtype": cfg.dtype,
            "data": "synthetic", "impl": "reference",
            "config": {"workload": _workload(cfg, tau, K_MAX.get(cfg.name)), "n": cfg.n, "d": cfg.d, "b": cfg.b,
                       "k_sample": k, "sample_rows": n_s},
            "cpu_baseline": {"value": v, "unit": "s", "cores": _threads(), "kind": "oracle",
                             "sample": (f"per step one {cfg.name} ID of the first {n_s} of {cfg.n} rows "
                                        f"({float(np.mean(times)):.3f} s measured), x {scale:g} (linear in n)")},
            "e2e": {"value": v, "unit": "s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def _measure(rb, cfg, X, tau, k_max, n_local, steps, warmup, form, seed, dev, dkw, barrier, world, clk=None):
    """Time `steps` IDs (after `warmup`) on resident X; returns (ms per ID, results)."""
    import torch

    from paper_2309_16002_b200 import dist as rdist
    ws = torch.empty(rb.workspace_size(X, tol=tau, b=cfg.b, k_max=k_max or 0, n_global=cfg.n,
                                       row_offset=dkw.get("row_offset", 0)), dtype=torch.uint8, device=dev)
    k_cap = k_max or min(cfg.n, cfg.d)
    Wbuf = torch.empty((n_local, k_cap), dtype=cfg.torch_dtype, device=dev)
    kw = dict(tol=tau, b=cfg.b, seed=seed, k_max=k_max or 0, workspace=ws, log_blocks=False, W_out=Wbuf,
              form=form, **dkw)
    for _ in range(warmup):
        rb.id(X, **kw)
    torch.cuda.synchronize()
    if clk:
        clk.start()
        time.sleep(0.3)
    stream = torch.cuda.current_stream(dev)
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    res_list = []
    barrier()
    torch.cuda.synchronize()
    if clk:
        clk.t0 = time.time()
    e0.record(stream)
    for _ in range(steps):
        r = rb.id(X, **kw)
        r.W = None
        res_list.append(r)
    e1.record(stream)
    torch.cuda.synchronize()
    barrier()
    if clk:
        clk.t1 = time.time()
        clk.stop()
    ms = e0.elapsed_time(e1) / steps
    if world > 1:
        ms = rdist.max_over_ranks(ms, device=dev)
    return ms, res_list, kw


def _kernel_label(cfg, bucket, form):
    """Which kernel(s) run a block of the dominant bucket (R28)."""
    what = "projection pass a4 (Alg. 2 l.13/l.16)" if form == "residual" else "read-only L-hat pass (l.13, l.16 downdate)"
    if cfg.dtype == "f32" and form == "residual":
        k = ("k_proj_tc32 (tcgen05 3xTF32), b' <= 64" if bucket <= 64
             else "k_proj_tc32 (tcgen05 3xTF32) in 64-column parts, b' > 64")
    else:
        k = {16: "k_lhat_paper<16> (FP64 DMMA), b' <= 16", 32: "k_lhat_paper<32> (FP64 DMMA), 16 < b' <= 32",
             64: "k_lhat64 (FP64 DMMA), 32 < b' <= 64"}.get(
            bucket, "k_lhat64 on a 64-column part + the remainder on its own kernel (FP64 DMMA), b' > 64")
    return f"{what}: {k}"


def _config_entry(cfg, tau, k_max, ms, res_list, n_local, form, steps):
    r0 = res_list[-1]
    dom = _roofline(cfg, res_list, n_local, form)
    proj_ms = sum(r.proj_ms for r in res_list)
    _, cp_label = _compute_peak(cfg)
    return {"workload": _workload(cfg, tau, k_max), "value": ms / 1e3, "unit": "s", "ms_per_step": ms,
            "steps": steps, "k": r0.k, "blocks": r0.nblocks, "b_prime": r0.b_prime, "resid_rel": r0.resid_rel,
            "tau": tau, "projection_share_of_step": proj_ms / steps / ms if ms > 0 else None,
            "gpu_launches_per_step": r0.launches,
            "roofline": (dict(dom, kernel=_kernel_label(cfg, dom["bucket"], form), compute_peak_note=cp_label,
                              traffic=_traffic_from_profile(cfg.name)) if dom else None)}


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
    k_max = K_MAX.get(cfg.name)
    # rows of X sharded over the ranks (contiguous, 4096-row aligned); every rank holds
    # only its shard; N = 1 is the single-GPU path (CUDA-graph loop)
    r0, n_local = rdist.partition_rows(cfg.n, world, rank)
    X = make(cfg, device=dev, row_offset=r0, n_local=n_local)
    tau = _tau(cfg, X, world)
    comm = rdist.Comm(dev) if world > 1 else None
    dkw = dict(n_global=cfg.n, row_offset=r0, comm=comm.handle) if comm else {}

    clk = Clocks(local)
    ms, res_list, kw = _measure(rb, cfg, X, tau, k_max, n_local, a.steps, a.warmup, a.form, a.seed, dev, dkw,
                                barrier, world, clk)
    head = _config_entry(cfg, tau, k_max, ms, res_list, n_local, a.form, a.steps)
    launches = sum(r.launches for r in res_list)
    r0res = res_list[-1]
    # per-phase breakdown from one eager, event-instrumented run (outside the timed region)
    rp = rb.id(X, profile=True, **kw)
    rp.W = None
    torch.cuda.synchronize()
    kw = None              # release the headline's workspace and W before the next measurement
    torch.cuda.empty_cache()

    alt = None
    if not a.no_alt_form:
        # side measurement of the other form of Alg. 2 on the same input (not the headline)
        other = "paper" if a.form == "residual" else "residual"
        ns = max(1, min(a.steps, 5))
        t2, rl2, kw2 = _measure(rb, cfg, X, tau, k_max, n_local, ns, 1, other, a.seed, dev, dkw, barrier, world)
        kw2 = None
        torch.cuda.empty_cache()
        e2 = _config_entry(cfg, tau, k_max, t2, rl2, n_local, other, ns)
        alt = {"form": other, "value": t2 / 1e3, "unit": "s", "steps": ns, "k": e2["k"],
               "b_prime": e2["b_prime"], "resid_rel": e2["resid_rel"], "roofline": e2["roofline"],
               "note": ("paper: Alg. 2 literally (X read only, CGS2 l.6, downdated norms l.16; "
                        "SURVEY NEXT-1)" if other == "paper" else "residual: north_star form")}
    torch.cuda.synchronize()
    torch.cuda.empty_cache()

    e2e = None
    if not a.no_e2e:
        # end to end through the C ABI with HOST buffers (rbrp_id_host): every step copies
        # X (pinned host -> HBM) and W (n x k) back to pinned host memory
        try:
            Xh = X.cpu().pin_memory()
            del X
            X = None
            torch.cuda.empty_cache()
            w = 8 if cfg.dtype == "f64" else 4
            hkw = dict(tol=tau, b=cfg.b, seed=a.seed, k_max=k_max or 0, form=a.form, device=dev, **dkw)
            rr, Wh = rb.id_host(Xh, **hkw)
            hws = None
            torch.cuda.synchronize()
            barrier()
            f0 = torch.cuda.Event(enable_timing=True)
            f1 = torch.cuda.Event(enable_timing=True)
            stream = torch.cuda.current_stream(dev)
            ne = max(1, min(a.steps, 3))
            ks = 0
            import paper_2309_16002_b200.rbrp as _r
            import ctypes
            sz = ctypes.c_size_t()
            p = _r._problem(Xh, tau, None, cfg.b, a.seed, k_max or 0, -1.0, 0, dkw.get("n_global"),
                            dkw.get("row_offset", 0), False)
            _r.lib().rbrp_workspace_size_host(ctypes.byref(p), ctypes.byref(sz))
            hws = torch.empty(sz.value, dtype=torch.uint8, device=dev)
            f0.record(stream)
            for _ in range(ne):
                rr, _W = rb.id_host(Xh, workspace=hws, W_host=Wh, **hkw)
                ks = rr.k
            f1.record(stream)
            torch.cuda.synchronize()
            te = f0.elapsed_time(f1) / ne
            if world > 1:
                te = rdist.max_over_ranks(te, device=dev)
            e2e = {"value": te / 1e3, "unit": "s", "h2d_bytes_per_step": n_local * cfg.d * w,
                   "d2h_bytes_per_step": n_local * ks * w + ks * 8, "steps": ne,
                   "note": "per step through rbrp_id_host (C ABI): X pinned host -> HBM (each rank its shard), "
                           "ID in place on the copy, W (n x k) -> pinned host"}
            del Xh, Wh, hws
        except Exception as ex:   # noqa: BLE001 -- host memory may not allow pinning 34 GB
            e2e = {"value": None, "unit": "s", "error": f"{type(ex).__name__}: {ex}"[:300]}
    X = None
    torch.cuda.empty_cache()

    configs = {}
    sk = None
    if world == 1 and not a.no_extra:
        for name in EXTRA:
            if name == cfg.name:
                continue
            c2 = CONFIGS[name]
            Xc = make(c2, device=dev)
            tc = _tau(c2, Xc)
            km = K_MAX.get(name)
            ns = max(1, min(a.steps, 10))
            mc, rlc, kwc = _measure(rb, c2, Xc, tc, km, c2.n, ns, 2, a.form, a.seed, dev, {}, barrier, world)
            configs[name] = _config_entry(c2, tc, km, mc, rlc, c2.n, a.form, ns)
            kwc = None
            torch.cuda.empty_cache()
            if name == "c2" and not a.no_sketch:
                sk = _sketch_side(rb, Xc, rlc[-1].k, a, dev, c2)
            del Xc
            torch.cuda.empty_cache()

    if rank != 0:
        if comm:
            comm.close()
        if world > 1:
            dist.destroy_process_group()
        return
    cpu = None
    if world == 1 and not a.no_cpu_baseline:
        cpu = _cpu_baseline(cfg, a.seed)
    dom = head["roofline"]
    line = {
        "metric": METRIC, "value": ms / 1e3, "unit": "s", "n_gpus": world, "steps": a.steps,
        "warmup": a.warmup, "ms_per_step": ms, "higher_is_better": False,
        "scaling": "strong" if world > 1 else "weak", "vs_baseline": None,
        "dtype": cfg.dtype, "data": "synthetic",
        "config": {"workload": head["workload"],
                   "n": cfg.n, "d": cfg.d, "b": cfg.b, "tau": tau, "k_max": k_max, "k": r0res.k,
                   "blocks": r0res.nblocks, "b_prime": r0res.b_prime, "resid_rel": r0res.resid_rel,
                   "form": a.form,
                   "parallelism": "single" if world == 1 else f"rows{world} (NCCL row sharding)",
                   "rows_per_rank": n_local, "graph_loop": r0res.graph,
                   "l2": "inputs larger than L2 (c5 X 34 GB + residual 34 GB vs 126 MB L2); no flush"},
        "roofline": dict(dom or {}, timing="in-kernel %globaltimer stamps per block (first CTA start -> last CTA "
                                           "end of the block's projection launches), K timed steps",
                         peak_source=PEAKS["source"] + " for HBM; FP64 = unit count x max clock (DESIGN.md §6)",
                         share_of_step=head["projection_share_of_step"]),
        "phase_ms_eager_profile": {k: v for k, v in rp.ms_phase.items() if k != "unused"},
        "gpu_launches": launches,
        "configs": configs,
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


def _sketch_side(rb, X, k_id, a, dev, cfg):
    """SkLUPP-OSID at the ID's rank, l = 3k, on the same X."""
    import torch
    from paper_2309_16002_b200 import sketch as rbs
    ksk = min(k_id, rbs.SK_MAX_K)
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
    stream = torch.cuda.current_stream(dev)
    g0.record(stream)
    for _ in range(ns):
        rs = rbs.sketch_id(X, **kws)
    g1.record(stream)
    torch.cuda.synchronize()
    ts = g0.elapsed_time(g1) / ns
    ph = rbs.sketch_id(X, profile=True, **kws).ms_phase
    lp = (3 * ksk + 7) // 8 * 8
    return {"config": cfg.name, "method": "SkLUPP-OSID (Alg. 4, l = 3k)", "value": ts / 1e3, "unit": "s",
            "steps": ns, "k": rs.k, "l": 3 * ksk, "ms_phase": ph, "launches": rs.launches,
            "sketch_gemm_tflops": 2 * cfg.n * cfg.d * lp / (ph["sketch"] * 1e9),
            "note": "SURVEY NEXT-4 (the paper's GPU competitor, Table 3 P:783); not the headline"}


if __name__ == "__main__":
    main()
