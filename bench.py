"""bench.py — throughput of the B200 hot path (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--dtype f64|f32]
                    [--no-adi] [--no-sweep] [--no-ch1d] [--no-dist] [--no-cpu]

Headline (``value``): the factor-once batched cyclic pentadiagonal solve of
configs[1] at its largest size (N = 8192 unknowns, batch M = 8192 systems,
fp64, interleaved, the thesis CH matrix sigma = 45.09), in M unknowns/s over
all ranks.  A "step" is one pent_solve of the whole batch (one kernel launch,
in place).  The 512 MiB right-hand side is 4x the 126 MB L2, so every step
streams from HBM (no flush needed).  Multi-GPU: every rank solves its own batch
(independent systems, no data-path collective) -> "scaling": "weak".

Secondary legs (each in the same JSON line):
  sweep   configs[1]: N = 256..8192 (batch = N) x {f64, f32}, hot (K solves
          replayed from a CUDA graph) and L2-cold (256 MiB flush before each
          solve, per-solve events)
  ch_adi  configs[3]: 512 CH ADI simulations at 512^2 (L = 4 pi), sharded
          over the ranks, sim-timesteps/s
  cfg3    configs[2]: one 1024^2 simulation (L = 8 pi), 1000 steps as 100
          replays of a 10-step CUDA graph, timesteps/s
  ch1d    thesis §6.2: 2^20 independent 1D CH systems x N = 256, steps/s
  dist    configs[4]: one 16384^2 grid row-partitioned over the ranks (at
          N = 1 the single-rank form of the same exchange code)
The oracle (``oracle/``) is executed only in the cpu_baseline leg and under
``--impl reference`` (rank 0), per the task contract.
"""
from __future__ import annotations

import argparse
import json
import math
import multiprocessing as mp
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import synth  # noqa: E402

METRIC = "penta solve Munknowns/s & % HBM peak; CH ADI timesteps/s at 1/2/4/8 B200"
PENTA_N = 8192          # configs[1], largest size: N = batch = 8192
SWEEP_N = (256, 512, 1024, 2048, 4096, 8192)
ADI_SIMS, ADI_N = 512, 512   # configs[3]
ADI_L = ADI_N * synth.DX_STATS  # 4 pi: dx = 2 pi / 256
CFG3_N = 1024
CFG3_L = CFG3_N * synth.DX_STATS  # 8 pi
CH_D, CH_GAMMA = 1.0, 0.01
CH1D_M, CH1D_N, CH1D_L = 1 << 20, 256, 2 * math.pi   # thesis §6.2.3: 2^20 systems, N = 256 on 2 pi
DIST_N = 16384                     # configs[4]: one 16384^2 grid over the ranks
FLUSH_BYTES = 256 << 20            # > 2x the 126 MB L2


# ------------------------------------------------------------------ host-side helpers (CPU-testable)
def shard(total: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous block [lo, hi) of `total` independent units owned by `rank`."""
    base, rem = divmod(total, world)
    lo = rank * base + min(rank, rem)
    return lo, lo + base + (1 if rank < rem else 0)


def max_over_ranks(x: float, device=None) -> float:
    """Max of a per-rank scalar (timings are reported as the slowest rank)."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(x)
    t = torch.tensor([float(x)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(x: float, device=None) -> float:
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(x)
    t = torch.tensor([float(x)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


def penta_matvec(a, b, c, d, e, x, periodic=True):
    """A x for one system with constant-or-vector diagonals (residual check of
    the bench line; a mat-vec, not a solve)."""
    n = x.shape[0]
    idx = np.arange(n)
    y = c * x
    for off, diag in ((-2, a), (-1, b), (1, d), (2, e)):
        j = idx + off
        if periodic:
            y = y + diag * x[j % n]
        else:
            ok = (j >= 0) & (j < n)
            y = y + np.where(ok, diag * x[np.clip(j, 0, n - 1)], 0.0)
    return y


def host_cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


class ClockSampler:
    """Samples SM clock and throttle reasons through NVML while running."""

    REASONS = {
        "gpu_idle": 0x1, "applications_clocks_setting": 0x2, "sw_power_cap": 0x4, "hw_slowdown": 0x8,
        "sync_boost": 0x10, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
        "hw_power_brake_slowdown": 0x80, "display_clock_setting": 0x100,
    }

    def __init__(self, index: int, period_s: float = 0.005):
        self.index, self.period = index, period_s
        self.samples, self.reasons = [], set()
        self.max_mhz = None
        self._stop = threading.Event()
        self._th = None
        self.ok = False

    def __enter__(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            self._nv = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM)
            self.ok = True
            self._th = threading.Thread(target=self._run, daemon=True)
            self._th.start()
        except Exception as ex:  # no NVML: recorded as unavailable
            self.err = str(ex)
        return self

    def _run(self):
        nv = self._nv
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self._h, nv.NVML_CLOCK_SM))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self._h)
                for k, bit in self.REASONS.items():
                    if r & bit and k != "gpu_idle":
                        self.reasons.add(k)
            except Exception:
                pass
            time.sleep(self.period)

    def __exit__(self, *exc):
        self._stop.set()
        if self._th:
            self._th.join()

    def summary(self):
        if not self.ok:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvml unavailable"]}
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None, "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


def measured_peak_hbm():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def ncu_traffic(key: str):
    """DRAM bytes per launch of `key` from the committed ncu --set full summary
    (profiles/ncu_traffic.json), else None."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(p) as f:
            return json.load(f).get(key)
    except Exception:
        return None


def roofline(alg_bytes, seconds, kernel, key=None, note=None):
    peak, src = measured_peak_hbm()
    ach = alg_bytes / seconds / 1e9
    r = {"bound": "hbm", "achieved": round(ach, 1), "peak": peak, "unit": "GB/s", "frac": round(ach / peak, 4),
         "traffic": ncu_traffic(key) if key else None, "algorithmic_bytes_per_launch": int(alg_bytes),
         "kernel": kernel, "peak_source": src}
    if note:
        r["note"] = note
    return r


# ------------------------------------------------------------------ CPU oracle legs
def _oracle_penta_worker(args):
    """One process: the oracle on `m` systems of the configs[1] workload, repeated
    until `budget` seconds; returns (unknowns, seconds)."""
    m, budget, seed = args
    import oracle
    n = PENTA_N
    s = synth.SIGMA_STATS
    diags = synth.const_penta(n, s, -4 * s, 1 + 6 * s, -4 * s, s)
    f = synth.rhs_uniform(n, m, seed=seed)
    oracle.penta_batch_solve(*diags, f, n=n, m=m, periodic=True)  # warm
    reps, t0 = 0, time.perf_counter()
    while True:
        oracle.penta_batch_solve(*diags, f, n=n, m=m, periodic=True)
        reps += 1
        el = time.perf_counter() - t0
        if el >= budget:
            return reps * n * m, el


def oracle_penta_sample(budget_s: float, cores: int, m_sample: int = 64):
    """The oracle as it stands (single-threaded C) on a bounded sample of the
    configs[1] workload: one process per host core, each solving m_sample
    systems of N = 8192 repeatedly for budget_s; aggregate unknowns/s."""
    if cores <= 1:
        u, el = _oracle_penta_worker((m_sample, budget_s, 2))
        return u / el, 1
    with mp.get_context("spawn").Pool(cores) as pool:
        res = pool.map(_oracle_penta_worker, [(m_sample, budget_s, 2 + k) for k in range(cores)])
    return sum(u / el for u, el in res), cores


def oracle_adi_sample(budget_s: float, sims: int = 2, steps: int = 1):
    import oracle
    c0 = synth.ch_ic_random(sims, ADI_N, seed=4)
    dt = synth.ch_dt(ADI_N, ADI_L)
    reps, t0 = 0, time.perf_counter()
    cn, cm = c0, c0
    while True:
        cn, cm = oracle.ch_adi_steps(cn, cm, steps, dt=dt, D=CH_D, gamma=CH_GAMMA, L=ADI_L)
        reps += 1
        el = time.perf_counter() - t0
        if el >= budget_s:
            break
    return reps * sims * steps / el, f"{reps} x oracle.ch_adi_steps({sims} sims x {ADI_N}^2, {steps} step), 1 core"


# ------------------------------------------------------------------ GPU legs
def _ev(torch):
    return torch.cuda.Event(enable_timing=True)


def thesis_handle(pb, torch, dev, n, m, dtype):
    s = synth.SIGMA_STATS
    diags = synth.const_penta(n, s, -4 * s, 1 + 6 * s, -4 * s, s)
    return pb.pent_factor(*[torch.from_numpy(v).to(dev) for v in diags], batch=m, n=n, periodic=True,
                          dtype=dtype), diags


def bench_penta(args, rank, world, dev):
    import torch
    import torch.distributed as dist
    import paper_2101_06550_b200 as pb

    n = m = PENTA_N
    tdt = torch.float64 if args.dtype == "f64" else torch.float32
    es = 8 if args.dtype == "f64" else 4
    st = torch.cuda.current_stream(dev)
    h, diags = thesis_handle(pb, torch, dev, n, m, args.dtype)
    f_host = synth.rhs_uniform(n, m, seed=2 + rank)
    f_dev = torch.from_numpy(f_host).to(dev, tdt)
    x = f_dev.clone()
    # residual of one solve on sampled systems (fp64 mat-vec on the host)
    h.solve(x)
    torch.cuda.synchronize(dev)
    X = x.double().cpu().numpy().reshape(n, m)
    F = f_dev.double().cpu().numpy().reshape(n, m)
    res = 0.0
    for sy in (0, 1, 4097, m - 1):
        r = penta_matvec(*(v[0] for v in diags), X[:, sy]) - F[:, sy]
        res = max(res, float(np.max(np.abs(r)) / np.max(np.abs(F[:, sy]))))
    for _ in range(args.warmup):   # in-place repeated solves: each step solves the previous result
        h.solve(x)
    torch.cuda.synchronize(dev)
    ev = [_ev(torch) for _ in range(2 * args.steps)]
    pb.reset_launch_count()
    if dist.is_initialized():
        dist.barrier()
    torch.cuda.synchronize(dev)
    with ClockSampler(dev.index if dev.index is not None else 0) as clk:
        t0, t1 = _ev(torch), _ev(torch)
        t0.record(st)
        for k in range(args.steps):
            ev[2 * k].record(st)
            h.solve(x)
            ev[2 * k + 1].record(st)
        t1.record(st)
        torch.cuda.synchronize(dev)
    launches = pb.launch_count()
    if dist.is_initialized():
        dist.barrier()
    ms_local = t0.elapsed_time(t1)
    kern_ms = statistics.mean(ev[2 * k].elapsed_time(ev[2 * k + 1]) for k in range(args.steps))
    ms = max_over_ranks(ms_local, dev)
    kern_ms_max = max_over_ranks(kern_ms, dev)
    value = world * n * m * args.steps / (ms * 1e-3) / 1e6
    alg_bytes = 2 * es * n * m  # read f once, write x once

    # e2e: the same metric through the public C-ABI call with HOST (pinned)
    # buffers: every step the library copies the RHS in and the solution out
    # (pipelined column blocks on two streams, pentab.h host-buffer contract)
    e2e_steps = max(3, min(args.steps, 10))
    xh = torch.from_numpy(f_host).to(tdt).pin_memory()
    h.solve(xh.numpy())  # warm the staging pool
    if dist.is_initialized():
        dist.barrier()
    torch.cuda.synchronize(dev)
    a0, a1 = _ev(torch), _ev(torch)
    w0 = time.perf_counter()
    a0.record(st)
    for _ in range(e2e_steps):
        h.solve(xh.numpy(), stream=st.cuda_stream)
    a1.record(st)
    torch.cuda.synchronize(dev)
    wall = time.perf_counter() - w0
    e2e_ms = max_over_ranks(max(a0.elapsed_time(a1), wall * 1e3), dev)
    e2e_val = world * n * m * e2e_steps / (e2e_ms * 1e-3) / 1e6
    h.close()
    del x, f_dev, xh
    torch.cuda.empty_cache()
    return {
        "value": value, "ms_per_step": ms / args.steps, "kern_ms": kern_ms_max, "launches": launches,
        "residual": res, "clocks": clk.summary(),
        "roofline": roofline(alg_bytes, kern_ms_max * 1e-3, "pent_solve: tp_p1_kernel -> tp_scan_kernel -> "
                             "tp_p2_kernel (3 launches, PDL-chained)", f"pent_solve_{args.dtype}"),
        "e2e": {"value": round(e2e_val, 2), "unit": "Munknowns/s", "steps": e2e_steps,
                "h2d_bytes_per_step": es * n * m, "d2h_bytes_per_step": es * n * m,
                "path": "pent_solve(handle, host pinned rhs) -> pitched H2D | solve | D2H of 16 column "
                        "blocks pipelined on 3 streams"},
    }


def bench_sweep(args, dev):
    """configs[1] sweep: N = 256..8192, batch = N, fp64 and fp32; hot = K solves
    replayed from a CUDA graph (per-solve time = graph time / K), cold = a
    256 MiB write before each solve (per-solve events around the solve only)."""
    import torch
    import paper_2101_06550_b200 as pb

    peak, _ = measured_peak_hbm()
    flush = torch.empty(FLUSH_BYTES // 4, dtype=torch.float32, device=dev)
    side = torch.cuda.Stream(dev)
    out = []
    for dt in ("f64", "f32"):
        tdt = torch.float64 if dt == "f64" else torch.float32
        es = 8 if dt == "f64" else 4
        for n in SWEEP_N:
            m = n
            h, _ = thesis_handle(pb, torch, dev, n, m, dt)
            x = torch.from_numpy(synth.rhs_uniform(n, m, seed=2)).to(dev, tdt)
            K = 20
            with torch.cuda.stream(side):
                for _ in range(3):
                    h.solve(x, stream=side)
                side.synchronize()
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g, stream=side):
                    for _ in range(K):
                        h.solve(x, stream=side)
                g.replay()
                side.synchronize()
                e0, e1 = _ev(torch), _ev(torch)
                e0.record(side)
                for _ in range(5):
                    g.replay()
                e1.record(side)
                side.synchronize()
            hot_us = e0.elapsed_time(e1) * 1e3 / (5 * K)
            host_us = None
            if n == SWEEP_N[0]:
                # host side of a pent_solve: 200 back-to-back calls without a graph,
                # wall clock (the C-ABI call, marshalling and 3 launches each)
                torch.cuda.synchronize(dev)
                w0 = time.perf_counter()
                for _ in range(200):
                    h.solve(x)
                torch.cuda.synchronize(dev)
                host_us = round((time.perf_counter() - w0) * 1e6 / 200, 2)
            cold = []
            for _ in range(10):
                flush.zero_()
                c0, c1 = _ev(torch), _ev(torch)
                c0.record()
                h.solve(x)
                c1.record()
                torch.cuda.synchronize(dev)
                cold.append(c0.elapsed_time(c1) * 1e3)
            cold_us = statistics.median(cold)
            b = 2 * es * n * m
            out.append({"N": n, "batch": m, "dtype": dt, **({"host_us_per_call": host_us} if host_us else {}),
                        "hot_us": round(hot_us, 2), "hot_Munknowns_s": round(n * m / hot_us, 1),
                        "hot_frac": round(b / (hot_us * 1e-6) / 1e9 / peak, 4),
                        "cold_us": round(cold_us, 2), "cold_Munknowns_s": round(n * m / cold_us, 1),
                        "cold_frac": round(b / (cold_us * 1e-6) / 1e9 / peak, 4)})
            h.close()
            del x, g
    del flush
    torch.cuda.empty_cache()
    return {"unit": "us per solve", "hot": "CUDA graph of 20 solves, 5 replays", "cold": "256 MiB write before each "
            "solve, median of 10", "frac": "16 (8) B per unknown / time / measured HBM peak", "rows": out}


def bench_adi(args, rank, world, dev):
    import torch
    import torch.distributed as dist
    import paper_2101_06550_b200 as pb

    lo, hi = shard(ADI_SIMS, world, rank)
    sims = hi - lo
    tdt = torch.float64 if args.dtype == "f64" else torch.float32
    es = 8 if args.dtype == "f64" else 4
    dt = synth.ch_dt(ADI_N, ADI_L)
    # IC U(-0.1, 0.1), sim k seeded 4 + k; generated on the device
    # from per-sim seeds for speed (parity tests use the host generator)
    g = torch.Generator(device=dev)
    c0 = torch.empty((sims, ADI_N, ADI_N), dtype=tdt, device=dev)
    for k in range(sims):
        g.manual_seed(4 + lo + k)
        c0[k].uniform_(-0.1, 0.1, generator=g)
    state = pb.CHState(c0)
    del c0
    st = torch.cuda.current_stream(dev)
    mass0 = float(state.c_cur.double().sum())
    pb.ch_adi_step(state, dt, D=CH_D, gamma=CH_GAMMA, L=ADI_L, nsteps=args.warmup)
    torch.cuda.synchronize(dev)
    steps = args.adi_steps
    pb.reset_launch_count()
    if dist.is_initialized():
        dist.barrier()
    torch.cuda.synchronize(dev)
    with ClockSampler(dev.index if dev.index is not None else 0) as clk:
        t0, t1 = _ev(torch), _ev(torch)
        t0.record(st)
        pb.ch_adi_step(state, dt, D=CH_D, gamma=CH_GAMMA, L=ADI_L, nsteps=steps)
        t1.record(st)
        torch.cuda.synchronize(dev)
    launches = pb.launch_count()
    ms = max_over_ranks(t0.elapsed_time(t1), dev)
    mass1 = float(state.c_cur.double().sum())
    drift = max_over_ranks(abs(mass1 - mass0) / (ADI_N * ADI_N * max(sims, 1)), dev)
    alg_bytes = 7 * es * ADI_N * ADI_N * sims  # 7 field passes per point and step
    del state
    torch.cuda.empty_cache()
    return {
        "value": round(ADI_SIMS * steps / (ms * 1e-3), 2), "unit": "sim-timesteps/s",
        "whole_batch_steps_per_s": round(steps / (ms * 1e-3), 2), "ms_per_step": ms / steps, "steps": steps,
        "config": {"workload": "configs[3]: 512 CH ADI sims at 512^2, L=4pi, dt=0.1dx, D=1, gamma=0.01",
                   "sims_per_rank": sims, "scaling": "weak (independent sims sharded, no collective)",
                   "dtype": args.dtype},
        "launches": launches, "mean_abs_mass_drift_per_point": drift, "clocks": clk.summary(),
        "roofline": roofline(sum_over_ranks(alg_bytes, dev) / world, ms / steps * 1e-3,
                             "one step: adi_rhs_kernel + fh_kernel<contiguous> (x-sweep) + fh_kernel<interleaved> "
                             "(y-sweep) + adi_combine_kernel", f"adi_step_{args.dtype}",
                             "algorithmic 56 B/point (7 field passes); this schedule moves 11 fp64-sized passes"),
    }


def bench_coarsen(args, dev):
    """SURVEY §8(f)2 on the configs[3] batch: 512 Cahn–Hilliard–Cook sims at
    512^2 from C = 0 (sigma = 1e-14), every step followed by the
    on-device free energy of all sims (the F(t) series beta is built from)."""
    import torch
    import paper_2101_06550_b200 as pb

    tdt = torch.float64 if args.dtype == "f64" else torch.float32
    dt = synth.ch_dt(ADI_N, ADI_L)
    st = pb.CHState(torch.zeros((ADI_SIMS, ADI_N, ADI_N), dtype=tdt, device=dev))
    F = torch.empty((args.adi_steps, ADI_SIMS), dtype=torch.float64, device=dev)
    pb.ch_adi_step_cook(st, dt, sigma=1e-14, seed=1, step0=0, L=ADI_L, nsteps=args.warmup)
    torch.cuda.synchronize(dev)
    e0, e1 = _ev(torch), _ev(torch)
    e0.record()
    for k in range(args.adi_steps):
        pb.ch_adi_step_cook(st, dt, sigma=1e-14, seed=1, step0=args.warmup + k, L=ADI_L, nsteps=1)
        pb.ch_free_energy(st, F[k], L=ADI_L)
    e1.record()
    torch.cuda.synchronize(dev)
    ms = e0.elapsed_time(e1) / args.adi_steps
    f0, f1 = F[0].mean().item(), F[-1].mean().item()
    del st, F
    torch.cuda.empty_cache()
    return {"value": round(ADI_SIMS / (ms * 1e-3), 2), "unit": "sim-timesteps/s", "ms_per_step": round(ms, 4),
            "config": {"workload": "SURVEY 8(f)2 on configs[3]: 512 CHC sims at 512^2 from C=0, sigma=1e-14, "
                                   "free energy of every sim after every step", "dtype": args.dtype},
            "mean_F_first_last": [f0, f1]}


def bench_regimes(args, dev):
    """SURVEY §8(f)3 solver regimes, each a step of stencil RHS + batched solve
    composed from the library calls (explicit half by stencil_apply, implicit
    half by the factor-once solve), 2^16 interleaved systems x N = 1024, fp64:
      cn_tri    CN diffusion, tridiagonal Thomas / Sherman–Morrison
      cn_penta  CN hyperdiffusion, uniform pentadiagonal
      rewrite   per-system pentadiagonal LHS re-factored every step, then solved
                (cuPentBatchRewrite)
    Steps/s and unknowns/s over 50 steps (after 3 warm-up steps)."""
    import torch
    import paper_2101_06550_b200 as pb

    n, m, steps = 1024, 1 << 16, 50
    out = {}
    x = torch.from_numpy(synth.rhs_uniform(n, m, seed=12)).to(dev).view(n, m)   # [row][system]
    f = torch.empty_like(x)
    dx = 1.0 / n

    def timed(step):
        for _ in range(3):
            step()
        torch.cuda.synchronize(dev)
        e0, e1 = _ev(torch), _ev(torch)
        e0.record()
        for _ in range(steps):
            step()
        e1.record()
        torch.cuda.synchronize(dev)
        return e0.elapsed_time(e1) / steps

    st = 1e-4 / (2 * dx * dx)
    ht = pb.tri_factor_uniform(-st, 1 + 2 * st, -st, batch=m, n=n, periodic=True)
    wt = np.array([st, 1 - 2 * st, st])

    buf = [x, f]   # the levels swap every step

    def tri_step():
        pb.stencil_apply(buf[0], buf[1], wt, left=0, right=0, top=1, bottom=1, periodic=True)
        ht.solve(buf[1])
        buf.reverse()
    ms = timed(tri_step)
    out["cn_tri"] = {"ms_per_step": round(ms, 4), "Munknowns_s": round(n * m / (ms * 1e-3) / 1e6, 1)}
    ht.close()
    sp = 1e-8 / (2 * dx ** 4)
    hp = pb.pent_factor_uniform(sp, -4 * sp, 1 + 6 * sp, -4 * sp, sp, batch=m, n=n, periodic=True)
    wp = np.array([-sp, 4 * sp, 1 - 6 * sp, 4 * sp, -sp])

    def pent_step():
        pb.stencil_apply(buf[0], buf[1], wp, left=0, right=0, top=2, bottom=2, periodic=True)
        hp.solve(buf[1])
        buf.reverse()
    ms = timed(pent_step)
    out["cn_penta"] = {"ms_per_step": round(ms, 4), "Munknowns_s": round(n * m / (ms * 1e-3) / 1e6, 1)}
    hp.close()
    mr = 1 << 14
    a, b, c, d, e = (torch.from_numpy(v).to(dev) for v in synth.dd_penta(n, mr, seed=13))
    hr = pb.pent_factor(a, b, c, d, e, batch=mr, n=n, lhs_count=mr, periodic=False)
    xr = torch.from_numpy(synth.rhs_uniform(n, mr, seed=14)).to(dev)

    def rewrite_step():
        hr.refactor(a, b, c, d, e)
        hr.solve(xr)
    ms = timed(rewrite_step)
    out["rewrite"] = {"ms_per_step": round(ms, 4), "Munknowns_s": round(n * mr / (ms * 1e-3) / 1e6, 1),
                      "batch": mr}
    hr.close()
    del x, f, buf, xr, a, b, c, d, e
    torch.cuda.empty_cache()
    out["config"] = {"workload": "SURVEY 8(f)3: 2^16 systems x N=1024 (rewrite: 2^14), fp64, 50 steps each",
                     "step": "stencil_apply + solve (CN); refactor + solve (rewrite)"}
    return out


def bench_cfg3(args, dev):
    """configs[2]: one 1024^2 simulation (L = 8 pi), 1000 steps = 100 replays of a
    10-step CUDA graph (launch-latency bound: 4 launches per step)."""
    import torch
    import paper_2101_06550_b200 as pb

    tdt = torch.float64 if args.dtype == "f64" else torch.float32
    es = 8 if args.dtype == "f64" else 4
    dt = synth.ch_dt(CFG3_N, CFG3_L)
    c0 = torch.from_numpy(synth.ch_ic_random(1, CFG3_N, seed=3)).to(dev, tdt)
    state = pb.CHState(c0)
    side = torch.cuda.Stream(dev)
    with torch.cuda.stream(side):
        pb.ch_adi_step(state, dt, D=CH_D, gamma=CH_GAMMA, L=CFG3_L, nsteps=4, stream=side)
        side.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=side):
            pb.ch_adi_step(state, dt, D=CH_D, gamma=CH_GAMMA, L=CFG3_L, nsteps=10, stream=side)
        g.replay()
        side.synchronize()
        e0, e1 = _ev(torch), _ev(torch)
        e0.record(side)
        for _ in range(100):
            g.replay()
        e1.record(side)
        side.synchronize()
    ms = e0.elapsed_time(e1)
    steps = 1000
    del state, g
    torch.cuda.empty_cache()
    return {"value": round(steps / (ms * 1e-3), 1), "unit": "timesteps/s", "us_per_step": round(ms * 1e3 / steps, 2),
            "config": {"workload": "configs[2]: one 1024^2 CH ADI sim, L=8pi, dt=0.1dx", "dtype": args.dtype,
                       "graph": "10 steps captured, 100 replays"},
            "effective_GBs": round(56 * CFG3_N * CFG3_N * steps / (ms * 1e-3) / 1e9 * es / 8, 1)}


def bench_ch1d(args, dev):
    """thesis §6.2.3: 2^20 independent 1D CH systems x N = 256 (L = 2 pi,
    dt = 0.1 dx, gamma = 0.01), U(-0.1, 0.1) quench; K steps in one call."""
    import torch
    import paper_2101_06550_b200 as pb

    tdt = torch.float64 if args.dtype == "f64" else torch.float32
    es = 8 if args.dtype == "f64" else 4
    dt = synth.ch_dt(CH1D_N, CH1D_L)
    g = torch.Generator(device=dev)
    g.manual_seed(6)
    c0 = torch.empty((CH1D_N, CH1D_M), dtype=tdt, device=dev).uniform_(-0.1, 0.1, generator=g)
    st = pb.CH1DState(c0)
    del c0
    pb.ch1d_step(st, dt, gamma=CH_GAMMA, L=CH1D_L, nsteps=args.warmup)
    torch.cuda.synchronize(dev)
    steps = args.steps
    e0, e1 = _ev(torch), _ev(torch)
    e0.record()
    pb.ch1d_step(st, dt, gamma=CH_GAMMA, L=CH1D_L, nsteps=steps)
    e1.record()
    torch.cuda.synchronize(dev)
    ms = e0.elapsed_time(e1)
    alg = 2 * es * CH1D_N * CH1D_M   # read C^n, write C^{n+1}
    del st
    torch.cuda.empty_cache()
    return {"value": round(steps / (ms * 1e-3), 2), "unit": "batch-timesteps/s",
            "system_steps_per_s": round(CH1D_M * steps / (ms * 1e-3), 1), "ms_per_step": round(ms / steps, 4),
            "config": {"workload": "thesis §6.2.3: 2^20 1D CH systems x N=256, L=2pi, dt=0.1dx", "dtype": args.dtype},
            "roofline": roofline(alg, ms / steps * 1e-3, "fh_kernel<MODE_CH1D> (RHS formed on chip, one launch per step)",
                                 f"ch1d_{args.dtype}")}


def bench_dist_adi(args, rank, world, dev):
    """configs[4]: one 16384^2 CH grid row-partitioned over the ranks, two
    all-to-all transposes per step (paper_2101_06550_b200.dist, NCCL).
    Time-steps/s of the whole grid; max over ranks."""
    import torch
    import torch.distributed as dist
    from paper_2101_06550_b200 import dist as pdist

    n = args.dist_n
    tdt = torch.float64 if args.dtype == "f64" else torch.float32
    dt = synth.ch_dt(n, n * synth.DX_STATS)
    prm = pdist.Params(n=n, parts=world, dt=dt, L=n * synth.DX_STATS)
    g = torch.Generator(device=dev)
    g.manual_seed(5 + rank)   # IC U(-0.1, 0.1), this rank's rows (synthetic)
    rows = torch.empty((prm.rows, n), dtype=tdt, device=dev).uniform_(-0.1, 0.1, generator=g)
    st = pdist.RankState(prm, rank, rows, rows, pdist.LibCompute(prm, dev, tdt))
    del rows
    ex = pdist.TorchExchange() if world > 1 else pdist.LocalExchange()
    for _ in range(max(args.warmup, 1)):
        pdist.step([st], ex)
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    steps = args.dist_steps
    e0, e1 = _ev(torch), _ev(torch)
    e0.record()
    for _ in range(steps):
        pdist.step([st], ex)
    e1.record()
    torch.cuda.synchronize(dev)
    ms = max_over_ranks(e0.elapsed_time(e1), dev)
    a2a = 2 * 8 * prm.rows * n * (world - 1) / world   # fp64 bytes each rank sends per step (two transposes)
    del st
    torch.cuda.empty_cache()
    return {"value": round(steps / (ms * 1e-3), 3), "unit": "grid-timesteps/s", "ms_per_step": ms / steps,
            "steps": steps, "config": {"workload": f"configs[4]: one {n}^2 CH grid, L=128pi, row-partitioned x{world}",
                                       "exchange": "2 all-to-all transposes + halo rows per step (torch.distributed)",
                                       "dtype": args.dtype},
            "a2a_bytes_per_rank_per_step": a2a}


def _leg(fn, *a):
    try:
        return fn(*a)
    except Exception as ex:  # reported, never fatal to the headline
        return {"error": f"{type(ex).__name__}: {ex}"[:300]}


def run_ours(args):
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        if world == 1 and args.gpus > 1:
            raise SystemExit("--gpus N>1 must be launched with torchrun (one process per GPU)")
    if not torch.cuda.is_available():
        raise SystemExit("bench.py needs a CUDA device (no CPU fallback)")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    import paper_2101_06550_b200 as pb
    pb.lib()
    r = bench_penta(args, rank, world, dev)
    adi = _leg(bench_adi, args, rank, world, dev) if not args.no_adi else None
    sweep = _leg(bench_sweep, args, dev) if (not args.no_sweep and rank == 0) else None
    cfg3 = _leg(bench_cfg3, args, dev) if (not args.no_adi and rank == 0) else None
    ch1d = _leg(bench_ch1d, args, dev) if (not args.no_ch1d and rank == 0) else None
    coarsen = _leg(bench_coarsen, args, dev) if (not args.no_adi and rank == 0) else None
    regimes = _leg(bench_regimes, args, dev) if (not args.no_sweep and rank == 0) else None
    dist_adi = _leg(bench_dist_adi, args, rank, world, dev) if not args.no_dist else None
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cores = host_cores()
        v1, _ = oracle_penta_sample(args.cpu_budget / 2, 1)
        vN, used = oracle_penta_sample(args.cpu_budget / 2, cores)
        va, sa = oracle_adi_sample(args.cpu_budget / 3)
        cpu = {"value": round(vN / 1e6, 3), "unit": "Munknowns/s", "cores": used, "kind": "oracle",
               "cpu_model": cpu_model(), "affinity_cores": cores,
               "sample": f"oracle.penta_batch_solve of 64 of the 8192 systems (N=8192, cyclic, fp64) repeated for "
                         f"{args.cpu_budget / 2:.0f} s in each of {used} processes (one per host core)",
               "single_core": {"value": round(v1 / 1e6, 3), "unit": "Munknowns/s", "cores": 1},
               "ch_adi": {"value": round(va, 3), "unit": "sim-timesteps/s", "sample": sa}}
    if rank == 0:
        line = {
            "metric": METRIC, "value": round(r["value"], 2), "unit": "Munknowns/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(r["ms_per_step"], 5),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": args.dtype,
            "data": "synthetic (seeded U(-1,1) RHS; thesis CH matrix sigma=45.09 at dx=2pi/256)",
            "config": {"workload": "configs[1]: batched cyclic penta solve, N=8192, batch=8192 per GPU, "
                                   "factor-once/solve-many, interleaved", "N": PENTA_N, "batch_per_gpu": PENTA_N,
                       "layout": "interleaved", "l2": "inputs (512 MiB fp64) larger than the 126 MB L2; no flush",
                       "parallelism": f"independent batches x{world}"},
            "roofline": r["roofline"], "cpu_baseline": cpu, "e2e": r["e2e"], "gpu_launches": r["launches"],
            "clocks": r["clocks"], "residual": r["residual"], "sweep": sweep, "ch_adi": adi, "cfg3": cfg3,
            "ch1d": ch1d, "coarsen": coarsen, "regimes": regimes, "dist_adi": dist_adi,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def run_reference(args):
    """Reference arm: the CPU oracle as it stands (this tier has no reference
    implementation), on the same workload/metric, rank 0 only, one process per
    host core."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    cores = host_cores()
    per_step = max(0.5, 60.0 / max(args.steps + args.warmup, 1))
    t0 = time.perf_counter()
    v, used = oracle_penta_sample(per_step * args.steps, cores)
    el = time.perf_counter() - t0
    sample = (f"oracle.penta_batch_solve of 64 of the 8192 systems (N=8192, cyclic, fp64) repeated in each of {used} "
              f"processes (one per host core) for {per_step * args.steps:.1f} s")
    vv = round(v / 1e6, 3)
    line = {
        "impl": "reference", "metric": METRIC, "value": vv, "unit": "Munknowns/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(PENTA_N * PENTA_N / v * 1e3, 3), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": "configs[1]: batched cyclic penta solve, N=8192, batch=8192 per GPU, "
                               "factor-once/solve-many, interleaved", "N": PENTA_N, "batch_per_gpu": PENTA_N},
        "cpu_baseline": {"value": vv, "unit": "Munknowns/s", "cores": used, "kind": "oracle", "sample": sample,
                         "cpu_model": cpu_model()},
        "e2e": {"value": vv, "unit": "Munknowns/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "wall_s": round(el, 2),
    }
    print(json.dumps(line), flush=True)


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--adi-steps", type=int, default=None, help="ADI steps timed (default: --steps)")
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--dtype", choices=["f64", "f32"], default="f64")
    ap.add_argument("--no-adi", action="store_true")
    ap.add_argument("--no-sweep", action="store_true")
    ap.add_argument("--no-ch1d", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-dist", action="store_true", help="skip the configs[4] row-partitioned leg")
    ap.add_argument("--dist-n", type=int, default=DIST_N)
    ap.add_argument("--dist-steps", type=int, default=10)
    ap.add_argument("--cpu-budget", type=float, default=12.0)
    args = ap.parse_args(argv)
    if args.warmup < 3:
        ap.error("--warmup must be >= 3")
    if args.adi_steps is None:
        args.adi_steps = args.steps
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
