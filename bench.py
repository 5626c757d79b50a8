#!/usr/bin/env python
"""bench.py -- headline benchmark of the B200 hot path (driver contract in DESIGN.md §6).

Workload (BASELINE.json configs[1]): Poisson stiffness cell matrices, Lagrange P4 on 65,536
seeded affine tetrahedra (reference tet + U(-0.15, 0.15) noise, seed 1 + rank), the
125-point collapsed Gauss-Jacobi rule, c(x) = 1 + 0.5 sin(2 pi x) cos(2 pi y) e^z, mixed
precision (u_p = fp32, G_K at u_g = fp64, u_q = fp32 TMEM accumulation, u_s = fp16
storage), 35 x 35 fp32 outputs. One step = vertices in HBM -> geometry/scaled weights (K1)
-> tcgen05 cell-matrix GEMM (K2) -> matrices in HBM.

  python bench.py [--gpus N --steps K --warmup W] [--impl reference] [--sweep]

N > 1 runs under torchrun: every rank processes its own 65,536 cells (weak scaling, no
collective on the data path); time is the max over ranks.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

P_DEG = 4
N_CELLS = 65536
METRIC = "cell matrices/s"
UNIT = "cells/s"


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as f:
            d = json.load(f)
        return d.get("hbm_gbs", 6650.0), d.get("bf16_tflops", 1590.0), d.get("bf16_tflops_sustained"), "measured"
    return 6650.0, 1590.0, 1400.0, "fallback"


def profiled_traffic(kernel_prefix="cellmat_tc2_kernel<0, 0>", fallback_prefix="cellmat_tc2_kernel"):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of the dominant kernel from the
    latest committed `ncu --set full` capture summary (profiles/r*_ncu_summary.json `ncu_full`,
    profiles/r*_zoo_summary.json `poisson_k2`: the headline workload), or None."""
    import glob

    def to_bytes(v):
        if isinstance(v, (int, float)):
            return float(v) * 1e6  # older summaries: bare Mbyte numbers
        num, _, unit = str(v).partition(" ")
        return float(num) * {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1e6)

    best = None
    paths = glob.glob(os.path.join(ROOT, "profiles", "r*_ncu_summary.json")) + \
        glob.glob(os.path.join(ROOT, "profiles", "r*_zoo_summary.json"))
    def round_key(path):  # r1k < r2a < r2x < r2ba: shorter round tags are older
        tag = os.path.basename(path).split("_")[0]
        return (len(tag), tag, os.path.basename(path))

    for path in sorted(paths, key=round_key):
        try:
            with open(path) as f:
                d = json.load(f)
            for k in list(d.get("ncu_full", [])) + list(d.get("poisson_k2", [])):
                name = k.get("kernel", "")
                if kernel_prefix in name or (fallback_prefix in name and "<" not in name):
                    best = {"bytes": to_bytes(k["dram__bytes_read.sum"]) + to_bytes(k["dram__bytes_write.sum"]),
                            "source": os.path.relpath(path, ROOT)}
        except Exception:
            continue
    return best


def nphi(p):
    return (p + 1) * (p + 2) * (p + 3) // 6


def work_per_cell(p, form, out_bytes=4):
    n = nphi(p)
    nq = (p + 1) ** 3
    nd = 3 if form == 1 else 1
    flops = 2.0 * n * n * nq * nd * nd          # SURVEY 8d F_cell (dense, reference Alg. 1 depth)
    bytes_ = 96.0 + out_bytes * n * n           # fp64 vertices in + full matrix out
    return flops, bytes_


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled while the timed region runs."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.lines: list[str] = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return None
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.t.join(timeout=2)
        sms, maxs, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sms.append(float(parts[0]))
                maxs.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[3:7]):
                if v.lower() == "active":
                    reasons.add(nm)
        if not sms:
            return None
        return {"sm_mhz": float(np.median(sms)), "sm_max_mhz": float(max(maxs)),
                "reasons": sorted(reasons), "samples": len(sms)}


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def host_cores():
    return len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count()


def cpu_run(p, form, cfg_tuple, verts, coef_kind, n):
    """One timed pass of the reference's own CPU path over the first n cells: oracle/_ref (the
    unmodified reference, compiled from its sources) under mpfem::parallel_for on every host
    core, or the C restatement (oracle/, one thread) where _ref was not built.
    Returns (seconds, kind, cores)."""
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from oracle_lib import Oracle, Reference, reference_available
    v = verts.reshape(-1, 12)[:n]
    if reference_available():
        cores = host_cores()
        secs, _ = Reference().cpu_baseline(p, form, cfg_tuple, v, coef_kind, None, cores)
        return secs, "reference", cores
    t = time.perf_counter()
    Oracle().bilinear(p, form, cfg_tuple, v, coef_kind, None)
    return time.perf_counter() - t, "port", 1


def cpu_sample_size(p, form, cfg_tuple, verts, coef_kind, target_s):
    """Cells per CPU step so that one step takes about target_s seconds (calibrated on a
    short run), capped at the whole workload."""
    cores = host_cores()
    n0 = min(verts.shape[0], 2 * cores)
    secs, _, _ = cpu_run(p, form, cfg_tuple, verts, coef_kind, n0)
    rate = n0 / max(secs, 1e-9)
    return int(min(verts.shape[0], max(n0, rate * target_s)))


def cpu_baseline(p, form, cfg_tuple, verts, coef_kind, target_s=10.0):
    """The reported CPU baseline of the main arm: the reference CPU path timed on a bounded
    prefix sample of the same cells. Returns (cells/s, kind, cores, sample)."""
    n = cpu_sample_size(p, form, cfg_tuple, verts, coef_kind, target_s)
    secs, kind, cores = cpu_run(p, form, cfg_tuple, verts, coef_kind, n)
    thr = f"MPFEM_THREADS={cores}" if kind == "reference" else "1 thread (C restatement)"
    return n / secs, kind, cores, f"first {n} of the {verts.shape[0]} cells, {thr}, {cpu_model()}"


MIXED_CFG = dict(u_p=2, u_g=3, u_q=2, u_s=1, engine=0)  # config 1: G_K at fp64


def workload_config():
    return {"workload": "config1: poisson P4 stiffness, 65536 seeded affine tets, mixed "
                        "(u_s=fp16, fp32 TMEM accumulation, G_K fp64), c(x)=1+0.5sin(2pi x)cos(2pi y)e^z",
            "p": P_DEG, "cells_per_gpu": N_CELLS, "form": "poisson", "mode": "mixed",
            "u_p": "fp32", "u_g": "fp64", "u_q": "fp32", "u_s": "fp16",
            "l2": "flushed before every timed step (256 MiB write)",
            "output": "fp32, 35x35 row-major per cell"}


def run_reference(args, rank, world):
    """--impl reference: the reference's own CPU implementation of the headline path, timed
    on this host's cores. The inputs come from the parity checker's generator (oracle/,
    bitwise the product's, tests/test_abi_cpu.py) so this process never maps the product
    library. Each step is the same bounded prefix sample of the 65,536 config-1 cells, sized
    so the warmup + steps run ends within about 2.5 minutes; ms_per_step is the measured
    wall time of one such step and value = sample cells / that time."""
    if rank != 0:
        return
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from oracle_lib import Oracle
    verts, _ = Oracle().gen_tets(0, 1, N_CELLS)
    cfg = (MIXED_CFG["u_p"], MIXED_CFG["u_g"], MIXED_CFG["u_q"], MIXED_CFG["u_s"], MIXED_CFG["engine"])
    per_step = max(0.2, min(args.ref_seconds, 150.0 / max(1, args.steps + args.warmup)))
    t_all = time.perf_counter()
    n = cpu_sample_size(P_DEG, 1, cfg, verts, 1, per_step)
    for _ in range(max(0, args.warmup - 1)):  # the calibration run is the first warmup step
        cpu_run(P_DEG, 1, cfg, verts, 1, n)
    secs = []
    kind, cores = None, None
    for _ in range(args.steps):
        s_, kind, cores = cpu_run(P_DEG, 1, cfg, verts, 1, n)
        secs.append(s_)
    wall = time.perf_counter() - t_all
    step_s = float(np.mean(secs))
    value = n / step_s
    thr = f"MPFEM_THREADS={cores}" if kind == "reference" else "1 thread (C restatement)"
    sample = (f"each step: the first {n} of the {N_CELLS} config-1 cells ({thr}); "
              f"host CPU: {cpu_model()}")
    conf = dict(workload_config(), cells_per_step=n)
    line = {"metric": METRIC, "value": value, "unit": UNIT, "impl": "reference", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * step_s,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "fp32",
            "data": "synthetic (seeded, oracle generator)", "config": conf,
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": kind,
                             "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "wall_s": wall}
    print(json.dumps(line), flush=True)


def run_sweep(mp, torch, dev, only=None):
    """BASELINE config 2: p = 1..8, mass and Poisson, in BASELINE's "mixed" mode (fp16
    storage, fp32 accumulation), the paper's bf16-storage mixed mode as an extra column, and
    fp64; the cell count per p is chosen so the outputs total 4 GiB (2^32 / (s_out n_phi^2),
    s_out = 4 for the fp32 outputs of the mixed modes, 8 for fp64)."""
    hbm, tc_peak, _, _ = peaks()
    res = []
    for p in range(1, 9):
        for form in (0, 1):
            for mode in ("mixed", "mixed_bf16", "fp64"):
                if only and (p, form, mode) not in only:
                    continue
                cfg = mp.mode_config(mode, form)
                ob = 8 if mode == "fp64" else 4
                n = (1 << 32) // (ob * nphi(p) ** 2)
                verts, _ = mp.gen_tets(0, 7 + p, n)
                vd = torch.from_numpy(verts).to(dev)
                s = mp.make_setup(p, cfg)
                s.reserve(n)
                out = torch.empty((n, nphi(p) ** 2), dtype=torch.float32 if ob == 4 else torch.float64, device=dev)
                s.cell_matrices(vd, None, 1, out=out)
                torch.cuda.synchronize()
                reps = 3 if mode != "fp64" or p < 6 else 1
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                for _ in range(reps):
                    s.cell_matrices(vd, None, 1, out=out)
                e1.record()
                torch.cuda.synchronize()
                ms = e0.elapsed_time(e1) / reps
                s.set_timing(True)
                s.cell_matrices(vd, None, 1, out=out)
                kt = s.last_timings()
                s.set_timing(False)
                s.synchronize()
                f, b = work_per_cell(p, form, ob)
                t_tc = n * f / (tc_peak * 1e12) if mode != "fp64" else 0.0
                t_roof = max(t_tc, n * b / (hbm * 1e9))
                res.append({"p": p, "form": "poisson" if form else "mass", "mode": mode, "cells": n,
                            "ms": ms, "cells_per_s": n / (ms * 1e-3),
                            "tflops_dense_equiv": n * f / (ms * 1e-3) / 1e12,
                            "hbm_gbs_algorithmic": n * b / (ms * 1e-3) / 1e9,
                            "bound": ("tensor" if t_tc * 1e9 > n * b / hbm else "hbm") if mode != "fp64" else "fp64",
                            "roofline_frac": (t_roof / (ms * 1e-3)) if mode != "fp64" else None,
                            "path": s.path, "kernels_ms": kt})
                del s, out, vd
                torch.cuda.empty_cache()
    return res


UNIT_ROUNDOFF = {0: 2.0 ** -8, 1: 2.0 ** -11, 2: 2.0 ** -24, 3: 2.0 ** -53}  # bf16 fp16 fp32 fp64


def timed_ms(torch, fn, reps=20, flush=None):
    """Mean CUDA-event time of fn on the current stream, L2 flushed before each call."""
    fn()
    torch.cuda.synchronize()
    tot = 0.0
    for _ in range(reps):
        if flush is not None:
            flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        tot += e0.elapsed_time(e1)
    return tot / reps


def fin(x):
    """JSON-safe float: non-finite values as strings."""
    x = float(x)
    return x if np.isfinite(x) else str(x)


def err_rel(torch, a, a64):
    """Per-cell max|A - A64| / max|A64| (errorlab.cpp:90-99), NaN as +inf."""
    n = a64.shape[0]
    d = (a.reshape(n, -1).double() - a64.reshape(n, -1)).abs().amax(dim=1)
    e = d / a64.reshape(n, -1).abs().amax(dim=1)
    return torch.nan_to_num(e, nan=float("inf")).cpu().numpy()


def run_modes(mp, torch, dev, flush):
    """BASELINE configs 0 (mass) and 1 (Poisson): 65,536 seeded P4 tets, c(x) at the quadrature
    points, every precision mode: cells/s of the device step and the per-cell error against
    the device fp64 mode (itself pinned to the fp64 oracle by tests/test_gpu_cells.py).
    Config 1 computes G_K at u_g = fp64 in every mode."""
    verts, _ = mp.gen_tets(0, 1, N_CELLS)
    vd = torch.from_numpy(verts).to(dev)
    res = []
    for form, name in ((0, "config0 mass"), (1, "config1 poisson")):
        ref = None
        for mode in ("fp64", "fp32", "fp16", "mixed", "mixed_bf16"):
            cfg = mp.mode_config(mode, form, geometry_fp64=(form == 1))
            s = mp.make_setup(P_DEG, cfg)
            s.reserve(N_CELLS)
            out = torch.empty((N_CELLS, s.n_phi ** 2), dtype=torch.float64 if s.path == 2 else torch.float32,
                              device=dev)
            ms = timed_ms(torch, lambda: s.cell_matrices(vd, None, mp.CoefKind.sincosexp, out=out), flush=flush)
            if mode == "fp64":
                ref = out.clone()
                e = np.zeros(1)
            else:
                e = err_rel(torch, out, ref)
            us = UNIT_ROUNDOFF[int(cfg.u_s)]
            res.append({"config": name, "mode": mode, "u_p/u_g/u_q/u_s": [int(cfg.u_p), int(cfg.u_g), int(cfg.u_q), int(cfg.u_s)],
                        "ms": ms, "cells_per_s": N_CELLS / (ms * 1e-3),
                        "max_err_rel": fin(e.max()), "max_err_over_u_s": fin(e.max() / us)})
            del s, out
        del ref
        torch.cuda.empty_cache()
    return res


def run_action(mp, torch, dev, flush, sm_mhz):
    """Algorithm 2 (action_kernel, kernels.cpp:269-304) on the config-0/1 workloads: 65,536
    seeded P4 tets, c(x) at the quadrature points, one w per cell, every precision mode.
    One launch per step (KA, bitwise the reference's op order); cells/s, error against the
    device fp64 action, and the issue roof: the reference rounds every product and sum, so
    each of the 2 n_phi n_d n_q multiply-adds per cell is two instructions (FMUL+FADD at 128
    lanes/clk/SM, or DMUL+DADD at 64/clk/SM in fp64 mode)."""
    verts, _ = mp.gen_tets(0, 1, N_CELLS)
    vd = torch.from_numpy(verts).to(dev)
    rng = np.random.default_rng(1)
    res = []
    clk = sm_mhz * 1e6
    for form, name in ((0, "config0 mass"), (1, "config1 poisson")):
        n_phi, n_q, n_d = nphi(P_DEG), (P_DEG + 1) ** 3, 3 if form else 1
        wd = torch.from_numpy(rng.uniform(-1.0, 1.0, size=(N_CELLS, n_phi))).to(dev)
        ref = None
        pairs = 2.0 * n_phi * n_d * n_q * N_CELLS
        for mode in ("fp64", "fp32", "fp16", "mixed", "mixed_bf16"):
            cfg = mp.mode_config(mode, form, geometry_fp64=(form == 1))
            cfg.mode = mp.ModeKind.action
            s = mp.make_setup(P_DEG, cfg)
            out = torch.empty((N_CELLS, n_phi), dtype=torch.float64 if mode == "fp64" else torch.float32,
                              device=dev)
            ms = timed_ms(torch, lambda: mp.action_kernel(s, vd, wd, coef_kind=mp.CoefKind.sincosexp, out=out),
                          flush=flush)
            if mode == "fp64":
                ref = out.clone()
                e = np.zeros(1)
            else:
                e = err_rel(torch, out, ref)
            bound = None
            if mode in ("mixed", "mixed_bf16"):  # every cell against kernel_bounds' bound_v
                b, v64 = s.action_bounds(vd, wd, coef_kind=mp.CoefKind.sincosexp, want_v64=True)
                ev = (out.double() - v64).abs().amax(dim=1) / v64.abs().amax(dim=1)
                r = (ev / (4.0 * b[:, 0])).cpu().numpy()
                bound = {"max_err_over_S_bound_v": fin(r.max()), "cells_violating": int((r > 1.0).sum())}
                del b, v64
            lanes = 64.0 if mode == "fp64" else 128.0
            t_issue = 2.0 * pairs / (148 * lanes * clk) * 1e3
            res.append({"config": name, "mode": mode, "ms": ms, "cells_per_s": N_CELLS / (ms * 1e-3),
                        "launches": s.last_launch_count(),
                        "gflop_per_s": 2.0 * pairs / (ms * 1e-3) / 1e9,
                        "issue_roof_ms": t_issue, "issue_frac": t_issue / ms,
                        "hbm_bytes": N_CELLS * (96 + 8 * n_phi + out.element_size() * n_phi),
                        "max_err_rel_vs_fp64": fin(e.max()),
                        "max_err_over_u_s": fin(e.max() / UNIT_ROUNDOFF[int(cfg.u_s)]),
                        "bound_check": bound})
            del s, out
        del ref, wd
        torch.cuda.empty_cache()
    return res


def run_hex(mp, torch, dev, flush, hbm, tc_peak):
    """Hexahedral cells: the paper's 55,296-hex case size (48 x 48 x 24 jittered
    lattice, seed 1), Q1-Q3 Poisson and mass, mixed (fp16 storage, fp32 accumulation), constant
    coefficient; geometry at every Gauss-Legendre point in K1, the tets' tcgen05 GEMM in K2."""
    lv, lc = mp.structured_tet_mesh(48, 48, 24, 1.0, 0.15, 1)
    nx, ny, nz = 48, 48, 24
    ii, jj, kk = np.meshgrid(np.arange(nx), np.arange(ny), np.arange(nz), indexing="ij")
    base = (ii + (nx + 1) * (jj + (ny + 1) * kk)).transpose(2, 1, 0).reshape(-1)
    offs = np.array([(b & 1) + (nx + 1) * (((b >> 1) & 1) + (ny + 1) * ((b >> 2) & 1)) for b in range(8)])
    cells = (base[:, None] + offs[None, :]).astype(np.int32)
    dv = torch.from_numpy(lv).to(dev)
    dc = torch.from_numpy(cells).to(dev)
    n = cells.shape[0]
    res = []
    for form in (0, 1):
        for p in (1, 2, 3):
            cfg = mp.mode_config("mixed", form)
            s = mp.make_setup(p, cfg, cell_kind=1)
            s.reserve(n)
            out = torch.empty((n, s.n_phi ** 2), dtype=torch.float32, device=dev)
            ms = timed_ms(torch, lambda: s.cell_matrices(dv, dc, mp.CoefKind.one, out=out), reps=10, flush=flush)
            s.set_timing(True)
            s.cell_matrices(dv, dc, mp.CoefKind.one, out=out)
            t = s.last_timings()
            s.set_timing(False)
            nd = 3 if form else 1
            f_cell = 2.0 * s.n_phi ** 2 * s.n_q * nd * nd
            b_cell = 8 * 3 * 4 + 4 * s.n_phi ** 2  # vertex ids + output (mesh-indexed)
            t_roof = max(f_cell * n / (tc_peak * 1e12), b_cell * n / (hbm * 1e9)) * 1e3
            res.append({"form": "poisson" if form else "mass", "p": p, "n_phi": s.n_phi, "cells": n,
                        "ms": ms, "cells_per_s": n / (ms * 1e-3), "k1_ms": t[0] if t else None,
                        "k2_ms": t[1] if len(t) > 1 else None,
                        "tflops_dense_equiv": f_cell * n / (ms * 1e-3) / 1e12,
                        "roofline_frac": t_roof / ms, "path": s.path})
            del s, out
            torch.cuda.empty_cache()
    return res


def run_robustness(mp, torch, dev):
    """BASELINE config 3: 65,536 anisotropic rotated tets, c = 10^(6 u(x)) with u affine per
    cell; P1-P6 mass and Poisson in fp16 and mixed (fp16 and bf16 storage): max per-cell error
    against the device fp64 mode, and over the storage unit roundoff."""
    verts, coef = mp.gen_tets(1, 1, N_CELLS)
    vd = torch.from_numpy(verts).to(dev)
    cd = torch.from_numpy(coef).to(dev)
    res = []
    for p in range(1, 7):
        for form in (0, 1):
            s64 = mp.make_setup(p, mp.mode_config("fp64", form))
            a64 = s64.cell_matrices(vd, None, mp.CoefKind.exp10_affine, cd)
            for mode in ("fp16", "mixed", "mixed_bf16"):
                cfg = mp.mode_config(mode, form)
                s = mp.make_setup(p, cfg)
                a, fl = s.cell_matrices(vd, None, mp.CoefKind.exp10_affine, cd, want_flags=True)
                e = err_rel(torch, a, a64)
                res.append({"p": p, "form": "poisson" if form else "mass", "mode": mode,
                            "max_err_rel": fin(e.max()), "median_err_rel": fin(np.median(e)),
                            "max_err_over_u_s": fin(e.max() / UNIT_ROUNDOFF[int(cfg.u_s)]),
                            "fp_flags": int(fl)})
                del s, a
            del s64, a64
            torch.cuda.empty_cache()
    return res


def max_over_ranks(torch, value, dev):
    import torch.distributed as dist
    on_cpu = dist.get_backend() == "gloo"
    t = torch.tensor([value], dtype=torch.float64, device="cpu" if on_cpu else dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def run_assembly(mp, torch, dev, rank, world, degrees=(2, 3), n=96):
    """BASELINE config 4: 96^3 hexes x 6 tets, Poisson with c(x), mixed (bf16 storage)
    cell kernels, deterministic CSR assembly (row pull) in fp32 and fp64. One GPU: the global pattern and
    pos_map; N GPUs: the partitioned z-slab assembly (per-rank numbering, pattern and plan of the
    slab + one halo layer, interface partial sums sent up). CUDA-event times, max over ranks."""
    from paper_2410_12614_b200 import assembly as am
    from paper_2410_12614_b200 import distributed as D
    hbm = peaks()[0]
    verts, cells = mp.structured_tet_mesh(n, n, n, 1.0, 0.15, 1)
    vd = torch.from_numpy(verts).to(dev)
    cdev = torch.from_numpy(cells).to(dev)
    cpl = 6 * n * n
    cb, ce = D.slab_cell_range(rank, world, n, cpl)
    out = []

    def timed(fn, reps=3):
        fn()
        torch.cuda.synchronize()
        if world > 1:
            torch.distributed.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            r = fn()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        if world > 1:
            ms = max_over_ranks(torch, ms, dev)
        return ms, r

    for p in degrees:
        s = mp.make_setup(p, mp.mode_config("mixed_bf16", mp.FormKind.poisson))
        s.reserve(ce - cb)
        local = torch.empty((ce - cb, nphi(p), nphi(p)), dtype=torch.float32, device=dev)
        t_cell, _ = timed(lambda: s.cell_matrices(vd, cdev[cb:ce], mp.CoefKind.sincosexp, out=local.view(ce - cb, -1)))
        if world > 1:
            # partitioned: per-rank numbering of slab + halo layer, all-gather of the new-dof
            # counts, local-row / global-column pattern and plan, exchange plan (distributed.py)
            be = am.CudaPartitionBackend()
            t_part, part = timed(lambda: D.build_partition(be, p, cdev, verts.shape[0], rank, world, n, cpl), 1)
            res = {"p": p, "n_dofs": part.n_dofs, "nnz_rank": part.pat.nnz, "cells_per_rank": ce - cb,
                   "halo_cells": cb - part.halo_begin, "partition_setup_ms": t_part, "cell_kernels_ms": t_cell,
                   "interface_values_sent": int(part.send_pos.numel())}
            for fmt in (2, 3):
                vals = torch.empty(part.pat.nnz, dtype=torch.float32 if fmt == 2 else torch.float64, device=dev)
                t_asm, _ = timed(lambda: D.assemble_partition(be, part, local, fmt, values=vals))
                res[f"assemble_{'fp32' if fmt == 2 else 'fp64'}_ms"] = t_asm
                del vals
            res["kernels_plus_assembly_fp32_ms"] = t_cell + res["assemble_fp32_ms"]
            out.append(res)
            del local, part, s
            torch.cuda.empty_cache()
            continue
        t_dof, dm = timed(lambda: am.build_dofmap(p, cdev, verts.shape[0]), 1)
        t_pat, pat = timed(lambda: am.csr_pattern(dm), 1)
        res = {"p": p, "n_dofs": dm.n_dofs, "nnz": pat.nnz, "cells_per_rank": ce - cb,
               "dofmap_ms": t_dof, "csr_pattern_ms": t_pat, "cell_kernels_ms": t_cell}
        # deterministic (default): row pull over the incidence lists + pull_pos. Algorithmic bytes:
        # local matrices (4 B) + positions (2 B pull_pos, 4 B pos_map) once per local entry, the
        # incidence list (8 B per pair), CSR values written once, row/inc pointers
        for fmt in (2, 3):
            sv = 4 if fmt == 2 else 8
            vals = torch.empty(pat.nnz, dtype=torch.float32 if fmt == 2 else torch.float64, device=dev)
            t_asm, _ = timed(lambda: am.assemble_matrix(local, dm, pat, fmt, am.DETERMINISTIC, values=vals))
            del vals
            nb = (ce - cb) * (nphi(p) ** 2 * (4 + (2 if pat.pull_pos is not None else 4)) + 8 * nphi(p)) \
                + pat.nnz * sv + 16 * (dm.n_dofs + 1)
            key = "fp32" if fmt == 2 else "fp64"
            res[f"assemble_{key}_ms"] = t_asm
            res[f"assemble_{key}_hbm_frac"] = nb / (t_asm * 1e-3) / 1e9 / hbm
        vals = torch.empty(pat.nnz, dtype=torch.float32, device=dev)
        t_at, _ = timed(lambda: am.assemble_matrix(local, dm, pat, 2, am.ATOMIC, values=vals))
        res["assemble_atomic_fp32_ms"] = t_at
        res["kernels_plus_assembly_fp32_ms"] = t_cell + res["assemble_fp32_ms"]
        # cell kernels fused with the atomic scatter (K2 adds from TMEM, no locals in HBM)
        vals.zero_()
        t_fused, _ = timed(lambda: am.assemble_cells(s, vd, cdev, dm, pat, 2, mp.CoefKind.sincosexp,
                                                     accumulate=True, values=vals))
        res["fused_kernels_atomic_scatter_fp32_ms"] = t_fused
        del vals, pat
        torch.cuda.empty_cache()
        # the seg_ptr/perm segment-gather kernel (patterns built with deterministic_plan=True)
        t_pat2, pat = timed(lambda: am.csr_pattern(dm, deterministic_plan=True), 1)
        vals = torch.empty(pat.nnz, dtype=torch.float32, device=dev)
        t_plan, _ = timed(lambda: am.assemble_matrix(local, dm, pat, 2, am.DETERMINISTIC, values=vals))
        res["csr_pattern_with_segment_plan_ms"] = t_pat2
        res["assemble_segment_gather_fp32_ms"] = t_plan
        del vals
        out.append(res)
        del local, pat, dm, s
        torch.cuda.empty_cache()
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=300)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--sweep", action="store_true", help="add the config-2 p=1..8 sweep")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-assembly", action="store_true", help="skip the config-4 assembly key")
    ap.add_argument("--ref-seconds", type=float, default=10.0)
    ap.add_argument("--no-modes", action="store_true", help="skip the configs 0/1 precision-mode table")
    ap.add_argument("--robustness", action="store_true", help="add the config-3 error table")
    ap.add_argument("--no-action", action="store_true", help="skip the Algorithm-2 action table")
    ap.add_argument("--no-hex", action="store_true", help="skip the hexahedral-cell table")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return

    import torch
    import paper_2410_12614_b200 as mp

    backend = os.environ.get("MPFEM_DIST_BACKEND", "nccl")  # gloo: test ranks sharing a GPU
    if world > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local % max(1, torch.cuda.device_count()))
        dist.init_process_group(backend)
    dev = torch.device("cuda", local % max(1, torch.cuda.device_count()))
    torch.cuda.set_device(dev)
    hbm, tc_peak, tc_sus, peak_src = peaks()

    verts_np, _ = mp.gen_tets(0, 1 + rank, N_CELLS)
    verts_pinned = torch.from_numpy(verts_np).pin_memory()
    vd = verts_pinned.to(dev)
    cfg = mp.KernelConfig(form=mp.FormKind.poisson, **{k: v for k, v in MIXED_CFG.items()})
    setup = mp.make_setup(P_DEG, cfg)
    setup.reserve(N_CELLS)
    n2 = setup.n_phi ** 2
    out = torch.empty((N_CELLS, n2), dtype=torch.float32, device=dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream()

    def step():
        setup.cell_matrices(vd, None, mp.CoefKind.sincosexp, out=out)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()

    # ---- timed region: K steps, L2 flushed before each, CUDA events on the launch stream
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    k_ms = []
    sampler = ClockSampler(local)
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    sampler.start()
    time.sleep(0.05)
    for i in range(args.steps):
        flush.zero_()
        ev[i][0].record(stream)
        step()
        ev[i][1].record(stream)
        k_ms.append(None)
        if i % 16 == 15 or i == args.steps - 1:
            pass
    torch.cuda.synchronize()
    clocks = sampler.stop()
    if world > 1:
        torch.distributed.barrier()
    step_ms = [a.elapsed_time(b) for a, b in ev]
    total_ms = float(np.sum(step_ms))
    launches = setup.last_launch_count() * args.steps

    # per-kernel durations (CUDA events recorded by the library on the launch stream) on a
    # short re-run of identical steps with K1/K2 unoverlapped; the dominant kernel is K2
    setup.set_timing(True)
    k1, k2 = [], []
    for _ in range(20):
        flush.zero_()
        step()
        t = setup.last_timings()
        k1.append(t[0])
        k2.append(t[1])
    setup.set_timing(False)
    k1_ms, k2_ms = float(np.median(k1)), float(np.median(k2))

    if world > 1:
        total_ms = max_over_ranks(torch, total_ms, dev)
    ms_per_step = total_ms / args.steps
    value = world * N_CELLS / (ms_per_step * 1e-3)

    # ---- end to end through the public host-buffer API (pinned host memory)
    out_host = torch.empty((N_CELLS, setup.n_phi, setup.n_phi), dtype=torch.float32).pin_memory()
    out_host_np = out_host.numpy()
    verts_host_np = verts_pinned.numpy()
    e2e_steps = max(3, min(args.steps, 20))
    setup.cell_matrices_host(verts_host_np, None, mp.CoefKind.sincosexp, out=out_host_np)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(e2e_steps):
        setup.cell_matrices_host(verts_host_np, None, mp.CoefKind.sincosexp, out=out_host_np)
    e1.record(stream)
    torch.cuda.synchronize()
    e2e_ms = e0.elapsed_time(e1) / e2e_steps
    if world > 1:
        e2e_ms = max_over_ranks(torch, e2e_ms, dev)
    e2e_value = world * N_CELLS / (e2e_ms * 1e-3)

    # ---- accuracy of the timed output against the device fp64 mode (u_p = u_g = u_q = u_s =
    # fp64, the path pinned to the fp64 oracle by tests/test_gpu_cells.py) on the same cells
    s64 = mp.make_setup(P_DEG, mp.KernelConfig(form=mp.FormKind.poisson))
    a64 = s64.cell_matrices(vd, None, mp.CoefKind.sincosexp)
    step()
    torch.cuda.synchronize()
    diff = (out.view(N_CELLS, -1).double() - a64.view(N_CELLS, -1)).abs().amax(dim=1)
    err = (diff / a64.view(N_CELLS, -1).abs().amax(dim=1)).cpu().numpy()
    del a64, s64, diff
    u_s = 2.0 ** -11  # fp16 unit roundoff
    # every cell against its own a-priori bound: kernel_bounds (bounds.cpp:29-281) on the GPU
    # (bitwise the reference's for nodal/constant coefficients, tests/test_gpu_bounds.py)
    torch.cuda.synchronize()
    tb0 = time.perf_counter()
    bnd, a_exact = setup.cell_bounds(vd, coef_kind=mp.CoefKind.sincosexp, want_a64=True)
    torch.cuda.synchronize()
    bound_ms = (time.perf_counter() - tb0) * 1e3
    e_exact = (out.view(N_CELLS, -1).double() - a_exact.view(N_CELLS, -1)).abs().amax(dim=1) / \
        a_exact.view(N_CELLS, -1).abs().amax(dim=1)
    ratio = (e_exact / (4.0 * bnd[:, 0])).cpu().numpy()  # S = 4: u_s coarser than u_p, u_g, u_q
    bound_check = {"cells": N_CELLS, "max_err_over_S_bound_a": float(ratio.max()),
                   "median_err_over_S_bound_a": float(np.median(ratio)),
                   "cells_violating": int((ratio > 1.0).sum()), "S": 4,
                   "bound_kernel_ms": bound_ms,
                   "note": "err vs the exact binary64 A of kernel_bounds, per cell, all cells"}
    del a_exact, bnd
    accuracy = {"vs": "device fp64 mode (oracle-pinned), same cells",
                "metric": "per-cell max|A - A64| / max|A64| (errorlab.cpp:90-99)",
                "max_err_rel": float(err.max()), "median_err_rel": float(np.median(err)),
                "max_err_over_u_s": float(err.max() / u_s), "u_s": "fp16"}

    f_cell, b_cell = work_per_cell(P_DEG, 1, 4)
    flops_launch = N_CELLS * f_cell
    achieved_tflops = flops_launch / (k2_ms * 1e-3) / 1e12
    executed = 2.0 * N_CELLS * setup.k * n2  # packed (s<=t) depth actually run
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "fp16 storage / fp32 accumulate",
        "data": "synthetic (seeded tets, gen kind 0, seed 1+rank)",
        "config": workload_config(),
        "tflops_dense_equiv": N_CELLS * world * f_cell / (ms_per_step * 1e-3) / 1e12,
        "kernels_ms": {"geom_w": k1_ms, "cellmat_tc": k2_ms},
        "roofline": {"bound": "tensor", "achieved": achieved_tflops, "peak": tc_peak,
                     "unit": "TFLOP/s", "frac": achieved_tflops / tc_peak,
                     "traffic": (lambda t: t["bytes"] if t else None)(profiled_traffic()),
                     "traffic_source": (lambda t: t["source"] if t else None)(profiled_traffic()),
                     "algorithmic_bytes": N_CELLS * b_cell,
                     "kernel": "cellmat_tc2_kernel",
                     "note": (f"achieved = dense-equivalent F_cell {f_cell:.0f} flop x {N_CELLS} cells / "
                              f"K2 duration; peak = {peak_src} bf16 burst; the kernel executes the "
                              f"(s<=t)-packed depth, {executed / flops_launch:.3f} of F_cell"),
                     "executed_flop_fraction": executed / flops_launch,
                     "step_hbm_frac": (N_CELLS * b_cell / (ms_per_step * 1e-3) / 1e9) / hbm},
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": int(verts_np.nbytes),
                "d2h_bytes_per_step": int(out_host_np.nbytes), "ms_per_step": e2e_ms},
        "gpu_launches": launches,
        "clocks": clocks,
        "accuracy": accuracy,
        "bound_check": bound_check,
    }
    if not args.no_assembly:
        line["assembly"] = {"workload": "config4: 96^3 x 6 tets, poisson P2/P3, mixed-bf16 kernels, "
                                        "deterministic CSR, partitioned z-slabs over ranks",
                            "results": run_assembly(mp, torch, dev, rank, world)}
    if not args.no_modes and rank == 0:
        line["modes"] = run_modes(mp, torch, dev, flush)
    if not args.no_action and rank == 0:
        line["action"] = {"workload": "configs 0/1 as action_kernel (Algorithm 2): 65536 P4 tets, "
                                      "c(x) at quadrature points, one random w per cell",
                          "results": run_action(mp, torch, dev, flush, clocks.get("sm_max_mhz") or 1965.0)}
    if not args.no_hex and rank == 0:
        line["hex"] = {"workload": "55,296 jittered hexes (48x48x24 lattice), Q1-Q3, mixed, constant c",
                       "results": run_hex(mp, torch, dev, flush, hbm, tc_peak)}
    if args.robustness and rank == 0:
        line["robustness"] = run_robustness(mp, torch, dev)
    if args.sweep and rank == 0:
        line["sweep"] = run_sweep(mp, torch, dev)
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cfg_t = (MIXED_CFG["u_p"], MIXED_CFG["u_g"], MIXED_CFG["u_q"], MIXED_CFG["u_s"], MIXED_CFG["engine"])
        r, kind, cores, sample = cpu_baseline(P_DEG, 1, cfg_t, verts_np, 1, target_s=args.ref_seconds)
        line["cpu_baseline"] = {"value": r, "unit": UNIT, "cores": cores, "kind": kind, "sample": sample}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
