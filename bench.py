"""Benchmark: DoFs/s per matrix-free Laplace apply (3D Q_k, FP64) on B200.

A "step" is one mf_apply -- the whole per-apply hot path of SURVEY.md §8(a)
(a3 gather .. a7 scatter + Dirichlet identity, and the a8 halo exchange when
N > 1) -- over one synthetic input vector.  Setup rows (a1 tables, a2 geometry,
a9 diagonal) run once before timing; a10 (the solver) is measured by
``--solve``.  Workload at N = 1: BASELINE.json configs[2], Q4 on a 64^3 unit
cube, affine, c = 1, Dirichlet on all faces (16,974,593 DoFs); src + dst =
272 MB > 126 MB L2, so every timed apply streams from HBM.  N > 1 (torchrun):
BASELINE.json configs[4], the 256^3 Q4 cube (1,076,890,625 DoFs) split into N
z-slabs (strong scaling, "scaling": "strong"), the shared planes exchanged with
NCCL; its single-GPU point is `--gpus 1 --config cfg5q4`.  The small configs
(cfg2/3/4, dg4, hex3) scale weakly when run on N > 1 (64 z-layers per rank).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl mf|reference]
                  [--config cfg3|cfg4|cfg2|cfg5q4|cfg5q6|dg4|hex3] [--solve]
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

# strong-scaling configs: the global mesh is fixed and split into N z-slabs (configs[4])
STRONG = {"cfg5q4", "cfg5q6"}
CONFIGS = {
    # name: (n_cells (per rank: z multiplied by N, unless strong), degree, geometry, coeff, description)
    "cfg3": ((64, 64, 64), 4, "cartesian", 1.0, "3D Laplace Q4 on 64^3 cube (~17M DoFs), affine, c=1"),
    "cfg4": ((64, 64, 64), 3, "sine", "variable", "3D variable-coefficient Laplace Q3 on deformed 64^3 cube, stored metric"),
    "cfg2": ((16, 16, 16), 2, "cartesian", 1.0, "3D Laplace Q2 on 16^3 affine cube"),
    "cfg5q4": ((256, 256, 256), 4, "cartesian", 1.0, "3D Laplace Q4 on 256^3 cube (~1.08B DoFs)"),
    "cfg5q6": ((256, 256, 256), 6, "cartesian", 1.0, "3D Laplace Q6 on 256^3 cube (~3.6B DoFs)"),
    # §8(f) f4: the discretization the paper's §6.1 experiment times
    "dg4": ((64, 64, 64), 4, "dg", 1.0, "3D Laplace, symmetric interior penalty DG Q4 on 64^3 cube (~32.8M DoFs)"),
    # §8(f) f3: general unstructured hex input (jittered trilinear cells, rotated local frames,
    # shuffled vertex numbers; DoFs numbered by mf_hex_number_dofs), variable coefficient
    "hex3": ((64, 64, 64), 3, "hex", "variable",
             "3D variable-coefficient Laplace Q3 on an unstructured 64^3-cell hex mesh (trilinear, jitter 0.2h)"),
}
METRIC = "DoFs/s per matrix-free Laplace apply (3D Q_k FP64)"


def lib_build():
    """sha1 (12 hex) of the library this run loads (matches profiles/traffic.json "build")."""
    import hashlib

    from paper_1910_13247_b200 import build as _b

    try:
        with open(os.environ.get("MF_LIB_PATH") or _b.LIB, "rb") as f:
            return hashlib.sha1(f.read()).hexdigest()[:12]
    except Exception:
        return None


def load_traffic(config):
    """ncu-measured DRAM bytes per launch of the timed region (profiles/traffic.json) with the
    profile files and the build they came from, or None."""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            e = json.load(f)[config]
        return e["bytes_per_launch"], {"source": e.get("source"), "build": e.get("build")}
    except Exception:
        return None, None


FP64_PEAK_TINSTR = 57.47 * 148 * 1.965e9 / 1e12  # measured DFMA issue rate (profiles/r01_microbench.json)
# measured DMMA m8n8k4 f64 rate: 18.5 T FMA/s = 72.3 G DMMA/s, sharing the FP64 pipe additively
# with DFMA (tools/micro/dmma_lat.cu, profiles/r02_dmma_microbench.txt)
DMMA_PEAK_G = 18.5e12 / 256 / 1e9


def fp64_roofline(config, n_dofs, kernel_ms):
    """FP64-pipe view of the same region: ncu-counted FP64 instructions per DoF
    (profiles/traffic.json) over the live kernel time, against the measured DFMA rate."""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            e = json.load(f)[config]
        ipd = e["fp64_instr_per_dof"]
    except Exception:
        return None
    achieved = ipd * n_dofs / (kernel_ms * 1e-3) / 1e12
    t_min = ipd * n_dofs / (FP64_PEAK_TINSTR * 1e12) * 1e3
    out = {"instr_per_dof": ipd, "achieved": achieved, "peak": FP64_PEAK_TINSTR, "unit": "T FP64 instr/s",
           "frac": achieved / FP64_PEAK_TINSTR, "t_min_ms": t_min}
    if e.get("dmma_per_dof"):  # tensor-core kernels: DMMA time on the same FP64 pipe
        t_dmma = e["dmma_per_dof"] * n_dofs / (DMMA_PEAK_G * 1e9) * 1e3
        out.update({"dmma_per_dof": e["dmma_per_dof"], "dmma_min_ms": t_dmma, "t_min_ms": t_min + t_dmma,
                    "pipe_frac": (t_min + t_dmma) / kernel_ms})
    return out


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return d["hbm_gbs"], "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """NVML samples of SM clock and throttle reasons during the timed region."""

    REASONS = {
        0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
        0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
        0x100: "display_clock_setting",
    }

    def __init__(self, device_index: int):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device_index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            # the first queries on a fresh box are slow; pay them before the timed region
            pynvml.nvmlDeviceGetClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            pynvml.nvmlDeviceGetCurrentClocksEventReasons(self.h)
        except Exception:
            self.nv = None

    def _run(self):
        while not self._stop.is_set():
            self.sample()
            time.sleep(0.0005)

    def sample(self):
        if self.nv is None:
            return
        try:
            self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
            r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
            for bit, name in self.REASONS.items():
                if r & bit and name != "gpu_idle":
                    self.reasons.add(name)
        except Exception:
            pass

    def __enter__(self):
        self.t = threading.Thread(target=self._run, daemon=True)
        self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self.t.join()

    def summary(self):
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons), "samples": len(self.samples)}


def _hex_oracle_matrix(cells, degree, coeff):
    """oracle/hex.py assembly on a cells^3 sub-mesh of the hex3 recipe (coordinate numbering)."""
    import synth
    from oracle import hex as ohex

    V, C = synth.hex_mesh((cells,) * 3, jitter=0.2, seed=0)
    cd, coords = ohex.number_by_coordinates(ohex.support_points(V, C, degree))
    dirichlet = ohex.boundary_dofs(coords, (0.0,) * 3, (1.0,) * 3)
    S = ohex.assemble(V, C, degree, cd, len(coords), dirichlet=dirichlet,
                      coeff="variable" if coeff == "variable" else "constant",
                      value=1.0 if coeff == "variable" else coeff)
    return S, len(coords)


def make_hex_operator(nc, k, coeff, device):
    """hex3: the synthetic unstructured mesh, numbered by the library (mf_hex_number_dofs)."""
    import numpy as np

    import synth
    from paper_1910_13247_b200 import HexOperator, hex_number_dofs

    V, C = synth.hex_mesh(nc, jitter=0.2, seed=0)
    cd, n, bnd = hex_number_dofs(C, k)
    dirichlet = np.nonzero(bnd)[0]
    return HexOperator(V, C, k, cd, n, (), dirichlet, coeff=coeff, device=device), dirichlet


def cpu_baseline_one_core(degree, geometry, coeff):
    """The same oracle SpMV on one host core (OMP_NUM_THREADS=1, fresh process), best of 5."""
    # k >= 5: an 8^3 sub-brick (the 16^3 assembly alone is ~300 core-seconds for Q6)
    cells = 8 if degree >= 5 else 16
    code = (f"import bench, json; v, nd, reps, el, ta, c = bench.cpu_baseline_sample({degree}, {geometry!r}, "
            f"{coeff!r}, seconds=5.0, cells={cells}); print(json.dumps([v, nd, c]))")
    env = dict(os.environ, OMP_NUM_THREADS="1")
    try:
        r = subprocess.run([sys.executable, "-c", code], cwd=ROOT, env=env, capture_output=True, text=True,
                           timeout=120)
        v, nd, c = json.loads(r.stdout.strip().splitlines()[-1])
        return {"value": v, "unit": "DoFs/s", "cores": c,
                "sample": f"{cells}^3-cell sub-brick, {nd} DoFs, best of 5 repeats of ~1 s"}
    except Exception as e:  # the baseline is context; never fail the bench line on it
        return {"value": None, "error": str(e)[:200]}


def cpu_baseline_sample(degree, geometry, coeff, seconds=10.0, cells=16):
    """The oracle as it stands (C/OpenMP CSR assembly + SpMV) on a bounded
    sample of the workload: the same element type and geometry on a cells^3
    sub-brick; SpMV repeated for ~`seconds` in 5 repeats, the best repeat's rate
    returned.  Returns DoFs/s and a description."""
    import numpy as np

    import oracle
    import synth

    t0 = time.perf_counter()
    if geometry == "hex":  # the unstructured-hex oracle's assembled matrix (scipy CSR SpMV)
        cells = min(cells, 6)
        S, n = _hex_oracle_matrix(cells, degree, coeff)
        mv = lambda x, y: y.__setitem__(slice(None), S @ x)  # noqa: E731
    elif geometry == "dg":  # the DG oracle's assembled matrix (scipy CSR SpMV)
        from oracle import dg

        cells = min(cells, 8)
        S = coeff * dg.assemble((cells,) * 3, degree)
        n = S.shape[0]
        mv = lambda x, y: y.__setitem__(slice(None), S @ x)  # noqa: E731
    else:
        p = oracle.problem(dim=3, n_cells=(cells,) * 3, degree=degree, geom=1 if geometry == "sine" else 0,
                           coeff_kind=1 if coeff == "variable" else 0,
                           coeff_value=1.0 if coeff == "variable" else coeff)
        A = oracle.CSR(p)
        n = A.n
        mv = A.matvec
    t_asm = time.perf_counter() - t0
    x = synth.vector(n, 0)
    y = np.empty_like(x)
    mv(x, y)
    best, reps_all, el_all = 0.0, 0, 0.0
    for _ in range(5):
        reps, t0 = 0, time.perf_counter()
        while True:
            mv(x, y)
            reps += 1
            el = time.perf_counter() - t0
            if el >= seconds / 5:
                break
        best = max(best, n * reps / el)
        reps_all += reps
        el_all += el
    return best, n, reps_all, el_all, t_asm, oracle.num_threads()


def run_reference(args, cfg):
    """--impl reference: the oracle timed as it stands on the host cores."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    nc, k, geom, coeff, desc = CONFIGS[cfg]
    import numpy as np

    import oracle
    import synth

    cells = 16
    if geom == "hex":
        cells = 6
        S, n = _hex_oracle_matrix(cells, k, coeff)
        mv = lambda x, y: y.__setitem__(slice(None), S @ x)  # noqa: E731
    elif geom == "dg":  # the DG oracle's assembled SIP matrix
        from oracle import dg

        cells = 8
        S = coeff * dg.assemble((cells,) * 3, k)
        n = S.shape[0]
        mv = lambda x, y: y.__setitem__(slice(None), S @ x)  # noqa: E731
    else:
        p = oracle.problem(dim=3, n_cells=(cells,) * 3, degree=k, geom=1 if geom == "sine" else 0,
                           coeff_kind=1 if coeff == "variable" else 0,
                           coeff_value=1.0 if coeff == "variable" else coeff)
        A = oracle.CSR(p)
        n = A.n
        mv = A.matvec
    x = synth.vector(n, 0)
    y = np.empty_like(x)
    for _ in range(args.warmup):
        mv(x, y)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        mv(x, y)
    el = time.perf_counter() - t0
    v = n * args.steps / el
    sample = f"oracle CSR SpMV (assembled by full Gauss quadrature) of the same Q{k} operator on a {cells}^3 sub-{'mesh' if geom == 'hex' else 'brick'} ({n} DoFs), one SpMV per step"
    world = int(os.environ.get("WORLD_SIZE", "1"))
    ncw = nc if cfg in STRONG else (nc[0], nc[1], nc[2] * world)
    n_full = (ncw[0] * ncw[1] * ncw[2] * (k + 1) ** 3 if geom == "dg"
              else (k * ncw[0] + 1) * (k * ncw[1] + 1) * (k * ncw[2] + 1))
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": v, "unit": "DoFs/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * el / args.steps, "higher_is_better": True,
        "scaling": "strong" if cfg in STRONG else "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": desc, "config": cfg, "n_cells": list(ncw), "degree": k, "n_dofs": n_full,
                   "geometry": geom, "coeff": coeff, "parallelism": f"zslab{world}", "sample": sample},
        "cpu_baseline": {"value": v, "unit": "DoFs/s", "cores": oracle.num_threads(), "kind": "oracle", "sample": sample},
        "e2e": {"value": v, "unit": "DoFs/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="mf", choices=["mf", "reference"])
    ap.add_argument("--config", default=None, choices=sorted(CONFIGS),
                    help="default: cfg3 on one GPU, cfg5q4 (strong scaling) on N > 1")
    ap.add_argument("--variant", default="auto")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--solve", action="store_true", help="also time one Chebyshev(6)-PCG solve")
    ap.add_argument("--solve-mg", action="store_true", help="also time one multigrid-preconditioned CG solve (1 GPU)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.config is None:
        args.config = "cfg3" if int(os.environ.get("WORLD_SIZE", str(args.gpus))) == 1 else "cfg5q4"
    strong = args.config in STRONG
    if args.impl == "reference":
        return run_reference(args, args.config)

    import numpy as np
    import torch
    import torch.distributed as dist

    import synth
    from paper_1910_13247_b200 import Operator

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    group = None
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        group = dist.group.WORLD
    nc, k, geom, coeff, desc = CONFIGS[args.config]
    if not strong:
        nc = (nc[0], nc[1], nc[2] * world)
    hex_dir = None
    if geom == "dg":
        if world > 1:
            raise SystemExit("the DG operator runs on one rank")
        op = Operator(nc, k, coeff=coeff, device=local, discretization="dg")
    elif geom == "hex":
        if world > 1:
            raise SystemExit("the unstructured hex operator runs on one rank")
        op, hex_dir = make_hex_operator(nc, k, coeff, local)
    else:
        op = Operator(nc, k, geometry=geom, coeff=coeff, group=group, device=local)
        op.set_variant(args.variant)
    n = op.n_local
    src = torch.from_numpy(synth.uniform(op.first_global, n, 0)).cuda()
    dst = torch.empty_like(src)
    stream = torch.cuda.current_stream()

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    for _ in range(args.warmup):
        op.apply(src, dst)
    barrier()
    info0 = op.info()
    clocks = ClockSampler(local)
    start, stop = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    op.kernel_timing(True)
    with clocks:
        barrier()
        start.record(stream)
        for _ in range(args.steps):
            op.apply(src, dst)
        stop.record(stream)
        barrier()
    op.kernel_timing(False)
    info1 = op.info()
    ms = start.elapsed_time(stop)
    kern_ms, kern_n = op.kernel_time()
    t = torch.tensor([ms, kern_ms / max(kern_n, 1)], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max, kern_avg_ms = t[0].item(), t[1].item()
    ms_per_step = ms_max / args.steps
    value = op.n_global * args.steps / (ms_max * 1e-3)
    launches = (info1["kernel_launches"] - info0["kernel_launches"])

    # end to end through the public C ABI with pinned host buffers (H2D + apply + D2H each step)
    hs = torch.from_numpy(synth.uniform(op.first_global, n, 0)).pin_memory()
    hd = torch.empty_like(hs).pin_memory()
    e2e_steps = max(3, min(args.steps, 20 if n < 200_000_000 else 3))
    op.apply_host_ptr(hs.data_ptr(), hd.data_ptr())
    barrier()
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        op.apply_host_ptr(hs.data_ptr(), hd.data_ptr())
    barrier()
    e2e_s = torch.tensor([time.perf_counter() - t0], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(e2e_s, op=dist.ReduceOp.MAX)
    e2e_val = op.n_global * e2e_steps / e2e_s.item()
    # parity spot check of the timed output (cheap invariant: identity rows)
    if geom == "hex":
        di = torch.from_numpy(hex_dir).cuda()
        ok = bool(torch.equal(dst[di], src[di]))
    else:
        ok = (bool(torch.equal(dst[:op.mesh.n_cells[0] * k + 1], src[:op.mesh.n_cells[0] * k + 1]))
              if rank == 0 and geom != "dg" else True)  # (DG has no identity rows)

    solve = None
    solve_mg = None
    if args.solve:
        b = torch.ones(n, dtype=torch.float64, device="cuda")
        op.cg_solve(b, rel_tol=1e-10)  # warm-up (diagonal, scratch; both solves below are timed warm)
        barrier()
        t0 = time.perf_counter()
        x, res = op.cg_solve(b, rel_tol=1e-10)
        barrier()
        solve = {"iterations": res.iterations, "seconds": time.perf_counter() - t0, "lambda_max": res.lambda_max}
        if world == 1 and geom in ("cartesian", "sine"):  # FP32 Chebyshev inside the FP64 CG (§8(f) f2)
            op.cg_solve(b, rel_tol=1e-10, precision="mixed")  # (allocates the FP32 buffers)
            barrier()
            t0 = time.perf_counter()
            x, res = op.cg_solve(b, rel_tol=1e-10, precision="mixed")
            barrier()
            solve["mixed"] = {"iterations": res.iterations, "seconds": time.perf_counter() - t0,
                              "final_rel_residual": res.final_rel_residual}
    if args.solve_mg and world == 1:
        from paper_1910_13247_b200 import Multigrid

        b = torch.ones(n, dtype=torch.float64, device="cuda")
        solve_mg = {}
        for prec in ("fp64", "mixed"):  # mixed: FP32 V-cycle in the FP64 CG (§8(f) f2)
            t0 = time.perf_counter()
            M = Multigrid(nc, k, geometry=geom, coeff=coeff, precision=prec)
            torch.cuda.synchronize()
            t_setup = time.perf_counter() - t0
            M.cg_solve(b, rel_tol=1e-10)  # warm-up
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            x, res = M.cg_solve(b, rel_tol=1e-10)
            torch.cuda.synchronize()
            t_solve = time.perf_counter() - t0
            ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            ev0.record()
            for _ in range(5):
                M.vcycle(b, x)
            ev1.record()
            torch.cuda.synchronize()
            solve_mg[prec] = {"levels": M.n_levels, "level_sizes": M.sizes, "iterations": res.iterations,
                              "final_rel_residual": res.final_rel_residual, "seconds": t_solve,
                              "setup_seconds": t_setup, "vcycle_ms": ev0.elapsed_time(ev1) / 5}
            M.close()

    if rank == 0:
        peak, peak_kind = load_peaks()
        bytes_per_launch = info1["bytes_algorithmic"]
        achieved = bytes_per_launch / (kern_avg_ms * 1e-3) / 1e9
        traffic, traffic_src = load_traffic(args.config)
        build = lib_build()
        fp64 = fp64_roofline(args.config, op.n_local, kern_avg_ms)
        # the binding roof: the larger of the HBM time of the algorithmic bytes and the FP64 time of
        # the counted instructions; frac below stays the north star's % of HBM
        t_hbm = bytes_per_launch / (peak * 1e9) * 1e3
        binding = {"hbm_min_ms": t_hbm, "fp64_min_ms": fp64["t_min_ms"] if fp64 else None,
                   "roof": "hbm" if not fp64 or t_hbm >= fp64["t_min_ms"] else "fp64",
                   "frac_of_binding": max(t_hbm, fp64["t_min_ms"] if fp64 else 0.0) / kern_avg_ms}
        out = {
            "metric": METRIC, "value": value, "unit": "DoFs/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "strong" if strong else "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": desc, "config": args.config, "n_cells": list(nc), "degree": k,
                       "n_dofs": op.n_global, "geometry": geom, "coeff": coeff, "parallelism": f"zslab{world}",
                       "apply_variant": info1["apply_variant"],
                       "l2": f"inputs larger than L2: {info1['bytes_algorithmic'] / 1e6:.0f} MB streamed per apply (src, dst, stored metric / indices) > 126 MB"},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic, "peak_kind": peak_kind,
                         "traffic_source": traffic_src,
                         "traffic_build_matches": bool(traffic_src and build and traffic_src.get("build") == build),
                         "build": build, "bytes_per_launch": bytes_per_launch, "kernel_ms": kern_avg_ms,
                         "kernel_share_of_step": kern_avg_ms / ms_per_step, "fp64": fp64, "binding": binding},
            "e2e": {"value": e2e_val, "unit": "DoFs/s", "h2d_bytes_per_step": 8 * n, "d2h_bytes_per_step": 8 * n,
                    "steps": e2e_steps},
            "gpu_launches": launches,
            "clocks": clocks.summary(),
            "identity_rows_exact": ok,
        }
        if solve:
            out["solve"] = solve
        if solve_mg:
            out["solve_mg"] = solve_mg
        if not args.no_cpu_baseline and world == 1:
            # all host cores and one core, best of 5 repeats each
            v, nd, reps, el, t_asm, cores = cpu_baseline_sample(k, geom, coeff)
            one = cpu_baseline_one_core(k, geom, coeff)
            out["cpu_baseline"] = {"value": v, "unit": "DoFs/s", "cores": cores, "kind": "oracle",
                                   "sample": f"oracle CSR SpMV of the same Q{k} operator on a sub-{'mesh' if geom == 'hex' else 'brick'} ({nd} DoFs), best of 5 repeats of ~2 s ({reps} SpMVs in {el:.1f} s in total; assembly {t_asm:.1f} s not timed)",
                                   "one_core": one}
        print(json.dumps(out))
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
