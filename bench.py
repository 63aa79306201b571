"""Benchmark: NystromNGD steps/sec on B200 (BASELINE.json metric) + evidence.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2] [--impl ours|reference]

Workload (default, BASELINE.json configs[1] = "C2"): 2D Poisson, MLP
2-64-64-64-1 tanh (p = 8577), fp64, 4096 interior + 512 boundary points,
Nystrom rank l = 300 (fixed), 50 PCG iterations per step (kappa = 1e-300 so
PCG runs to maxit unless it breaks down), mu floor
1e-6 * ||grad L||.  One bench "step" = one NGD iteration: linearise + gradient
+ l-column sketch + Nystrom factorisation + PCG + Armijo line search + update.

value     : NGD steps/s, device-timed (CUDA events around each step on the
            compute stream, L2 flushed between steps outside the events,
            inputs resident in HBM), max over ranks.
e2e       : the same metric through the public API (nystrom_ngd_run) with
            HOST numpy inputs every step (theta0 + quadrature uploaded,
            theta + records read back), wall clock.
roofline  : the dominant kernel class of the step, timed live inside the
            timed region by CUDA events around each of its launches.
cpu_baseline / --impl reference : the CPU oracle (numpy restatement of the
            reference, oracle/ngd_oracle.py) on a bounded sample of the same
            workload, extrapolated to one NGD step.
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

CONFIGS = {
    # name: widths, kind, n_int, n_bnd, ell, cg_maxit
    "c1": ((2, 32, 32, 1), "sin2d", 900, 120, 100, 20),
    "c2": ((2, 64, 64, 64, 1), "sin2d", 4096, 512, 300, 50),
    "c3": ((5, 128, 128, 128, 1), "sinsum", 16384, 4096, 500, 100),
    "c4": ((2, 256, 256, 256, 1), "lap", 65536, 0, 512, 20),
    "c5": ((10, 256, 256, 256, 256, 1), "gauss", 131072, 16384, 1000, 100),
}
KIND_NAMES = {1: "jet_fwd", 2: "jet_rev", 3: "gram_phaseA", 4: "gram_phaseB", 5: "jacobian_rows", 6: "precond",
              7: "vector", 8: "pack", 9: "jacobi_svd", 10: "cholesky", 11: "cublas", 12: "cusolver", 13: "trsm", 14: "fused_matvec"}
OWN_KINDS = tuple(range(1, 11)) + (13, 14)  # our kernels; 11/12 are library calls (reported, never the roofline kernel)


def load_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    peaks = {"hbm_gbs": 6650.0, "source": "fallback (B200_PROFILING.md)"}
    if os.path.exists(path):
        with open(path) as f:
            d = json.load(f)
        peaks["hbm_gbs"] = float(d.get("hbm_gbs", 6650.0))
        peaks["source"] = "MEASURED_PEAKS.json"
    # FP64 peak: not in MEASURED_PEAKS.json; measured on this pool's B200 by
    # tools/probe/fp64_peak.cu (profiles/r01_fp64_peak.txt): DMMA m16n8k16 36.99 TF/s,
    # DFMA 36.63 TF/s, cuBLAS DGEMM 8192^3 35.45 TF/s.
    peaks["fp64_tflops"] = 36.99
    return peaks


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = "clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown," \
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown," \
             "clocks_event_reasons.sw_power_cap"

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "20"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                smax = float(parts[1])
            except ValueError:
                continue
            for nm, val in zip(names, parts[3:7]):
                if val.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": smax, "reasons": sorted(reasons),
                "samples": len(sm)}


def make_problem(ngd, name, world=1, rank=0):
    widths, kind, n_int, n_bnd, ell, maxit = CONFIGS[name]
    top = ngd.MlpTopology(widths)
    if kind == "sin2d":
        prob = ngd.Poisson2D(top)
    elif kind == "lap":
        prob = ngd.LaplacianStack(top)
    else:
        prob = ngd.PoissonND(top, kind)
    # weak scaling: every rank carries the single-GPU point count
    quad = prob.sample_quadrature(n_int * world, n_bnd * world, 0)
    theta0 = ngd.init(top, 0).values
    cfg = ngd.NystromNgdConfig(ell0=ell, ell_max=ell, cg_maxit=maxit, kappa=1e-300, mu_floor_mode="grad-power",
                               mu_floor_coeff=1e-6, mu_floor_exponent=1.0, iterations=1, seed=0, fixed_rank=True,
                               omega_source="device")
    return prob, quad, theta0, cfg


# ---------------------------------------------------------------------------
# CPU baseline: the oracle on a bounded sample, extrapolated to one NGD step
# ---------------------------------------------------------------------------


def cpu_step_sample(name, n_mv=6):
    """Seconds for one NGD step of the CPU oracle (numpy/OpenBLAS, all host threads),
    extrapolated from: 1 linearisation, 1 gradient, n_mv Gramian matvecs, 1 dense
    Nystrom factorisation at (p, l), 1 preconditioner apply, 1 loss."""
    import scipy.linalg

    from oracle import ngd_oracle as O

    widths, kind, n_int, n_bnd, ell, maxit = CONFIGS[name]
    okind = {"sin2d": "sin2d", "lap": "sin2d", "sinsum": "sinsum", "gauss": "gauss"}[kind]
    prob = O.PoissonProblem(widths, kind=okind, interior_only=(kind == "lap"))
    quad = prob.sample_quadrature(n_int, n_bnd, 0)
    theta = O.init_theta(widths, 0)
    p = len(theta)
    t0 = time.perf_counter()
    loss = prob.loss_value(theta, quad)
    t_loss = time.perf_counter() - t0
    t0 = time.perf_counter()
    gop = O.GramianOracle(prob, theta, quad)
    t_lin = time.perf_counter() - t0
    t0 = time.perf_counter()
    gop.lin.vjp(prob.residual_weights(quad) * (gop.lin.value + prob.data_offsets(quad)))
    t_grad = time.perf_counter() - t0
    rng = np.random.default_rng(0)
    v = rng.standard_normal(p)
    t0 = time.perf_counter()
    for _ in range(n_mv):
        v = gop.matvec(v) / 1e3
    t_mv = (time.perf_counter() - t0) / n_mv
    # dense part of sketch.py:74-86 at (p, ell) on a synthetic SPD sketch
    om = rng.standard_normal((p, ell))
    t0 = time.perf_counter()
    om, _ = np.linalg.qr(om)
    y = om * np.linspace(1.0, 1e-9, ell)[None, :] + 1e-3 * rng.standard_normal((p, ell))
    y = om @ (om.T @ y)
    shift = np.finfo(float).eps * np.linalg.norm(y, "fro")
    ys = y + shift * om
    try:
        c = scipy.linalg.cholesky(om.T @ ys + 1e-6 * np.eye(ell), lower=False)
        b = scipy.linalg.solve_triangular(c, ys.T, lower=False, trans="T").T
        u, s, _ = np.linalg.svd(b, full_matrices=False)
    except Exception:
        u = om
    t_fact = time.perf_counter() - t0
    pre = O.PreconditionerOracle(O.NystromFactorOracle(u, np.sort(rng.random(ell))[::-1]), 1e-3)
    t0 = time.perf_counter()
    pre.apply(v)
    t_pre = time.perf_counter() - t0
    n_matvecs = ell + maxit + 1 + maxit // 50
    step = t_loss + t_lin + t_grad + n_matvecs * t_mv + t_fact + maxit * t_pre + 2 * t_loss
    sample = (f"oracle {name}: 1 loss + 1 linearisation + 1 gradient + {n_mv} Gramian matvecs + 1 dense Nystrom "
              f"factorisation ({p}x{ell}) + 1 preconditioner apply, extrapolated to one NGD step "
              f"({n_matvecs} matvecs, {maxit} PCG its)")
    return step, sample, {"t_matvec_s": t_mv, "t_factor_s": t_fact, "t_linearize_s": t_lin}


def host_cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


# ---------------------------------------------------------------------------
# reference arm
# ---------------------------------------------------------------------------


def run_reference(args, rank):
    if rank != 0:
        return
    name = args.config
    for _ in range(args.warmup):
        cpu_step_sample(name, n_mv=2)
    times = []
    sample = ""
    for _ in range(args.steps):
        t, sample, _ = cpu_step_sample(name, n_mv=4)
        times.append(t)
    ms = 1e3 * float(np.mean(times))
    value = 1e3 / ms
    widths, kind, n_int, n_bnd, ell, maxit = CONFIGS[name]
    line = {
        "impl": "reference", "metric": f"NGD steps/sec ({name})", "value": value, "unit": "steps/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded quadrature, reference init)",
        "config": config_dict(name, args.gpus),
        "cpu_baseline": {"value": value, "unit": "steps/s", "cores": host_cores(), "kind": "port", "sample": sample,
                         "cpu_model": cpu_model()},
        "e2e": {"value": value, "unit": "steps/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def config_dict(name, world):
    widths, kind, n_int, n_bnd, ell, maxit = CONFIGS[name]
    return {"workload": f"{name}: Poisson ({kind}) MLP {'-'.join(map(str, widths))} tanh, fp64, "
                        f"{n_int}+{n_bnd} pts per GPU, Nystrom l={ell} fixed, PCG maxit={maxit}, kappa=1e-300",
            "points_per_gpu": n_int + n_bnd, "ell": ell, "pcg_maxit": maxit, "parallelism": f"point-shard dp{world}",
            "l2": "flushed between steps (256 MB write)", "omega": "device Philox Gaussian (throughput mode)"}


# ---------------------------------------------------------------------------
# rooflines
# ---------------------------------------------------------------------------


def roofline_entry(kind, widths, n_int, n_bnd, ell, p, sweeps, count, total_ms, peaks, sweeps_f32=0):
    """Algorithmic work per launch of kernel class `kind` / average duration."""
    d = widths[0]
    S = n_int * (d + 2) + n_bnd
    nl = len(widths) - 1
    pw = sum(i * o for i, o in zip(widths[:-1], widths[1:]))
    n_pts = n_int + n_bnd
    bound, unit, peak = "tensor", "TFLOP/s", peaks["fp64_tflops"]
    if kind in (3, 4):  # one launch = all layers: 2 Pw S FLOP
        work = 2.0 * pw * S
    elif kind in (1, 2):  # one launch = one layer, one point segment (average)
        work = 2.0 * pw * S / (2 * nl)
    elif kind == 9:  # one-sided Jacobi on X = R^T with rotation accumulation: ~9 ell^2 (ell-1) per sweep;
        # svd=3 runs two launches per factorisation (FP32 pre-sweeps, FP64 finish): their average
        launches = 2 if sweeps_f32 > 0 else 1
        work = 9.0 * ell * ell * (ell - 1) * (max(sweeps, 1) + sweeps_f32) / launches
    elif kind == 10:
        work = ell ** 3 / 3.0
    elif kind == 14:  # fused narrow matvec: one launch = one full J^T diag(w) J v
        work = 4.0 * pw * S
    elif kind == 13:  # right triangular solve p x ell (2 launches: diagonal-block inverse + solve): p ell^2 FLOP
        work = p * ell * ell / 2.0
    else:  # memory-bound classes
        bound, unit, peak = "hbm", "GB/s", peaks["hbm_gbs"]
        if kind == 5:
            work = 8.0 * p * min(n_pts, max(1, (8 << 30) // (8 * p)))  # one Jacobian-row chunk written
        elif kind == 6:
            work = 8.0 * p * ell  # one pass over U
        else:
            work = 8.0 * 3 * p
    avg_s = total_ms * 1e-3 / max(count, 1)
    achieved = (work / max(avg_s, 1e-30)) / (1e12 if unit == "TFLOP/s" else 1e9)
    return {"bound": bound, "kernel": KIND_NAMES.get(kind, str(kind)), "achieved": achieved, "peak": peak,
            "unit": unit, "frac": achieved / peak, "traffic": None, "launches": int(count),
            "avg_launch_us": avg_s * 1e6, "algorithmic_work_per_launch": work,
            "peak_source": "FP64: DMMA measured on this pool (tools/probe/fp64_peak.cu, profiles/r01_fp64_peak.txt); "
                           f"HBM: {peaks['hbm_gbs']} GB/s from {peaks['source']}"}


def cpu_model():
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def standalone_rooflines(ngd, _lib, lib, prob, quad, theta0, widths, n_int, n_bnd, ell, peaks, reps=5):
    """Gramian matvec (phase A + phase B) and the sketch block (J rows + 2 DGEMMs), timed standalone."""
    import torch

    d = widths[0]
    S = n_int * (d + 2) + n_bnd
    pw = sum(i * o for i, o in zip(widths[:-1], widths[1:]))
    gop = ngd.GramianOperator.from_problem(prob, _lib.to_device(theta0), quad)
    p = gop.dim
    v = torch.randn(p, dtype=torch.float64, device="cuda")
    out = {}
    for kind in (3, 4):
        gop.matvec_device(v)
        _lib.check(lib.ngd_probe_start(kind, 64))
        for _ in range(reps):
            gop.matvec_device(v)
        tt, cc = _lib.ctypes.c_double(), _lib.ctypes.c_int64()
        _lib.check(lib.ngd_probe_stop(_lib.ctypes.byref(tt), _lib.ctypes.byref(cc)))
        out[KIND_NAMES[kind]] = roofline_entry(kind, widths, n_int, n_bnd, ell, p, 0, cc.value, tt.value, peaks)
    s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for _ in range(2):
        s0.record()
        gop.matvec_device(v)
        s1.record()
        s1.synchronize()
    mv_ms = s0.elapsed_time(s1)
    out["gram_matvec"] = {"ms": mv_ms, "tflops": 4.0 * pw * S / (mv_ms * 1e-3) / 1e12,
                          "frac_fp64": 4.0 * pw * S / (mv_ms * 1e-3) / 1e12 / peaks["fp64_tflops"],
                          "note": "4 Pw S FLOP (factored Jacobian, phase A + phase B + reductions)"}
    n_pts = n_int + n_bnd
    Vcm = torch.randn((ell, p), dtype=torch.float64, device="cuda")
    Ycm = torch.empty_like(Vcm)
    gop.matmat_colmajor(Vcm, Ycm)
    s0.record()
    gop.matmat_colmajor(Vcm, Ycm)
    s1.record()
    s1.synchronize()
    sk_ms = s0.elapsed_time(s1)
    fl = 4.0 * n_pts * p * ell
    out["sketch_block"] = {"ms": sk_ms, "tflops": fl / (sk_ms * 1e-3) / 1e12,
                           "frac_fp64": fl / (sk_ms * 1e-3) / 1e12 / peaks["fp64_tflops"],
                           "note": "4 N p ell FLOP (J-chunk: J rows + J Omega + J^T(w S) on DMMA)"}
    return out


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c2", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--probe", type=int, default=0, help="kernel class to time for the roofline (0 = auto)")
    ap.add_argument("--phases", action="store_true", help="print a per-phase breakdown to stderr")
    ap.add_argument("--no-cpu", action="store_true", help="skip the CPU baseline leg")
    args = ap.parse_args()

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank)
        return

    import torch

    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    import paper_2505_11638_b200 as ngd
    from paper_2505_11638_b200 import _lib, distributed
    from paper_2505_11638_b200.optim import NystromNgdRunner

    lib = _lib.load()
    prob, quad, theta0, cfg = make_problem(ngd, args.config, world, rank)
    if world > 1:
        distributed.attach(prob, distributed.NcclComm())
    runner = NystromNgdRunner(prob, theta0, cfg, quad)
    for _ in range(args.warmup):
        runner.step()
    torch.cuda.synchronize()
    if args.phases and rank == 0:
        from paper_2505_11638_b200.optim import _StepTimer

        tm = _StepTimer(True)
        runner.step(timer=tm)
        torch.cuda.synchronize()
        ev = tm.events
        parts = {ev[i + 1][0]: ev[i][1].elapsed_time(ev[i + 1][1]) for i in range(len(ev) - 1)}
        print("phases_ms", json.dumps(parts), file=sys.stderr, flush=True)
        for kind in KIND_NAMES:
            _lib.check(lib.ngd_probe_start(kind, 4096))
            runner.step()
            tt, cc = _lib.ctypes.c_double(), _lib.ctypes.c_int64()
            _lib.check(lib.ngd_probe_stop(_lib.ctypes.byref(tt), _lib.ctypes.byref(cc)))
            print(f"kernel_class {KIND_NAMES[kind]}: {cc.value} launches, {tt.value:.3f} ms total per step",
                  file=sys.stderr, flush=True)

    widths = CONFIGS[args.config][0]
    n_int, n_bnd = CONFIGS[args.config][2], CONFIGS[args.config][3]
    # dominant kernel class of OUR kernels: one probed step per class (cheap configs only), then the
    # class with the largest device time is bracketed by events inside the timed region
    ell = CONFIGS[args.config][4]
    class_ms = {}
    if not args.probe and rank == 0:
        t0 = time.perf_counter()
        runner.step()
        torch.cuda.synchronize()
        if time.perf_counter() - t0 < 0.5:
            for kind in KIND_NAMES:
                _lib.check(lib.ngd_probe_start(kind, 8192))
                runner.step()
                tt, cc = _lib.ctypes.c_double(), _lib.ctypes.c_int64()
                _lib.check(lib.ngd_probe_stop(_lib.ctypes.byref(tt), _lib.ctypes.byref(cc)))
                class_ms[KIND_NAMES[kind]] = (round(tt.value, 4), int(cc.value))
    if args.probe:
        probe_kind = args.probe
    elif class_ms:
        own = {KIND_NAMES[k] for k in OWN_KINDS}
        name = max((k for k in class_ms if k in own), key=lambda k: class_ms[k][0])
        probe_kind = {v: k for k, v in KIND_NAMES.items()}[name]
    else:
        probe_kind = 4
    if world > 1:
        t = torch.tensor([probe_kind], device="cuda")
        dist.broadcast(t, 0)
        probe_kind = int(t.item())
    flush = torch.empty(256 * 1024 * 1024 // 8, dtype=torch.float64, device="cuda")
    clocks = ClockSampler(local)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clocks.start()
    launches0 = lib.ngd_launch_count()
    _lib.check(lib.ngd_probe_start(probe_kind, 8192))
    step_ms = []
    matvecs = 0
    for _ in range(args.steps):
        flush.zero_()
        s = torch.cuda.Event(enable_timing=True)
        e = torch.cuda.Event(enable_timing=True)
        s.record()
        rec = runner.step()
        e.record()
        e.synchronize()
        step_ms.append(s.elapsed_time(e))
        matvecs += runner.last_matvecs
    launches = lib.ngd_launch_count() - launches0
    ktot = _lib.ctypes.c_double()
    kcnt = _lib.ctypes.c_int64()
    _lib.check(lib.ngd_probe_stop(_lib.ctypes.byref(ktot), _lib.ctypes.byref(kcnt)))
    clk = clocks.stop()
    total_ms = float(np.sum(step_ms))
    if world > 1:
        t = torch.tensor([total_ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
        dist.barrier()
    ms_per_step = total_ms / args.steps
    value = world * 1e3 / ms_per_step  # weak scaling: each rank's share is one C-size problem

    # roofline of the probed kernel class: algorithmic work per launch / average launch time
    peaks = load_peaks()
    avg_ms = ktot.value / max(kcnt.value, 1)
    sweeps = _lib.ctypes.c_int64()
    runner.ctx.call("ngd_get_stat", b"jacobi_sweeps", _lib.ctypes.byref(sweeps))
    sweeps_f32 = _lib.ctypes.c_int64()
    runner.ctx.call("ngd_get_stat", b"jacobi_sweeps_f32", _lib.ctypes.byref(sweeps_f32))
    roof = roofline_entry(probe_kind, widths, n_int, n_bnd, ell, len(theta0), abs(sweeps.value), kcnt.value,
                          ktot.value, peaks, sweeps_f32=abs(sweeps_f32.value))
    if probe_kind == 9:
        roof["sweeps"] = {"fp64": abs(sweeps.value), "fp32": abs(sweeps_f32.value)}
    try:  # measured DRAM traffic of this kernel at this config (one ncu --set full capture)
        with open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles", "traffic_r01.json")) as fh:
            tr = json.load(fh).get(f"{args.config}/{roof['kernel']}")
        if tr:
            roof["traffic"] = tr["bytes_per_launch"]
            roof["traffic_source"] = tr["source"]
    except (OSError, ValueError):
        pass
    roof["class_ms_per_step"] = class_ms
    # north-star kernels measured standalone after the timed region (they run inside CUDA graphs in PCG)
    extra = standalone_rooflines(ngd, _lib, lib, prob, quad, theta0, widths, n_int, n_bnd, ell, peaks) if rank == 0 else {}

    # e2e through the public API with host buffers
    e2e = None
    if rank == 0 or world > 1:
        e2e_ms = []
        p = len(theta0)
        th_host = np.array(theta0)
        for k in range(max(2, min(args.steps, 5))):
            q = ngd.QuadratureSet(quad.interior_points.copy(), quad.interior_weights.copy(),
                                  quad.boundary_points.copy(), quad.boundary_weights.copy())
            c1 = ngd.NystromNgdConfig(**{**cfg.__dict__, "iterations": 1, "seed": k})
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            th_host, recs = ngd.nystrom_ngd_run(prob, th_host, c1, q)
            _ = [r.loss for r in recs]
            e2e_ms.append(1e3 * (time.perf_counter() - t0))
        npts = len(quad.interior_points) + len(quad.boundary_points)
        h2d = 8 * (p + npts * (widths[0] + 2))
        e2e_v = world * 1e3 / float(np.mean(e2e_ms[1:]))
        e2e = {"value": e2e_v, "unit": "steps/s", "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(8 * p + 64),
               "note": "nystrom_ngd_run(iterations=1) per step from host numpy theta + fresh host quadrature"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        t_cpu, sample, cpu_parts = cpu_step_sample(args.config)
        cpu = {"value": 1.0 / t_cpu, "unit": "steps/s", "cores": host_cores(), "kind": "port", "sample": sample,
               "cpu_model": cpu_model(), **{k: round(v, 6) for k, v in cpu_parts.items()}}

    if rank == 0:
        line = {
            "metric": f"NGD steps/sec ({args.config})", "value": value, "unit": "steps/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded quadrature, reference init)",
            "config": config_dict(args.config, world),
            "matvecs_per_sec": world * matvecs / (total_ms * 1e-3), "matvecs_per_step": matvecs / args.steps,
            "roofline": roof, "north_star_kernels": extra, "cpu_baseline": cpu, "e2e": e2e,
            "gpu_launches": int(launches), "clocks": clk,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
