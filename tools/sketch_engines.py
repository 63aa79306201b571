"""Sketch block Y = G Omega at a BASELINE config on both engines (DMMA FP64 vs INT8 Ozaki II):
wall time per block, per-class breakdown, and the INT8 engine's deviation from the DMMA one."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2505_11638_b200 as ngd  # noqa: E402
from paper_2505_11638_b200 import _lib  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c5"
engines = [int(x) for x in (sys.argv[2] if len(sys.argv) > 2 else "1,0").split(",")]
prob, quad, theta0, _ = bench.make_problem(ngd, cfg)
ell = bench.CONFIGS[cfg][4]
gop = ngd.GramianOperator.from_problem(prob, theta0, quad)
V = torch.randn((ell, gop.dim), dtype=torch.float64, device="cuda")
n = len(quad.interior_points) + len(quad.boundary_points)
lib = _lib.load()
out = {}
for eng in engines:
    with _lib.option("sketch_gemm", eng):
        Y = torch.empty_like(V)
        gop.matmat_colmajor(V, Y)
        torch.cuda.synchronize()
        s = torch.cuda.Event(enable_timing=True)
        e = torch.cuda.Event(enable_timing=True)
        s.record()
        gop.matmat_colmajor(V, Y)
        e.record()
        e.synchronize()
        ms = s.elapsed_time(e)
        cls = bench.probe_all(_lib, lib, lambda: (gop.matmat_colmajor(V, Y), torch.cuda.synchronize()))
        out[eng] = Y.clone()
        print(f"{cfg} engine {eng}: sketch block ({ell} columns) {ms:.1f} ms = "
              f"{4.0 * n * gop.dim * ell / ms / 1e9:.2f} TFLOP/s (FP64-equivalent); classes {cls}", flush=True)
if 0 in out and 1 in out:
    d = (torch.linalg.norm(out[1] - out[0], dim=1) / torch.linalg.norm(out[0], dim=1)).max().item()
    print(f"{cfg}: max column rel diff INT8 vs DMMA {d:.3e}")
