"""bench.py's JSON contract on CPU: the reference arm (the oracle port timed on host cores) prints
one well-formed line, and the roofline work model is consistent with the documented FLOP counts."""

import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_line():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--config", "c1",
                          "--steps", "1", "--warmup", "0"], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
                "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e", "impl"):
        assert key in d, key
    assert d["impl"] == "reference" and d["value"] > 0 and d["unit"] == "steps/s"
    assert d["cpu_baseline"]["kind"] == "port" and d["cpu_baseline"]["value"] == d["value"]
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["config"]["workload"].startswith("c1")


def test_roofline_work_model():
    sys.path.insert(0, ROOT)
    import bench

    peaks = {"fp64_tflops": 36.99, "hbm_gbs": 6550.7, "source": "test"}
    widths, _, n_int, n_bnd, ell, _ = bench.CONFIGS["c2"]
    pw = sum(i * o for i, o in zip(widths[:-1], widths[1:]))
    S = n_int * (widths[0] + 2) + n_bnd
    # phase B: one launch = all layers = 2 Pw S FLOP; 1 ms per launch -> 2 Pw S / 1e-3 FLOP/s
    r = bench.roofline_entry(4, widths, n_int, n_bnd, ell, 8577, 10, 10.0, peaks)
    assert r["algorithmic_work_per_launch"] == pytest.approx(2.0 * pw * S)
    assert r["achieved"] == pytest.approx(2.0 * pw * S / 1e-3 / 1e12)
    assert r["frac"] == pytest.approx(r["achieved"] / 36.99) and r["bound"] == "tensor"
    # DMMA GEMM: the library's count of 2 M N K over the probed launches
    r = bench.roofline_entry(14, widths, n_int, n_bnd, ell, 8577, 4, 2.0, peaks, gemm_flops=8e12)
    assert r["algorithmic_work_per_launch"] == pytest.approx(2e12) and r["achieved"] == pytest.approx(4000.0)
    # Jacobi SVD (mixed precision): 9 FP32 + 2 FP64 sweeps of 9 ell^2 (ell - 1) FLOP over two launches
    r8 = bench.roofline_entry(15, widths, n_int, n_bnd, ell, 8577, 4, 2.0, {**peaks, "int8_tops": 3267.0},
                              i8_ops=1.6e13)
    assert r8["unit"] == "TOPS" and abs(r8["achieved"] - 1.6e13 / 4 / 0.5e-3 / 1e12) < 1e-6
    assert abs(r8["frac"] - r8["achieved"] / 3267.0) < 1e-12
    r = bench.roofline_entry(9, widths, n_int, n_bnd, ell, 8577, 2, 5.0, peaks, sweeps=(2, 9))
    assert r["algorithmic_work_per_launch"] == pytest.approx(9.0 * ell * ell * (ell - 1) * 11 / 2)


def test_cpu_step_sample_scaling():
    """The CPU baseline runs one real oracle NGD step on a point subset and scales only the
    point-proportional part: at C1 with the full point set the scale factor is 1."""
    sys.path.insert(0, ROOT)
    import bench

    t_full, sample, parts = bench.cpu_step_sample("c1")
    assert parts["scale"] == 1.0 and parts["n_sub"] == 1020 and parts["matvecs"] == 121
    assert t_full == pytest.approx(parts["fixed_s"] + parts["point_calls_s"])
    assert "real NGD step" in sample
