"""The C-ABI library builds, loads and exports every symbol include/ngd.h declares (CPU only)."""

import os
import re

import pytest

from paper_2505_11638_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared():
    text = open(os.path.join(ROOT, "include", "ngd.h")).read()
    return sorted(set(re.findall(r"^(?:int|int64_t|double|const char\*)\s+(ngd_\w+)\(", text, re.M)))


def test_header_declares_the_protocol():
    names = declared()
    for required in ("ngd_ctx_create", "ngd_set_points", "ngd_linearize", "ngd_loss_grad", "ngd_gram_matvec",
                     "ngd_gram_matmat", "ngd_nystrom_prepare", "ngd_nystrom_finish", "ngd_precond_apply",
                     "ngd_pcg", "ngd_ctx_set_comm"):
        assert required in names


def test_library_exports_every_declared_symbol():
    if not os.path.exists(_lib.LIB_PATH):
        from paper_2505_11638_b200 import build

        build.build()
    lib = _lib.load()
    for name in declared():
        assert hasattr(lib, name), name
    assert set(declared()) == set(_lib.SIGNATURES), "ctypes table and header disagree"
    assert lib.ngd_version() == 1


def test_sass_uses_fp64_tensor_cores():
    """The jet GEMMs must lower to DMMA (FP64 tensor-core MMA), not DFMA loops."""
    import shutil
    import subprocess

    if not shutil.which("cuobjdump") and not os.path.exists("/usr/local/cuda/bin/cuobjdump"):
        pytest.skip("cuobjdump unavailable")
    exe = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    out = subprocess.run([exe, "-sass", _lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "DMMA.8x8x4" in out
    assert "sm_100a" in subprocess.run([exe, "-lelf", _lib.LIB_PATH], capture_output=True, text=True).stdout


def test_sass_gemm_is_tma_fed_dmma():
    """The sketch / factorisation GEMM (ngd_gemm.cu) issues DMMA fed by TMA (UTMALDG) and no
    library GEMM is linked in: cuBLAS is not a dependency of the library."""
    import shutil
    import subprocess

    exe = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(exe):
        pytest.skip("cuobjdump unavailable")
    out = subprocess.run([exe, "-sass", _lib.LIB_PATH], capture_output=True, text=True).stdout
    gemm = [s for s in out.split("Function : ") if s.split("\n", 1)[0].find("dgemm_kernel") >= 0]
    assert len(gemm) == 8  # the four operand layouts x the two CTA tile shapes (128x128, 256x64)
    for s in gemm:
        assert "DMMA.8x8x4" in s and "UTMALDG.2D" in s
    needed = subprocess.run(["readelf", "-d", _lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "libcublas" not in needed  # direct dependencies only (cuSOLVER pulls cuBLAS in itself)
