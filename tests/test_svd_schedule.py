"""The block-exchange Jacobi's exchange schedule (ngd_svd.cu jsvd_make_plan, compiled for the host
with g++): block pairing per round, data flow through the three / four block buffers, and random
asynchronous executions of the point-to-point exchange protocol (tools/probe/jsvd_pool_check.py)."""
import os
import shutil
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.skipif(shutil.which("g++") is None, reason="needs g++")
def test_exchange_schedule_protocol():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "probe", "jsvd_pool_check.py")],
                         capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stdout + out.stderr
    lines = [l for l in out.stdout.splitlines() if "protocol ok" in l]
    assert len(lines) == 8, out.stdout
