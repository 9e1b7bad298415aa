"""Bounds-checked engine build (libgfcuda_checked.so, -DGF_CHECKS).

compute-sanitizer is not available on this GPU pool (runs under it left GPUs
needing a reset), so the engine carries its own device asserts: every fused
tile address is an XOR of per-slot columns, and the checked build traps
unless each column, each pair / tuple offset and every global tile address
stays in range.  This test runs the sanitizer workload (multi-tile,
multi-pass, multi-direction, sector) through the checked library and
requires it to finish cleanly with results equal to the production build's.
"""

import os
import subprocess
import sys

import pytest

from conftest import ROOT

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover - CPU container
    pytest.skip("needs a CUDA GPU", allow_module_level=True)

LIB = os.path.join(ROOT, "paper_2506_23775_b200", "libgfcuda_checked.so")


def _run(env_extra):
    env = dict(os.environ, **env_extra)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "sanitize_case.py")], capture_output=True,
                       text=True, timeout=900, cwd=ROOT, env=env)
    return r


def test_checked_build_runs_the_sanitizer_workload_cleanly():
    assert os.path.exists(LIB), "build() must produce libgfcuda_checked.so"
    chk = _run({"GF_LIB_PATH": LIB, "GF_EXPECT_LIB": "libgfcuda_checked.so"})
    assert chk.returncode == 0, (chk.stdout[-2000:], chk.stderr[-3000:])
    assert "GF_CHECKS" not in chk.stdout + chk.stderr
    ref = _run({})
    assert ref.returncode == 0, ref.stderr[-3000:]
    line = lambda out: [x for x in out.splitlines() if x.startswith("sanitize case ok")][-1]
    assert line(chk.stdout) == line(ref.stdout)
