"""The reference package's OWN test suite (pkg/tests, 158 tests) run with a
third backend: the CUDA kernel seam (paper_2408_05462_b200.shim installed
into isochr.kernels, SURVEY §8(b) plug level 1; the reference's tests switch
backends through conftest.py:14-21 and every caller reaches the kernels
through the module attribute).

Needs the reference install under baseline/_ref (tools/install_ref.sh: the
unmodified package + a copy of its tests; git-ignored, it travels to the GPU
box with the repo).  Skipped when absent."""

import os
import re
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")
SUITE = os.path.join(REF, "isochr_tests")


@pytest.mark.skipif(not os.path.isdir(SUITE), reason="reference install absent (tools/install_ref.sh)")
def test_reference_suite_with_cuda_seam():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([REF, ROOT, env.get("PYTHONPATH", "")])
    env.setdefault("NUMBA_CACHE_DIR", "/tmp/chr_numba_cache")
    cmd = [sys.executable, "-m", "pytest", SUITE, "-q", "-p", "no:cacheprovider", "-p",
           "paper_2408_05462_b200.shim_plugin", "-x"]
    out = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=1200)
    tail = out.stdout[-3000:] + out.stderr[-2000:]
    log = os.path.join(ROOT, "gpurun_out", "reference_suite_cuda.log")
    if os.path.isdir(os.path.dirname(log)):
        with open(log, "w") as fh:
            fh.write(out.stdout + out.stderr)
    assert out.returncode == 0, tail
    m = re.search(r"(\d+) passed", out.stdout)
    assert m and int(m.group(1)) >= 150, tail
