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
           "paper_2408_05462_b200.shim_plugin", "-rf"]
    out = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=1200)
    text = out.stdout + out.stderr
    passed = int(m.group(1)) if (m := re.search(r"(\d+) passed", out.stdout)) else 0
    failed = re.findall(r"^FAILED (\S+)", out.stdout, re.M)
    retried = []
    if out.returncode != 0 and failed and all(TIMED.search(f) for f in failed):
        # the reference's wall-clock criteria (e.g. test_acceptance.py criterion 9,
        # relaxed-accuracy speedup of its own CPU pipeline) are timing-noise
        # sensitive on a shared host: re-run just those once
        again = subprocess.run(cmd[:3] + [os.path.join(ROOT, f) for f in failed] + cmd[4:],
                               cwd=ROOT, env=env, capture_output=True, text=True, timeout=1200)
        text += "\n==== re-run of timing criteria ====\n" + again.stdout + again.stderr
        if again.returncode == 0:
            retried = failed
            passed += len(failed)
    tail = text[-5000:]
    log = os.path.join(ROOT, "gpurun_out", "reference_suite_cuda.log")
    if os.path.isdir(os.path.dirname(log)):
        with open(log, "w") as fh:
            fh.write(text)
    assert out.returncode == 0 or (failed and retried == failed), tail
    assert passed >= 150, tail


# reference tests whose assertion is a wall-clock ratio (retried once on failure)
TIMED = re.compile(r"speedup|throughput|timing")
