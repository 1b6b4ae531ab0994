"""The reference's own tests, run against the GPU kernels through the C-ABI.

``integration/mwfloat_gpu.py`` is the binding a maintainer would add to the
reference: it rebinds ``batch._BATCH_ADD/_BATCH_MUL``
(``batch.py:178-194``) and ``linalg._naive_mm`` (``linalg.py:368-375``) of
the UNMODIFIED reference package -- installed into ``baseline/_ref`` by
``scripts/install_reference.sh`` -- to ``mw_ew_add/mw_ew_mul/mw_gemm``.  The
reference's test files for the bound paths then run unchanged:
``test_batch.py`` (lanes == scalar kernels bitwise, ``:86-122``),
``test_linalg.py`` (naive == blocked, thread invariance, identity,
Strassen, 3M, ``:100-151``), ``test_poly.py`` (Horner / Estrin vs the
oracle, lanes == scalar, ``:33-154``) and ``test_roots.py`` (Aberth init,
DK fixed points, collisions, convergence, determinism, ``:35-190``).
"""

import json
import os
import subprocess
import sys

import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(REPO, "baseline", "_ref")
FILES = ["test_batch.py", "test_linalg.py", "test_poly.py", "test_roots.py"]


def _have_ref():
    return os.path.exists(os.path.join(REF, "mwfloat", "__init__.py")) and os.path.isdir(os.path.join(REF, "ref_tests"))


def test_binding_module_imports_without_gpu():
    sys.path.insert(0, REPO)
    from integration import mwfloat_gpu

    assert callable(mwfloat_gpu.install) and mwfloat_gpu.LIB_PATH.endswith("libmwgpu.so")


@pytest.mark.gpu
@pytest.mark.skipif(not _have_ref(), reason="baseline/_ref not installed (scripts/install_reference.sh)")
def test_reference_suite_runs_on_the_gpu_kernels(tmp_path):
    calls_out = tmp_path / "calls.json"
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([REF, REPO, env.get("PYTHONPATH", "")])
    env["MWGPU_CALLS_OUT"] = str(calls_out)
    cmd = [sys.executable, "-m", "pytest", "-q", "-p", "integration.pytest_gpu_plugin", "-p", "no:cacheprovider",
           "--rootdir", os.path.join(REF, "ref_tests")] + [os.path.join(REF, "ref_tests", f) for f in FILES]
    r = subprocess.run(cmd, cwd=str(tmp_path), env=env, capture_output=True, text=True, timeout=1500)
    tail = (r.stdout + r.stderr)[-4000:]
    os.makedirs(os.path.join(REPO, "gpurun_out"), exist_ok=True)
    with open(os.path.join(REPO, "gpurun_out", "reference_suite_on_gpu.log"), "w") as f:
        f.write(r.stdout + r.stderr)
    assert r.returncode == 0, tail
    info = json.loads(calls_out.read_text())
    calls = info["calls"]
    assert info["mwfloat"].startswith(REF), info
    # the device path ran, for the lane tables and the GEMM
    assert calls.get("mw_ew_add", 0) > 1000 and calls.get("mw_ew_mul", 0) > 1000, calls
    assert calls.get("mw_gemm", 0) > 10, calls
