"""pytest plugin: run the reference's OWN test files with its dispatch points
bound to libmwgpu.so (integration/mwfloat_gpu.py).

    PYTHONPATH=baseline/_ref:. python -m pytest -p integration.pytest_gpu_plugin \
        baseline/_ref/ref_tests/test_batch.py ...

At session end the per-entry-point call counts are written to
$MWGPU_CALLS_OUT (JSON) so the caller can prove the device path ran.
"""

import json
import os

from integration import mwfloat_gpu


def pytest_configure(config):
    import mwfloat

    calls = mwfloat_gpu.install()
    calls["mwfloat_file"] = 0
    config._mwgpu_mwfloat = mwfloat.__file__


def pytest_sessionfinish(session, exitstatus):
    out = os.environ.get("MWGPU_CALLS_OUT")
    if out:
        calls = dict(mwfloat_gpu.CALLS)
        calls.pop("mwfloat_file", None)
        with open(out, "w") as f:
            json.dump({"calls": calls, "mwfloat": getattr(session.config, "_mwgpu_mwfloat", None),
                       "exitstatus": int(exitstatus)}, f)
