"""The reference's OWN test suites, run against the B200 engine.

The unmodified reference is installed under baseline/_ref by tools/install_reference.sh (with a
copy of its tests/); integration/segconv_gpu.py (INTEGRATION.md option B) routes its segregated
engine -- PreparedLayer, layer_forward, transpose_conv_segregated, the harness, and the counted
scalar engines -- to libsegb200.so. The suites that form the parity contract
must then pass unchanged: test_engines.py, test_acceptance.py (the 8 acceptance criteria,
including the 1000-case oracle sweep) and test_segregation.py.
"""

import json
import os
import subprocess
import sys

import pytest

from tests.conftest import ROOT

pytestmark = pytest.mark.gpu

REF = os.path.join(ROOT, "baseline", "_ref")
SUITES = ["test_engines.py", "test_acceptance.py", "test_segregation.py"]


@pytest.mark.skipif(not os.path.isdir(os.path.join(REF, "tests")),
                    reason="baseline/_ref not installed (tools/install_reference.sh)")
def test_reference_suites_pass_on_the_gpu_engine(tmp_path):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    report = tmp_path / "route.json"
    env = dict(os.environ, PYTHONPATH=os.pathsep.join([REF, ROOT]), SEGB200_ROUTE_REPORT=str(report),
               PYTHONDONTWRITEBYTECODE="1")
    cmd = [sys.executable, "-m", "pytest", "-q", "-p", "integration.pytest_route_gpu", "-p", "no:cacheprovider",
           "--rootdir", REF] + [os.path.join(REF, "tests", s) for s in SUITES]
    res = subprocess.run(cmd, cwd=REF, env=env, capture_output=True, text=True, timeout=1200)
    tail = (res.stdout + res.stderr)[-4000:]
    with open(os.path.join(ROOT, "gpurun_out", "reference_suite.log") if os.path.isdir(
            os.path.join(ROOT, "gpurun_out")) else os.devnull, "w") as f:
        f.write(res.stdout + res.stderr)
    assert res.returncode == 0, tail
    calls = json.loads(report.read_text())
    assert calls["forward"] > 1000 and calls["prepare"] > 1000 and calls["counted"] > 10, calls
