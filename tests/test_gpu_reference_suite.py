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


@pytest.mark.skipif(not os.path.isdir(os.path.join(REF, "segconv")),
                    reason="baseline/_ref not installed (tools/install_reference.sh)")
def test_reference_harness_with_gpu_columns():
    """the reference's own run_benchmark / emit_report over GAN_SUITE layers, segregated engine on
    the GPU, GPU columns added"""
    import json

    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    if REF not in sys.path:
        sys.path.insert(0, REF)
    import segconv

    from integration import segconv_gpu
    configs = [c for c in segconv.GAN_SUITE if c.name in ("dcgan_l5", "ebgan_l4", "gpgan_l3")]
    opts = segconv.bench.RunOptions(seed=7, repeats=2, verify=True)
    report = segconv_gpu.run_benchmark_gpu(segconv, configs, opts, batch=32, compute="fp32")
    for rec in report.layers:
        assert rec["error"] is None and rec["equivalence"]["passed"], rec
        g = rec["gpu"]
        assert g["batch"] == 32 and g["useful_gmacs"] > 0 and g["kernel"].startswith("K")
    doc = json.loads(segconv.bench.emit_report(report, "json"))
    assert doc["format_version"] == 1 and len(doc["layers"]) == 3
    assert "|" in segconv.bench.emit_report(report, "markdown")
