"""pytest plugin: run the reference's own test suites with its segregated engine routed to the
B200 path (integration/segconv_gpu.py). Used by tests/test_gpu_reference_suite.py:

    PYTHONPATH=baseline/_ref:. python -m pytest -p integration.pytest_route_gpu baseline/_ref/tests/...

At session end the number of GPU prepare / forward / counted calls is written to the file named
by SEGB200_ROUTE_REPORT (evidence that the reference's calls really reached the device)."""

import json
import os


def pytest_configure(config):
    import segconv

    from integration import segconv_gpu
    segconv_gpu.route(segconv)


def pytest_sessionfinish(session, exitstatus):
    from integration import segconv_gpu
    path = os.environ.get("SEGB200_ROUTE_REPORT")
    if path:
        with open(path, "w") as f:
            json.dump(segconv_gpu.calls, f)
