"""pytest plugin: run the REFERENCE's own test suite with its hot path on the GPU.

Loaded with ``-p shim_plugin`` by tests/test_gpu_refsuite.py.  Before any
reference test module is imported it calls ``shim.install(count=True)``, so
every ``from spikedigits.x import y`` in the tests and in the reference's own
modules (cli, evaluate, estimator, service, ...) resolves to the GPU versions;
it points ``sys.executable`` at ``pyshim`` so the tests that launch the
reference CLI in a subprocess (test_cli.py:98, test_acceptance.py:303) run
it through ``python -m paper_1711_03637_b200.shim`` as well; at exit it writes
the per-entry-point GPU call counts to $SNN_SHIM_REPORT (JSON).
"""
from __future__ import annotations

import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))


def pytest_configure(config):
    from paper_1711_03637_b200 import shim
    bound = shim.install(count=True)
    os.environ["SNN_REAL_PYTHON"] = sys.executable
    sys.executable = os.path.join(HERE, "pyshim")
    config._snn_bound = bound


def pytest_unconfigure(config):
    from paper_1711_03637_b200 import shim
    out = os.environ.get("SNN_SHIM_REPORT")
    if out:
        import spikedigits.network as net
        report = {"bound": getattr(config, "_snn_bound", 0), "calls": shim.call_counts(),
                  "network.run_presentation": f"{net.run_presentation.__module__}.{net.run_presentation.__name__}"}
        with open(out, "w") as f:
            json.dump(report, f)
