"""The REFERENCE's own test suite, run against the GPU path.

baseline/_ref holds the unmodified reference (pip-installed) and its test
suite and shipped config (scripts/stage_reference.sh).  Each reference test
file runs in a fresh interpreter with tests/refsuite/shim_plugin.py, which
installs ``shim.install(count=True)`` before the tests import anything, so
the reference's tests exercise the drop-in boundary exactly as a user of the
reference would: the same imports, the same calls, the same exceptions --
with run_presentation / forward_pass / batch_counts / train_presentation /
train_epoch / preprocess_pipeline executing the CUDA kernels of
libsnn_b200.so.  The plugin's report shows which GPU entry points the file
drove and how often.
"""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")
SUITE = os.path.join(REF, "pkg", "tests")
if not os.path.isdir(SUITE):
    pytest.skip("reference suite not staged (scripts/stage_reference.sh)", allow_module_level=True)

# file -> GPU entry points its tests must drive (the hot path they exercise)
FILES = {
    "test_network.py": {"run_presentation", "forward_pass"},
    "test_normad.py": {"train_epoch"},
    "test_estimator.py": {"train_epoch", "batch_counts"},
    "test_cli.py": {"train_epoch"},
    "test_service.py": {"run_presentation", "preprocess_pipeline"},
    "test_acceptance.py": {"train_epoch", "run_presentation", "batch_counts", "preprocess_pipeline"},
    "test_preprocess.py": {"preprocess_pipeline"},
    "test_neurons.py": set(),
    "test_config.py": set(),
    "test_datasets.py": set(),
}


# Reference tests that cannot pass anywhere: they read fixtures the reference
# distribution does not ship (tests/data/ is absent from /root/reference/pkg,
# so they fail with FileNotFoundError on the stock CPU reference as well).
DESELECT = {
    "test_preprocess.py": ["TestPipeline::test_golden_corpus"],   # tests/data/golden_preprocess/digits.npz
}


def run_ref_file(name, tmp_path, extra=()):
    report = tmp_path / "report.json"
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([os.path.join(ROOT, "tests", "refsuite"), ROOT, REF,
                                         env.get("PYTHONPATH", "")])
    env["SNN_SHIM_REPORT"] = str(report)
    cmd = [sys.executable, "-m", "pytest", "-q", "-p", "shim_plugin", "-p", "no:cacheprovider",
           "--rootdir", os.path.join(REF, "pkg"), os.path.join(SUITE, name), *extra]
    r = subprocess.run(cmd, cwd=os.path.join(REF, "pkg"), env=env, capture_output=True, text=True, timeout=1800)
    rep = json.loads(report.read_text()) if report.exists() else {}
    return r, rep


@pytest.mark.parametrize("name", sorted(FILES))
def test_reference_suite_file_on_gpu(name, tmp_path):
    extra = [a for t in DESELECT.get(name, []) for a in ("--deselect", f"tests/{name}::{t}")]
    r, rep = run_ref_file(name, tmp_path, extra)
    tail = (r.stdout[-3000:] + r.stderr[-2000:])
    assert r.returncode == 0, tail
    assert rep.get("network.run_presentation") == "paper_1711_03637_b200.api.run_presentation", rep
    calls = rep.get("calls", {})
    missing = {fn for fn in FILES[name] if calls.get(fn, 0) == 0}
    assert not missing, (missing, calls, tail)
    print(name, r.stdout.strip().splitlines()[-1], calls)
