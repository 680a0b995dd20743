"""The reference's own entry points running on the GPU path through
shim.install(): `spikedigits train` / `eval` (cli.py:142-212) on IDX files,
checkpoints in the reference's SNNW format (datasets.py:146-200).

Needs the unmodified reference package importable -- from baseline/_ref (the
pip install of /root/reference, git-ignored, shipped with the GPU snapshot) or
/root/reference in the build container; skipped otherwise.
"""
import os
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for cand in (os.path.join(ROOT, "baseline", "_ref"), "/root/reference/pkg/src"):
    if os.path.isdir(os.path.join(cand, "spikedigits")) and cand not in sys.path:
        sys.path.append(cand)
        break
pytest.importorskip("PIL")
pytest.importorskip("sklearn")
sdr = pytest.importorskip("spikedigits")


@pytest.fixture(scope="module")
def idx_dir(tmp_path_factory, workloads):
    from spikedigits.datasets import write_idx_images, write_idx_labels
    root = tmp_path_factory.mktemp("idx")
    write_idx_images(root / "train-images-idx3-ubyte", workloads["c2_images"][:150])
    write_idx_labels(root / "train-labels-idx1-ubyte", workloads["c2_labels"][:150])
    write_idx_images(root / "t10k-images-idx3-ubyte", workloads["c3_images"][:60])
    write_idx_labels(root / "t10k-labels-idx1-ubyte", workloads["c3_labels"][:60])
    return root


def test_reference_cli_train_eval_on_gpu(idx_dir, tmp_path, workloads, oracle, capsys):
    from spikedigits.cli import main
    from spikedigits.datasets import load_checkpoint
    from spikedigits.estimator import epoch_permutation

    from paper_1711_03637_b200 import api, shim
    shim.install()
    try:
        import spikedigits.cli as cli
        assert cli.train_epoch is api.train_epoch
        ck1, ck2 = tmp_path / "a.snnw", tmp_path / "b.snnw"
        assert main(["train", "--mnist-dir", str(idx_dir), "--epochs", "2", "--out", str(ck1)]) == 0
        assert main(["train", "--mnist-dir", str(idx_dir), "--epochs", "2", "--out", str(ck2)]) == 0
        assert ck1.read_bytes() == ck2.read_bytes()  # bit-identical checkpoints (test_acceptance.py:294-318)
        w, cfg, bank = load_checkpoint(ck1)
        # the same two epochs with the CPU oracle (cli.py:142-173: seed-permuted selection,
        # then epoch_permutation per epoch, from zero weights)
        x, y = cli.select_subset(workloads["c2_images"][:150], workloads["c2_labels"][:150], None,
                                 list(range(10)), 0)
        wo = np.zeros((8112, 10))
        p = oracle.params_from_reference(cfg, bank)
        for e in range(2):
            order = epoch_permutation(0, e, len(x))
            wo, _ = oracle.train_epoch(x[order], y[order], wo, p)
        assert np.abs(w - wo).max() / np.abs(wo).max() <= 1e-9
        capsys.readouterr()
        assert main(["eval", "--weights", str(ck1), "--mnist-dir", str(idx_dir)]) == 0
        out = capsys.readouterr().out
        assert '"accuracy"' in out
    finally:
        shim.uninstall()
