"""The C ABI library loads on a CPU-only host, exports every symbol that
include/snn_b200.h declares, and the ctypes structs match the C layout."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "snn_b200.h")


def declared_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:const\s+)?[\w]+\s*\*?\s*(snn_\w+)\s*\(", text, flags=re.M)))


def test_header_declares_entry_points():
    fns = declared_functions()
    for name in ("snn_abi_version", "snn_last_error", "snn_input_table", "snn_infer_workspace",
                 "snn_infer", "snn_train_workspace", "snn_train"):
        assert name in fns


def test_library_exports_every_declared_symbol():
    from paper_1711_03637_b200 import _native
    lib = _native.load()
    for name in declared_functions():
        assert hasattr(lib, name), name
    assert {s[0] for s in _native.SIGNATURES} == set(declared_functions())
    assert lib.snn_abi_version() == _native.ABI_VERSION == 2


def test_workspace_queries_need_no_gpu():
    from paper_1711_03637_b200 import _native
    lib = _native.load()
    c = _native.ConstsC()
    c.n_steps = 100
    c.dt = 1e-3
    c.lif_hid.refr = 3.0
    assert lib.snn_infer_workspace(ctypes.byref(c), 10) >= 10 * 22 * 100 * 64   # raster upper bound
    assert lib.snn_train_workspace(ctypes.byref(c), 10) > 0
    c.n_steps = 0
    assert lib.snn_infer_workspace(ctypes.byref(c), 10) == 0


def test_invalid_consts_rejected_without_gpu():
    from paper_1711_03637_b200 import _native
    lib = _native.load()
    c = _native.ConstsC()
    c.n_steps = 0
    rc = lib.snn_input_table(ctypes.byref(c), None, None, None)
    assert rc == _native.SNN_EINVAL
    assert b"n_steps" in lib.snn_last_error()
    with pytest.raises(ValueError):
        _native.check(rc)


def test_struct_layout_matches_c(tmp_path):
    """Compile a probe against the header with gcc and compare sizeof/offsetof."""
    from paper_1711_03637_b200 import _native
    probe = tmp_path / "probe.c"
    probe.write_text(r'''
#include <stdio.h>
#include <stddef.h>
#include "snn_b200.h"
int main(void) {
  printf("%zu %zu %zu %zu %zu %zu %zu %zu %zu\n", sizeof(snn_consts_t), offsetof(snn_consts_t, lif_hid),
         offsetof(snn_consts_t, inhibition), offsetof(snn_consts_t, taps), sizeof(snn_lif_t),
         sizeof(snn_infer_out_t), offsetof(snn_infer_out_t, v_hid), offsetof(snn_infer_out_t, near_ties),
         offsetof(snn_infer_out_t, hidden_redo));
  return 0;
}
''')
    exe = tmp_path / "probe"
    subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), str(probe), "-o", str(exe)], check=True)
    got = list(map(int, subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout.split()))
    C = _native.ConstsC
    want = [ctypes.sizeof(C), C.lif_hid.offset, C.inhibition.offset, C.taps.offset,
            ctypes.sizeof(_native.LifC), ctypes.sizeof(_native.InferOutC), _native.InferOutC.v_hid.offset,
            _native.InferOutC.near_ties.offset, _native.InferOutC.hidden_redo.offset]
    assert got == want


def test_missing_library_fails_loudly(monkeypatch, tmp_path):
    from paper_1711_03637_b200 import _native
    monkeypatch.setattr(_native, "_LIB", None)
    monkeypatch.setattr(_native, "LIB_PATH", str(tmp_path / "nope.so"))
    with pytest.raises(ImportError, match="no CPU fallback"):
        _native.load()
