"""CPU-side checks of the C-ABI boundary: the library loads, exports every symbol that
include/lapssd.h declares, sizes workspaces, and rejects bad arguments synchronously
(no compute call is made: there is no GPU here)."""
import ctypes as C
import os
import re
import subprocess

import pytest

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "lapssd.h")


def declared_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    names = re.findall(r"^\s*(?:const\s+)?[A-Za-z_][A-Za-z0-9_]*\s*\*?\s*([a-z_][a-z0-9_]*)\s*\(",
                       text, flags=re.M)
    return sorted(set(names))


def test_header_declares_the_hot_path_calls():
    names = declared_functions()
    for must in ("spec_verify", "laps_update", "laps_select", "laps_step", "laps_step_dist",
                 "laps_candidates", "laps_merge", "lapssd_create", "lapssd_destroy",
                 "lapssd_read_state", "lapssd_check", "lapssd_last_error"):
        assert must in names


def test_library_exports_every_declared_symbol():
    import paper_2505_17074_b200 as L
    out = subprocess.run(["nm", "-D", "--defined-only", L.library_path()], capture_output=True,
                         text=True, check=True).stdout
    exported = {line.split()[-1] for line in out.splitlines() if " T " in line}
    missing = [n for n in declared_functions() if n not in exported]
    assert not missing, missing


def test_library_is_sm100a():
    import paper_2505_17074_b200 as L
    out = subprocess.run(["cuobjdump", "--list-elf", L.library_path()], capture_output=True,
                         text=True, check=True).stdout
    assert "sm_100a" in out


def test_workspace_sizes():
    import paper_2505_17074_b200 as L
    assert L.spec_verify_workspace_bytes(512, 128256) >= 512 * 16 * 8 * 8 + 512 * 4 + 512 * 32
    assert L.spec_verify_workspace_bytes(0, 16) > 0
    cfg = L.SchedConfig(k=8)
    n = L._lib.lapssd_workspace_bytes(C.byref(cfg.c()), 2048, 512, 128256, 1)
    assert n > 2048 * 64


def test_create_rejects_bad_config_without_touching_the_gpu():
    import numpy as np

    import paper_2505_17074_b200 as L
    for bad in (dict(K=0), dict(K=17), dict(s1_up_us=0), dict(M=1.0), dict(gamma=1),
                dict(delta=-0.1), dict(k=0), dict(k=17), dict(policy=9)):
        cfg = L.SchedConfig(**bad)
        h = C.c_void_p()
        a = np.zeros(4, np.int64)
        lt = np.ones(4, np.int32)
        req = L._Requests(a.ctypes.data, lt.ctypes.data, lt.ctypes.data, 4, 0, 1)
        rc = L._lib.lapssd_create(C.byref(cfg.c()), C.byref(req), 8, 1024, None, 0, None,
                                  C.byref(h))
        assert rc == -1, bad
        assert L._lib.lapssd_last_error().decode()


def test_spec_verify_rejects_bad_rows():
    import paper_2505_17074_b200 as L
    # V*sizeof not a multiple of 16 (bf16, V=12) -> EINVAL before any launch
    rc = L._lib.spec_verify(16, 16, L.BF16, 12, 4, None, None, None, None, 1, 0, 0, None, None,
                            None, None, 0, None)
    assert rc == -1
    rc = L._lib.spec_verify(16, 16, L.F32, 16, 0, None, None, None, None, 1, 0, 0, None, None,
                            None, None, 0, None)
    assert rc == -1
    rc = L._lib.spec_verify(16, 16, 7, 16, 4, None, None, None, None, 1, 0, 0, None, None, None,
                            None, 0, None)
    assert rc == -1


def test_spec_verify_logits_rejects_bad_arguments():
    """f1 entry: the same row checks, V <= 2^23 (integer softmax masses), workspace size,
    NULL pointers -- all EINVAL / ENOMEM before any launch; B == 0 is a no-op."""
    import paper_2505_17074_b200 as L
    f = L._lib.spec_verify_logits
    assert f(16, 16, L.BF16, 12, 4, None, None, None, None, 1, 0, 0, None, None, None, None, 0, None) == -1
    assert f(16, 16, L.F32, 16, 0, None, None, None, None, 1, 0, 0, None, None, None, None, 0, None) == -1
    assert f(16, 16, L.F32, 16, 17, None, None, None, None, 1, 0, 0, None, None, None, None, 0, None) == -1
    assert f(16, 16, L.BF16, (1 << 23) + 8, 4, None, None, None, None, 1, 0, 0, None, None, None, None, 0,
             None) == -1
    assert f(16, 16, L.BF16, 16, 4, None, None, None, None, 1, 0, 0, None, None, None, None, 0, None) == -1
    assert f(16, 16, L.BF16, 16, 4, 16, None, 16, 16, 1, 0, 0, 16, 16, None, 16, 0, None) == -5  # ENOMEM
    assert f(16, 16, L.BF16, 16, 4, None, None, None, None, 0, 0, 0, None, None, None, None, 0, None) == 0
    assert L._lib.spec_verify_logits_workspace_bytes(512, 8, 128256, 1) >= 512 * 17 * 12
    assert L._lib.spec_verify_logits_workspace_bytes(1, 0, 1024, 1) == 0
    assert L._lib.spec_verify_logits_workspace_bytes(1, 4, 1024, 7) == 0


def test_binding_fails_loudly_without_library(tmp_path, monkeypatch):
    """The product path has no fallback: a missing .so is an ImportError."""
    import importlib.util
    src = os.path.join(ROOT, "paper_2505_17074_b200", "__init__.py")
    pkg = tmp_path / "paper_2505_17074_b200"
    pkg.mkdir()
    (pkg / "__init__.py").write_text(open(src).read())
    spec = importlib.util.spec_from_file_location("lapssd_nolib", pkg / "__init__.py")
    mod = importlib.util.module_from_spec(spec)
    with pytest.raises(ImportError):
        spec.loader.exec_module(mod)


def test_product_never_imports_oracle():
    for dirpath, _, files in os.walk(os.path.join(ROOT, "paper_2505_17074_b200")):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                text = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in text and "from oracle" not in text, f
                assert "lapssd_oracle" not in text, f


def test_laps_step_logits_rejects_bad_arguments():
    """f1 inside the step: a NULL handle, B < 1, NULL rows -- EINVAL before any launch; the
    workspace covers spec_verify_logits' plus the slot counters, and rejects what it does."""
    import paper_2505_17074_b200 as L
    f = L._lib.laps_step_logits
    assert f(None, None, 1, None, None, None, None, None, 0, None) == -1
    assert L._lib.lapssd_last_error().decode()
    ws = L._lib.laps_step_logits_workspace_bytes
    assert ws(512, 8, 128256, 1) >= L._lib.spec_verify_logits_workspace_bytes(512, 8, 128256, 1) + 3 * 512 * 4
    assert ws(1, 0, 1024, 1) == 0 and ws(1, 4, 1024, 7) == 0
