"""CPU-only checks of the boundary: libfold.so builds for sm_100a, loads, and exports
every function include/*.h declares (fold.h, fold_mo.h; no compute calls without a GPU)."""
import ctypes
import os
import re

import pytest

from paper_1702_02181_b200 import build as fbuild

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared(headers=("fold.h", "fold_mo.h")):
    names = set()
    for h in headers:
        src = open(os.path.join(ROOT, "include", h)).read()
        src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
        names |= set(re.findall(r"\b(fold_[a-z0-9_]+)\s*\(", src))
    return sorted(names)


def test_header_declares_the_boundary():
    names = _declared()
    for n in ("fold_schedule", "fold_forward", "fold_backward", "fold_sgd_update",
              "fold_schedule_workspace", "fold_forward_workspace", "fold_backward_workspace"):
        assert n in names


def test_library_builds_and_exports_all_symbols():
    path = fbuild.build()
    lib = ctypes.CDLL(path)
    for n in _declared():
        assert hasattr(lib, n), n
    from paper_1702_02181_b200 import fold, fold_mo
    assert set(fold.EXPORTED) == set(_declared(("fold.h",)))
    assert set(fold_mo.EXPORTED) == set(_declared(("fold_mo.h",)))


def test_library_host_only_calls():
    """Calls that touch no device memory: version, status strings, workspace sizes."""
    fbuild.build()
    from paper_1702_02181_b200 import fold
    L = fold.load()
    assert L.fold_abi_version() == 6
    assert L.fold_status_string(6) == b"FOLD_E_CYCLE"
    assert L.fold_schedule_workspace(1000, 10) > 0
    assert L.fold_schedule_workspace(2_000_000, 8192) > L.fold_schedule_workspace(1000, 10)


def test_sass_is_blackwell_native():
    """The shipped kernels use tcgen05 MMA, TMEM loads and TMA tile loads — SASS check."""
    import shutil
    import subprocess
    if not shutil.which("cuobjdump"):
        pytest.skip("cuobjdump not available")
    path = fbuild.build()
    sass = subprocess.run(["cuobjdump", "-sass", path], capture_output=True, text=True).stdout
    assert "UTCHMMA" in sass and "LDTM" in sass and "UTMALDG.2D" in sass
    assert "HMMA" not in sass.replace("UTCHMMA", "")


def test_mo_host_only_calls():
    """fold_mo.h calls that touch no device memory: table validation via the workspace query
    (0 for a malformed table), the TYPE status string."""
    fbuild.build()
    import ctypes
    import foldgen
    from paper_1702_02181_b200 import fold, fold_mo
    L = fold_mo.load()
    t = fold_mo.table_struct(foldgen.mo_table_c6())
    assert L.fold_mo_schedule_workspace(ctypes.byref(t), 1000, 10) > 0
    bad = fold_mo.table_struct(foldgen.mo_table_c6())
    bad.in_type[1] = 1   # an LSTM whose input type differs from its output type
    assert L.fold_mo_schedule_workspace(ctypes.byref(bad), 1000, 10) == 0
    assert fold.load().fold_status_string(13) == b"FOLD_E_TYPE"
