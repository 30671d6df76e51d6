"""Host-side checks that need no GPU: the C-ABI library loads and exports every symbol
include/tactic.h declares, the binding declares a signature for each, and status
strings are stable.  No compute call is made here."""
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "tactic.h")


def _declared():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(tactic_[a-z0-9_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def L():
    from paper_2502_12216_b200 import build as B
    B.build()
    from paper_2502_12216_b200 import tactic
    return tactic.lib()


def test_header_declares_the_boundary():
    names = _declared()
    for must in ("tactic_build_index", "tactic_decode", "tactic_dense_decode", "tactic_index_import",
                 "tactic_index_export", "tactic_decode_debug", "tactic_lse_merge", "tactic_decode_stage1",
                 "tactic_decode_stage1b", "tactic_decode_stage2", "tactic_last_error"):
        assert must in names


def test_library_exports_every_declared_symbol(L):
    for name in _declared():
        assert hasattr(L, name), name


def test_binding_covers_every_entry_point(L):
    from paper_2502_12216_b200 import tactic
    covered = set(tactic._SIGS) | {"tactic_index_destroy", "tactic_status_string", "tactic_last_error",
                                   "tactic_version"}
    assert set(_declared()) <= covered


def test_status_strings_and_version(L):
    assert L.tactic_status_string(0) == b"TACTIC_OK"
    assert L.tactic_status_string(6) == b"TACTIC_ERR_UNSUPPORTED"
    assert L.tactic_status_string(99) == b"TACTIC_ERR_UNKNOWN"
    assert b"sm_100a" in L.tactic_version()
    assert L.tactic_last_error() is not None


def test_kernels_are_sm100a_tensor_core_and_tma():
    """SASS evidence: tcgen05 MMA (UTCHMMA), TMEM loads (LDTM), bulk/TMA copies."""
    import shutil
    import subprocess
    from paper_2502_12216_b200 import build as B
    lib = B.build()
    exe = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(exe):
        pytest.skip("cuobjdump not available")
    sass = subprocess.run([exe, "-sass", lib], capture_output=True, text=True).stdout
    for mnem in ("UTCHMMA", "LDTM", "UBLKCP", "UTMALDG", "HMMA.16816.F32.BF16"):
        assert mnem in sass, mnem
    assert "sm_100a" in subprocess.run([exe, "-lelf", lib], capture_output=True, text=True).stdout
