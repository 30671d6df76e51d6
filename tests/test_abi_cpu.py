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


def test_library_sample_constants_equal_the_oracle_rule(L):
    """tactic_sample_constants (host logic, no device) against the oracle's ppm rule
    (readings 8-10) for default and custom fractions over many n, and its
    argument validation."""
    import numpy as np

    from oracle import tactic_oracle as O
    from paper_2502_12216_b200 import tactic
    rng = np.random.default_rng(5)
    ns = list(range(1, 3000)) + [int(x) for x in rng.integers(3000, 1 << 20, 2000)]
    fracs = [None, dict(exact_frac=0.01, p1=0.2, p2=0.5, window_half_frac=0.01),
             dict(exact_frac=0.015, p1=0.25, p2=0.75, window_half_frac=0.001),
             dict(exact_frac=0.05, p1=0.1, p2=0.9, window_half_frac=0.0005)]
    for f in fracs:
        for n in ns[::3]:
            got = tactic.sample_constants(n, f)
            ref = O.sample_constants(n, **(f or {}))
            assert {k: got[k] for k in ref} == ref, (n, f)
            assert got["slots"] == (n if ref["fallback"] else ref["N"] + 2 * (2 * ref["w"] + 1))
    for bad in [dict(p1=0.6, p2=0.1), dict(p2=1.0), dict(exact_frac=-0.1)]:
        with pytest.raises(tactic.TacticError):
            tactic.sample_constants(1000, bad)


def test_ctypes_structs_match_the_header(tmp_path):
    """The binding's ctypes mirrors of the boundary's structs have the C layout: a C program
    compiled against include/tactic.h (gcc) prints sizeof / offsetof of every field."""
    import ctypes
    import shutil
    import subprocess
    gcc = shutil.which("gcc")
    if gcc is None:
        pytest.skip("gcc not available")
    from paper_2502_12216_b200 import tactic
    structs = {"tactic_kv_desc_t": tactic.KvDesc, "tactic_params_t": tactic.Params,
               "tactic_sample_constants_t": tactic.SampleConstants, "tactic_index_info_t": tactic.IndexInfo}
    lines = ['#include <stdio.h>', '#include <stddef.h>', f'#include "{HEADER}"', "int main(void) {"]
    for cname, py in structs.items():
        lines.append(f'  printf("{cname} size %zu\\n", sizeof({cname}));')
        for f, _ in py._fields_:
            lines.append(f'  printf("{cname} {f} %zu\\n", offsetof({cname}, {f}));')
    lines += ["  return 0;", "}"]
    src = tmp_path / "layout.c"
    src.write_text("\n".join(lines) + "\n")
    exe = tmp_path / "layout"
    subprocess.run([gcc, "-std=c99", "-o", str(exe), str(src)], check=True, capture_output=True)
    got = {}
    for ln in subprocess.run([str(exe)], check=True, capture_output=True, text=True).stdout.splitlines():
        c, f, v = ln.split()
        got[(c, f)] = int(v)
    for cname, py in structs.items():
        assert got[(cname, "size")] == ctypes.sizeof(py), cname
        for f, _ in py._fields_:
            assert got[(cname, f)] == getattr(py, f).offset, (cname, f)
