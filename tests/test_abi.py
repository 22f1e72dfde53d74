"""The C-ABI library builds, loads without a GPU, and exports exactly the
entry points include/mrep.h declares; the product fails loudly without a
device (no CPU fallback)."""
import os
import re

import pytest

from conftest import ROOT


def header_symbols():
    src = open(os.path.join(ROOT, "include", "mrep.h")).read()
    return sorted(set(re.findall(r"MREP_API\s+[\w\s\*]+?\b(mrep_\w+)\s*\(", src)))


def test_header_declares_expected_entries():
    syms = header_symbols()
    for must in ("mrep_project", "mrep_project_host", "mrep_project_block", "mrep_table_pack",
                 "mrep_decompose", "mrep_approx_run", "mrep_quartic_roots"):
        assert must in syms


def test_library_exports_every_declared_symbol():
    from paper_2504_11498_b200 import _lib
    lib = _lib.load_library()
    for s in header_symbols():
        assert hasattr(lib, s), s


def test_binding_table_matches_header():
    from paper_2504_11498_b200 import _lib
    assert sorted(_lib.exported_symbols()) == header_symbols()


def test_library_is_sm100a():
    import subprocess
    from paper_2504_11498_b200 import _lib
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _lib.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_cpu_calls_without_gpu_are_loud():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    from paper_2504_11498_b200 import _lib, fixtures, project_points
    lib = _lib.load_library()
    assert lib.mrep_version() >= 100
    with pytest.raises(RuntimeError):
        project_points(fixtures.single_span_cubic(), [[0.5, 0.5]])


def test_table_bytes():
    from paper_2504_11498_b200 import _lib
    lib = _lib.load_library()
    # header 64 + 32 doubles per cubic + 6 per box (8-ary levels incl. root)
    # + the float copy of every box (6 floats = 3 doubles) + the compact seam
    # block (3 doubles per seam), rounded to 4 doubles, + the tensor-core
    # B fragments (32 doubles per cubic, two zero fragments of slack)
    def expect(S, boxes):
        n = 64 + 32 * S + 9 * boxes + 3 * (S + 1)
        return (((n + 3) // 4) * 4 + 32 * (S + 2)) * 8
    assert lib.mrep_table_bytes(1) == expect(1, 2)
    assert lib.mrep_table_bytes(510) == expect(510, 510 + 64 + 8 + 1)
    assert lib.mrep_table_bytes(0) < 0
