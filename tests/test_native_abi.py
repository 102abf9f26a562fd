"""The C-ABI library loads (no GPU needed for dlopen) and exports exactly
the entry points include/*.h declares, with matching ctypes signatures."""

from __future__ import annotations

import re
import subprocess
from pathlib import Path

import pytest

from paper_2404_06430_b200 import native

ROOT = Path(__file__).resolve().parent.parent


def _declared() -> dict[str, int]:
    names = {}
    for h in (ROOT / "include").glob("*.h"):
        text = re.sub(r"/\*.*?\*/", "", h.read_text(), flags=re.S)
        for m in re.finditer(r"\b(?:void|int|int64_t|const char\*)\s+(fb_\w+)\s*\(([^)]*)\)\s*;", text):
            args = [a for a in m.group(2).split(",") if a.strip() and a.strip() != "void"]
            names[m.group(1)] = len(args)
    return names


def test_header_declares_entry_points():
    assert len(_declared()) >= 10


def test_library_exports_every_declared_symbol():
    if not native.LIB_PATH.exists():
        pytest.skip("library not built (run __graft_entry__.build())")
    out = subprocess.run(["nm", "-D", "--defined-only", str(native.LIB_PATH)], capture_output=True, text=True,
                         check=True).stdout
    exported = {line.split()[-1] for line in out.splitlines() if " T " in line}
    missing = set(_declared()) - exported
    assert not missing, f"declared but not exported: {sorted(missing)}"


def test_ctypes_signatures_match_header():
    declared = _declared()
    assert set(native.SIGNATURES) == set(declared)
    for name, n in declared.items():
        assert len(native.SIGNATURES[name][1]) == n, name


def test_library_loads_and_reports_abi():
    if not native.LIB_PATH.exists():
        pytest.skip("library not built")
    lib = native.load_library()
    assert lib.fb_abi_version() == native.ABI_VERSION
    assert lib.fb_last_error() is not None
    # size queries need no device
    assert lib.fb_weighted_sum_workspace_bytes(1000, 10_000_000) == 0
