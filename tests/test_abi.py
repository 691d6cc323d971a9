"""The C-ABI library loads and exports every symbol include/grinder_b200.h
declares (no compute calls: runs on CPU)."""

from __future__ import annotations

import ctypes
import re
from pathlib import Path

from paper_2605_11517_b200 import _lib

HEADER = Path(__file__).resolve().parents[1] / "include" / "grinder_b200.h"


def header_functions() -> list[str]:
    text = re.sub(r"/\*.*?\*/", "", HEADER.read_text(), flags=re.S)
    return sorted(set(re.findall(r"\b(grd_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_header_symbol():
    names = header_functions()
    assert len(names) >= 20
    lib = ctypes.CDLL(str(_lib.LIB_PATH))
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing


def test_binding_table_matches_header():
    assert sorted(_lib.SIGNATURES) == header_functions()


def test_abi_version_and_error_slot():
    L = _lib.lib()
    assert L.grd_abi_version() == 1
    assert L.grd_last_error() is not None


def test_library_is_sm100a():
    data = _lib.LIB_PATH.read_bytes()
    assert b"sm_100a" in data


def test_integration_doc_struct_matches_the_abi():
    """INTEGRATION.md's reference-side ctypes binding lists GrdAggArgs field
    for field (a stale copy would make the library read past the struct)."""
    import re
    from pathlib import Path
    from paper_2605_11517_b200 import _lib
    doc = (Path(__file__).resolve().parents[1] / "INTEGRATION.md").read_text()
    body = doc[doc.index("class GrdAggArgs"):doc.index("def aggregate_mean")]
    names = re.findall(r'\("(\w+)", ctypes\.c_', body)
    assert names == [f[0] for f in _lib.GrdAggArgs._fields_]
