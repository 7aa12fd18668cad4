"""The C-ABI library loads (no GPU needed) and exports every entry point that
include/blast.h declares; the ctypes prototypes cover exactly that set."""
import ctypes
import re
from pathlib import Path

import pytest

from paper_2507_03117_b200 import _lib

HEADER = Path(__file__).resolve().parent.parent / "include" / "blast.h"


def declared_symbols():
    text = HEADER.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(?:int|const char\*)\s+(blast_\w+)\s*\(", text)))


def test_header_parses():
    syms = declared_symbols()
    assert "blast_bspmm" in syms and "blast_topk_mask" in syms
    assert len(syms) >= 20


def test_library_exports_all_declared_symbols():
    lib = ctypes.CDLL(str(_lib.LIB_PATH))
    missing = [s for s in declared_symbols() if not hasattr(lib, s)]
    assert not missing, missing


def test_prototypes_match_header():
    assert sorted(_lib.EXPORTED) == declared_symbols()


def test_load_and_version():
    lib = _lib.load()
    assert lib.blast_version() == 1


def test_error_mapping():
    with pytest.raises(ValueError):
        _lib.check(_lib.EMISMATCH, "x")
    with pytest.raises(_lib.BlastError):
        _lib.check(_lib.ECUDA, "x")
