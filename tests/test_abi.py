"""The C-ABI library loads without a GPU and exports every entry point that
include/fastecot.h declares (no compute calls)."""

import ctypes
import re
from pathlib import Path

import pytest

from paper_2506_07639_b200 import engine as E

HEADER = Path(__file__).resolve().parents[1] / "include" / "fastecot.h"


def declared_functions() -> list[str]:
    text = HEADER.read_text()
    return sorted(set(re.findall(r"^\s*(?:int|const char\*)\s+(fe_\w+)\s*\(", text, flags=re.M)))


def test_header_declares_the_binding_table():
    names = declared_functions()
    assert len(names) >= 20
    assert set(names) == set(E.EXPORTS)


def test_library_exports_every_declared_symbol():
    lib = E.load_library()
    missing = [n for n in declared_functions() if not hasattr(lib, n)]
    assert missing == []


def test_errors_surface_through_last_error_without_a_gpu():
    lib = E.load_library()
    rc = lib.fe_seq_create(None, ctypes.byref(ctypes.c_int32()))
    assert rc != 0
    assert b"null engine" in lib.fe_last_error()


def test_config_struct_matches_header():
    # fe_config: 10 int32 + 2 float ... laid out without padding
    text = HEADER.read_text()
    body = text[text.index("typedef struct fe_config"):text.index("} fe_config;")]
    fields = re.findall(r"(int32_t|float)\s+([\w ,]+);", body)
    names = [n.strip() for _, group in fields for n in group.split(",")]
    assert names == [f[0] for f in E.FeConfig._fields_]
    assert ctypes.sizeof(E.FeConfig) == 4 * len(names)


def test_product_path_has_no_cpu_fallback(monkeypatch, tmp_path):
    monkeypatch.setattr(E, "_lib", None)
    with pytest.raises(E.EngineError):
        E.load_library(tmp_path / "missing.so")
