"""The C-ABI library loads and exports every symbol include/gqm3d.h declares
(no device calls: runs without a GPU)."""

import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared():
    src = open(os.path.join(ROOT, "include", "gqm3d.h")).read()
    return sorted(set(re.findall(r"\b(gq_[a-z_0-9]+)\s*\(", src)))


def test_header_declares_the_boundary():
    names = declared()
    for n in ("gq_create", "gq_destroy", "gq_refine", "gq_export_mesh", "gq_export_constraints",
              "gq_export_rounds", "gq_export_skipped", "gq_quality", "gq_last_error", "gq_batch"):
        assert n in names


def test_library_exports_every_declared_symbol():
    from paper_1903_03406_b200 import build
    path = build.SO
    if not os.path.exists(path):
        pytest.skip("libgqm3d.so not built (run __graft_entry__.build())")
    lib = ctypes.CDLL(path)
    for n in declared():
        assert hasattr(lib, n), n


def test_python_binding_names_match():
    from paper_1903_03406_b200 import _native
    assert set(_native.EXPORTS) <= set(declared())
