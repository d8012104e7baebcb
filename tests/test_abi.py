"""The C-ABI library loads on a GPU-less host and exports every symbol that
include/rlb.h declares (no compute calls here)."""
import ctypes
import os
import re

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    text = open(os.path.join(ROOT, "include", "rlb.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(rlb_[a-z_0-9]+)\s*\(", text)))


def test_header_declares_the_path_entry_points():
    syms = header_symbols()
    for name in ("rlb_instance_create", "rlb_submit", "rlb_submit_varlen", "rlb_step",
                 "rlb_cancel", "rlb_export_partials", "rlb_status", "rlb_load_weights",
                 "rlb_ipc_handle", "rlb_ipc_open", "rlb_last_error"):
        assert name in syms


def test_library_exports_every_declared_symbol():
    from paper_2510_19225_b200 import _lib
    lib = _lib.lib()
    missing = [s for s in header_symbols() if not hasattr(lib, s)]
    assert not missing, missing


def test_python_binding_covers_header():
    from paper_2510_19225_b200 import _lib
    assert sorted(_lib.EXPORTED) == header_symbols()


def test_struct_sizes_match_header_layout():
    from paper_2510_19225_b200 import _lib
    assert ctypes.sizeof(_lib.ModelCfg) == 10 * 4
    assert ctypes.sizeof(_lib.EngineCfg) == 8 * 4
    assert ctypes.sizeof(_lib.Stats) == 8 * 8
    assert ctypes.sizeof(_lib.PullStats) == 16


def test_product_path_has_no_oracle_import():
    """The product package never imports the oracle (test infrastructure)."""
    pkg = os.path.join(ROOT, "paper_2510_19225_b200")
    for name in os.listdir(pkg):
        if name.endswith(".py"):
            src = open(os.path.join(pkg, name)).read()
            assert "oracle" not in re.findall(r"^\s*(?:from|import)\s+(\w+)", src, re.M), name
