"""The C-ABI library loads without a GPU and exports every symbol include/geer.h declares."""

import ctypes
import os
import re

from paper_2505_24053_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    with open(os.path.join(ROOT, "include", "geer.h")) as f:
        text = f.read()
    return sorted(set(re.findall(r"^\s*(?:[\w\s\*]+?)\b(geer_\w+)\s*\(", text, flags=re.M)))


def test_header_declares_the_bound_symbols():
    assert sorted(_lib.EXPORTED) == declared_symbols()


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(_lib.LIB_PATH)
    missing = [s for s in declared_symbols() if not hasattr(lib, s)]
    assert not missing, missing


def test_abi_version_and_struct_layouts():
    lib = _lib.load()
    assert lib.geer_abi_version() == 1
    assert ctypes.sizeof(_lib.GeerCamera) == 16 + 8 * (9 + 3 + 6 + 4)
    assert ctypes.sizeof(_lib.GeerConfig) == 8 * 4 + 16
    assert ctypes.sizeof(_lib.GeerScene) == 16 + 5 * 8


def test_errors_without_device_are_reported_not_crashed():
    # with no GPU, context creation must fail loudly (no CPU fallback)
    import torch

    if torch.cuda.is_available():
        return
    lib = _lib.load()
    assert not lib.geer_create(0)
    assert _lib.last_error()
