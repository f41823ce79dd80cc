"""CPU checks of the C-ABI boundary: libprism.so loads and exports every
entry point include/prism.h declares (no compute calls without a GPU)."""

from __future__ import annotations

import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared() -> list[str]:
    with open(os.path.join(ROOT, "include", "prism.h")) as fh:
        text = fh.read()
    return sorted(set(re.findall(r"\b(prism_[a-z_0-9]+)\s*\(", text)))


def test_header_declares_entry_points():
    names = _declared()
    for must in ("prism_tree_create", "prism_match", "prism_insert", "prism_release", "prism_evict",
                 "prism_set_protection", "prism_note_active", "prism_admit_wave", "prism_qas_round"):
        assert must in names


def test_library_exports_every_declared_symbol():
    from paper_2605_08581_b200 import build as B

    B.build(verbose=False)
    lib = ctypes.CDLL(B.LIB)
    missing = [n for n in _declared() if not hasattr(lib, n)]
    assert not missing, f"missing exports: {missing}"


def test_no_cpu_fallback_without_device():
    from paper_2605_08581_b200 import _lib

    if _lib.lib().prism_device_count() > 0:
        pytest.skip("a CUDA device is present")
    from paper_2605_08581_b200.dart import DeviceRadixCache
    from paper_2605_08581_b200.types import CacheConfig

    with pytest.raises(_lib.PrismError):
        DeviceRadixCache(CacheConfig(capacity_tokens=100))
