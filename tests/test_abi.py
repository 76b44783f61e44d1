"""The C-ABI library loads without a GPU and exports every entry point
include/rlx.h declares; the ctypes mirror matches the header."""

import ctypes as C
import os
import re

import pytest

from helpers import ROOT
from paper_2604_23838_b200 import abi

HEADER = os.path.join(ROOT, "include", "rlx.h")


def _declared():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:int|void|const char\*)\s+(rlx_\w+)\s*\(", src, re.M)))


def test_header_declares_exported_set():
    assert sorted(abi.EXPORTED) == _declared()


def test_abi_version_matches_header():
    src = open(HEADER).read()
    assert int(re.search(r"#define RLX_ABI_VERSION (\d+)", src).group(1)) == abi.RLX_ABI_VERSION
    for name in ("RLX_F_REUSE_PLAN", "RLX_F_SHARD", "RLX_NALLOC", "RLX_NPARTNER", "RLX_MAX_MEMBERS"):
        v = int(re.search(rf"#define {name} (\d+)", src).group(1))
        assert v == getattr(abi, name), name


def test_library_loads_and_exports():
    from paper_2604_23838_b200 import native

    if not os.path.exists(native.LIB_PATH):
        pytest.skip("librlx.so not built")
    lib = C.CDLL(native.LIB_PATH)
    for sym in abi.EXPORTED:
        assert hasattr(lib, sym), sym
    abi.bind(lib)
    assert lib.rlx_abi_version() == abi.RLX_ABI_VERSION


def test_no_cpu_fallback_without_device():
    """On a box without a CUDA device the evaluator refuses to run."""
    import torch

    from paper_2604_23838_b200 import native

    if torch.cuda.is_available() or not os.path.exists(native.LIB_PATH):
        pytest.skip("has a GPU / library not built")
    with pytest.raises(native.NativeUnavailable):
        native.Evaluator(None)


def test_struct_sizes():
    # RlxDecision/RlxAction layouts are part of the ABI (checked against the
    # compiled offsets in tests/test_gpu_parity.py on the device)
    assert C.sizeof(abi.RlxAction) == 4 * (6 + abi.RLX_MAX_MEMBERS)
    assert C.sizeof(abi.RlxKey) == 32
