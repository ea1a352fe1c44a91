"""The C-ABI library loads and exports every symbol include/sdpc.h declares (no GPU needed)."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "sdpc.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(sdpc_[a-z0-9_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def libpath():
    import __graft_entry__
    __graft_entry__.build()
    from paper_1310_6919_b200 import LIB_PATH
    return LIB_PATH


def test_library_exports_every_declared_symbol(libpath):
    lib = ctypes.CDLL(libpath)
    names = declared_symbols()
    assert len(names) >= 18
    missing = [n for n in names if not hasattr(lib, n)]
    assert missing == []


def test_binding_covers_header(libpath):
    from paper_1310_6919_b200.sdpc import SYMBOLS
    assert sorted(SYMBOLS) == declared_symbols()


def test_status_strings_and_no_device(libpath):
    from paper_1310_6919_b200 import sdpc
    L = sdpc.lib()
    assert L.sdpc_status_string(2) == b"not positive definite"
    # no GPU here: creation must fail loudly (CUDA error), never fall back to the CPU
    import numpy as np
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(sdpc.SdpcError) as e:
        sdpc.Handle(1, 1, np.array([0, 0, 1]), np.array([0]), np.array([0]), np.array([1.0]), np.array([1.0]))
    assert e.value.status == sdpc.SDPC_ERR_CUDA
