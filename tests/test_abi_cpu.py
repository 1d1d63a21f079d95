"""The drop-in boundary (CPU): libflexmoe_b200.so loads without a GPU and
exports every entry point include/flexmoe_b200.h declares; host-only entry
points honour the reference's error convention (status codes + messages)."""
import ctypes as C
import re
from pathlib import Path

import numpy as np
import pytest

from paper_2304_03946_b200 import _lib as L

HEADER = Path(__file__).resolve().parents[1] / "include" / "flexmoe_b200.h"


def declared_symbols():
    text = HEADER.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:const\s+)?\w+\*?\s+\*?(fm_\w+)\s*\(", text, flags=re.M)))


def test_header_declares_the_boundary():
    syms = declared_symbols()
    for must in ["fm_route_counts", "fm_route_counts_device", "fm_balance_ratio",
                 "fm_static_ep_kept", "fm_largest_remainder_round", "fm_grouped_gemm",
                 "fm_layer_create", "fm_layer_forward", "fm_layer_backward", "fm_layer_route",
                 "fm_layer_dispatch", "fm_layer_expert_forward", "fm_layer_combine"]:
        assert must in syms, must


def test_library_exports_every_declared_symbol():
    lib = L.lib()
    missing = [s for s in declared_symbols() if not hasattr(lib, s)]
    assert not missing, missing
    # and the Python binding knows every one of them
    assert set(declared_symbols()) <= set(L.exported_symbols())


def test_version_and_error_convention():
    lib = L.lib()
    assert b"sm_100a" in lib.fm_version()
    D = np.array([[5, 0]], np.int64)
    cnt = np.zeros((1, 2), np.int32)
    flows = np.zeros((1, 2, 2), np.int64)
    st = lib.fm_route_counts(D.ctypes.data, cnt.ctypes.data, 1, 2, flows.ctypes.data)
    assert st == L.FM_ERR_INVALID_ARGUMENT
    assert b"expert 0 has demand but no replica" in lib.fm_last_error()
    with pytest.raises(L.InvalidArgument):
        L.call("fm_route_counts", D.ctypes.data, cnt.ctypes.data, 1, 2, flows.ctypes.data)
    # balance_ratio on an empty plan: invalid_argument with the reference's text
    r = C.c_double()
    assert lib.fm_balance_ratio(flows.ctypes.data, 1, 2, C.byref(r)) == L.FM_ERR_INVALID_ARGUMENT
    assert b"zero total tokens" in lib.fm_last_error()
