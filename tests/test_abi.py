"""The C-ABI library loads without a GPU and exports every symbol the
header declares (no compute calls here)."""

import ctypes
import os
import re

from conftest import ROOT
from paper_2505_13723_b200 import _native

HEADER = os.path.join(ROOT, "include", "sapgp_b200.h")


def declared():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:int|size_t|long long \*|long long|const char \*|int \*)\s*(sap_\w+)\(", text, re.M)))


def test_header_declares_the_boundary():
    names = declared()
    for must in ("sap_krows_times", "sap_ktile", "sap_grad_gather", "sap_pq_update",
                 "sap_prepare_points", "sap_gather_points", "sap_combine", "sap_last_error"):
        assert must in names


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(_native.LIB_PATH)
    for name in declared():
        assert hasattr(lib, name), name
    assert set(declared()) == set(_native.SIGNATURES)


def test_abi_version_and_workspace_query():
    lib = _native.load()
    assert lib.sap_abi_version() == _native.ABI_VERSION
    ws = lib.sap_krows_workspace(2000, 65, 1_000_000)
    assert ws > 0 and ws % 4 == 0
    assert lib.sap_krows_workspace(2000, 65, 64) == 0  # too few tiles to split


def test_contract_errors_need_no_device():
    lib = _native.load()
    rc = lib.sap_krows_times(None, None, 12, 10, None, 0, None, None, None, 0, 9, None, None, 10,
                             65, 1.0, 0.0, 0, 1.0, None, 65, 0, None, 0, None)
    assert rc == _native.SAP_ERR_CONTRACT
    assert b"bad shape" in lib.sap_last_error()
