"""CPU checks of the drop-in boundary: the C-ABI library loads and exports
every symbol declared in include/pc_b200.h (no compute calls without a GPU)."""

import ctypes
import re

from conftest import ROOT


def declared_symbols():
    text = (ROOT / "include" / "pc_b200.h").read_text()
    return sorted(set(re.findall(r"PC_API\s+[\w\s\*]+?\b(pc_\w+)\s*\(", text)))


def test_header_declares_reference_ops():
    names = declared_symbols()
    for want in ("pc_conv2d_forward", "pc_conv2d_backward", "pc_fc_forward", "pc_fc_backward",
                 "pc_relu_forward", "pc_relu_backward", "pc_maxpool_forward", "pc_maxpool_backward",
                 "pc_softmax_xent", "pc_sgd_step"):
        assert want in names


def test_library_exports_every_declared_symbol():
    from paper_1312_5853_b200._lib import LIB_PATH, SIGNATURES
    dll = ctypes.CDLL(str(LIB_PATH))
    for name in declared_symbols():
        assert hasattr(dll, name), name
        assert name in SIGNATURES, f"{name} has no ctypes signature"
    dll.pc_version.restype = ctypes.c_int
    assert dll.pc_version() == 1
    dll.pc_last_error.restype = ctypes.c_char_p
    assert dll.pc_last_error() == b""
