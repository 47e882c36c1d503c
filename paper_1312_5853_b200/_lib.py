"""ctypes binding of libpcb200.so (the C ABI declared in include/pc_b200.h).

No torch types cross this boundary: device pointers are plain integers
(``tensor.data_ptr()``), the stream is the raw ``cudaStream_t`` handle. A
missing or unloadable library raises immediately — there is no CPU or
eager-PyTorch fallback behind these calls.
"""

from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

from .errors import status_error

LIB_PATH = Path(__file__).resolve().parent / "libpcb200.so"

PC_FP32, PC_BF16, PC_TF32, PC_FP64 = 0, 1, 2, 3
PC_RELU, PC_WANT_DX, PC_WANT_DW, PC_MASK_DX, PC_WT_PRESET, PC_ZERO_TAIL16 = 1, 2, 4, 8, 16, 32

_vp, _i, _ll, _sz, _f, _d = C.c_void_p, C.c_int, C.c_longlong, C.c_size_t, C.c_float, C.c_double


class ConvGeom(C.Structure):
    _fields_ = [("B", _i), ("H", _i), ("W", _i), ("C", _i), ("N", _i), ("k", _i), ("stride", _i),
                ("pad", _i), ("Ho", _i), ("Wo", _i), ("cs", _i), ("cstride", _ll)]


class Mat(C.Structure):
    _fields_ = [("ptr", _vp), ("ld", _ll), ("cb", _ll), ("bstride", _ll)]


class SgdTensor(C.Structure):
    _fields_ = [("p", _vp), ("v", _vp), ("g", _vp), ("p_lowp", _vp), ("n", _ll)]


class SgdFuse(C.Structure):
    _fields_ = [("p", _vp), ("v", _vp), ("p_lowp", _vp), ("lr", _f), ("momentum", _f), ("weight_decay", _f)]


_P = C.POINTER
SIGNATURES = {
    "pc_last_error": (C.c_char_p, []),
    "pc_version": (_i, []),
    "pc_launch_count": (C.c_ulonglong, []),
    "pc_contraction_counts": (None, [_vp, _vp]),
    "pc_has_tcgen05": (_i, []),
    "pc_tf32_contractions": (C.c_ulonglong, []),
    "pc_debug_trace_gemm": (None, [_vp]),
    "pc_conv2d_forward": (_i, [_P(ConvGeom), _vp, _vp, _vp, _vp, _i, _i, _vp]),
    "pc_conv2d_backward_workspace": (_sz, [_P(ConvGeom), _i]),
    "pc_conv2d_backward": (_i, [_P(ConvGeom), _vp, _vp, _vp, _vp, _vp, _vp, _vp, _i, _i, _vp, _sz, _vp]),
    "pc_fc_forward": (_i, [_i, _i, _i, _P(Mat), _vp, _vp, _vp, _i, _i, _vp]),
    "pc_fc_backward_workspace": (_sz, [_i, _i, _i, _i]),
    "pc_fc_forward_workspace": (_sz, [_i, _i, _i, _i]),
    "pc_fc_forward_ex": (_i, [_i, _i, _i, _P(Mat), _vp, _vp, _vp, _i, _i, _vp, _sz, _vp]),
    "pc_fc_backward": (_i, [_i, _i, _i, _P(Mat), _vp, _vp, _P(Mat), _vp, _vp, _vp, _i, _i, _vp, _sz, _vp]),
    "pc_fc_backward_ex": (_i, [_i, _i, _i, _P(Mat), _vp, _vp, _P(Mat), _vp, _vp, _vp, _i, _i, _vp, _sz,
                               _P(SgdFuse), _vp]),
    "pc_conv2d_backward_ex": (_i, [_P(ConvGeom), _vp, _vp, _vp, _vp, _vp, _vp, _vp, _i, _i, _vp, _sz,
                                   _P(SgdFuse), _vp]),
    "pc_relu_forward": (_i, [_ll, _vp, _vp, _i, _vp]),
    "pc_relu_backward": (_i, [_ll, _vp, _vp, _vp, _i, _vp]),
    "pc_maxpool_forward": (_i, [_i, _i, _i, _i, _i, _i, _vp, _vp, _vp, _i, _vp]),
    "pc_maxpool_backward": (_i, [_i, _i, _i, _i, _i, _i, _vp, _vp, _vp, _vp, _i, _vp]),
    "pc_softmax_xent": (_i, [_i, _i, _vp, _vp, _d, _vp, _vp, _vp, _i, _vp]),
    "pc_sum_f64": (_i, [_i, _vp, _vp, _vp]),
    "pc_sgd_step": (_i, [_i, _vp, _ll, _f, _f, _f, _vp]),
    "pc_sgd_step_ex": (_i, [_i, _vp, _ll, _f, _f, _f, _i, _vp]),
    "pc_space_to_depth": (_i, [_i, _i, _i, _i, _i, _i, _i, _vp, _i, _vp, _vp]),
    "pc_mask_f32": (_i, [_ll, _vp, _vp, _vp]),
    "pc_maxpool_backward_bias_workspace": (_sz, [_i]),
    "pc_maxpool_backward_bias": (_i, [_i, _i, _i, _i, _i, _i, _vp, _vp, _vp, _vp, _i, _vp, _vp, _sz, _vp]),
    "pc_set_grid_cap": (_i, [_i]),
    "pc_conv2d_dgrad_weights": (_i, [_P(ConvGeom), _vp, _vp, _i, _vp]),
    "pc_bias_grad_workspace": (_sz, [_ll, _i, _i]),
    "pc_bias_grad": (_i, [_ll, _i, _vp, _i, _vp, _vp, _sz, _i, _vp]),
    "pc_space_to_depth_ex": (_i, [_i, _i, _i, _i, _i, _i, _i, _vp, _i, _i, _vp, _vp]),
    "pc_s2d_wgrad_finish": (_i, [_i, _i, _i, _vp, _vp, _vp, _vp]),
    "pc_lrn_forward": (_i, [_ll, _i, _i, _f, _f, _f, _vp, _vp, _i, _vp]),
    "pc_lrn_backward": (_i, [_ll, _i, _i, _f, _f, _f, _vp, _vp, _vp, _i, _vp]),
    "pc_space_to_depth_f32": (_i, [_i, _i, _i, _i, _i, _i, _i, _vp, _i, _i, _vp, _vp]),
    "pc_im2col_ex": (_i, [_i, _i, _i, _i, _i, _i, _i, _i, _vp, _i, _vp, _i, _vp]),
    "pc_enable_peer_access": (_i, [_i]),
    "pc_copy_async": (_i, [_vp, _vp, _sz, _vp]),
    "pc_softmax_xent_loss": (_i, [_i, _i, _vp, _vp, _d, _vp, _vp, _vp, _vp, _vp, _i, _vp]),
    "pc_synthetic_rows": (_i, [_i, _i, _ll, C.c_ulonglong, _i, _vp, _i, _f, _vp, _i, _vp]),
    "pc_gather_rows": (_i, [_i, _ll, _vp, _vp, _vp, _vp]),
    "pc_dropout": (_i, [_i, _i, _i, _i, _i, _i, _ll, C.c_ulonglong, _vp, _i, C.c_ulonglong, _f, _vp, _vp, _i, _vp]),
    "pc_counter_add": (_i, [_vp, _ll, _vp]),
    "pc_nchw_to_nhwc": (_i, [_i, _i, _i, _i, _i, _vp, _vp, _i, _vp]),
    "pc_im2col": (_i, [_i, _i, _i, _i, _i, _i, _i, _i, _vp, _i, _vp, _vp]),
    "pc_sum_buffers": (_i, [_i, _ll, _vp, _vp, _i, _vp]),
    "pc_cast": (_i, [_ll, _vp, _i, _vp, _i, _vp]),
    "pc_scale": (_i, [_ll, _vp, _vp, _f, _i, _vp]),
}


class _Lib:
    def __init__(self, path: Path):
        if not path.exists():
            raise ImportError(f"{path} is missing: build it with `python -c 'import __graft_entry__ as g; "
                              "g.build()'` (make -C paper_1312_5853_b200/csrc)")
        self.path = path
        self.dll = C.CDLL(str(path), mode=os.RTLD_NOW | getattr(os, "RTLD_GLOBAL", 0))
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(self.dll, name)
            fn.restype, fn.argtypes = res, args

    def call(self, name: str, *args):
        rc = getattr(self.dll, name)(*args)
        if rc != 0:
            msg = self.dll.pc_last_error().decode(errors="replace")
            raise status_error(rc, f"{name}: {msg}")
        return rc

    def raw(self, name: str):
        return getattr(self.dll, name)


_LIB: _Lib | None = None


def lib() -> _Lib:
    global _LIB
    if _LIB is None:
        _LIB = _Lib(LIB_PATH)
    return _LIB
