"""The two-accumulator im2col GEMM (A_IM2COL_K2, csrc/umma_gemm.cu) computes the
same tiles as the one-accumulator A_IM2COL_K in the same k-block order, so the
bf16 conv forward (bias + ReLU epilogue) and data gradient (ReLU-mask epilogue)
must be bit-identical between PC_K2=2 (always) and PC_K2=0 (never), including
partial 512-row tiles (B = 7, 20). The default (PC_K2=1) picks it per layer;
its numerics are covered against the oracle by the AlexNet b256 step tests."""

import os
import subprocess
import sys

import numpy as np
import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu


def test_k2_bit_identical_to_k1(tmp_path):
    res = {}
    for mode in ("0", "2"):
        out = tmp_path / f"k{mode}.npz"
        env = dict(os.environ, PC_K2=mode)
        r = subprocess.run([sys.executable, str(ROOT / "tests" / "k2_conv_worker.py"), str(out)], env=env,
                           capture_output=True, text=True, timeout=600)
        assert r.returncode == 0, r.stderr[-2000:]
        res[mode] = np.load(out)
    for key in res["0"].files:
        assert np.array_equal(res["0"][key], res["2"][key]), key
