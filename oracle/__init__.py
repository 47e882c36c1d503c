"""TEST INFRASTRUCTURE ONLY — the CPU oracle for the parity gate.

This package is a float64 numpy restatement of the reference's training
step (`/root/reference/pkg/src/parconv/kernels.py` and
`schemes.py:342-569`). It is imported only by ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs, always as the checker or the timed CPU baseline,
never as the product path. The product package ``paper_1312_5853_b200``
never imports it.

Pinning: ``tests/test_oracle_golden.py`` checks every function here against
golden vectors produced by the real reference (``tests/golden/make_golden.py``
imports ``parconv`` from ``/root/reference/pkg/src`` in the build container
and writes ``tests/golden/*.npz``), plus the reference's own known-answer
tests re-stated (`pkg/tests/test_kernels.py`). Parity is therefore pinned.
"""

from .ref_kernels import (  # noqa: F401
    conv2d_backward,
    conv2d_forward,
    fc_backward,
    fc_forward,
    maxpool_backward,
    maxpool_forward,
    relu_backward,
    relu_forward,
    sgd_step,
    softmax_xent,
    softmax_xent_scaled,
)
from .ref_engine import (  # noqa: F401
    OracleFabric,
    column_fwd_bwd,
    reference_step,
)
