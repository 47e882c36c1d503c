"""Golden vectors for the cost model from the REAL reference
(build container only): ``python tests/golden/make_golden_costmodel.py`` imports
``parconv`` from /root/reference/pkg/src and writes costmodel.npz next to this
script — step times of several plans / batches / parameter sets, predicted
days, and the reference's calibration of its Table-1 rows."""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg")
sys.path.insert(0, str(REF / "src"))

from parconv import costmodel as CM  # noqa: E402
from parconv.netdef import load_network  # noqa: E402
from parconv.schemes import ParallelPlan  # noqa: E402

OUT = Path(__file__).resolve().parent
CONFIGS = Path(__file__).resolve().parents[2] / "configs"
CROSS = (3, 6, 8, 10)
PLANS = [(1, 1, ()), (2, 1, ()), (4, 1, ()), (1, 2, CROSS), (2, 2, CROSS), (1, 2, (6,)), (4, 2, (6,))]
PARAMS = [(1e12, 4e9, 1e-3, 32.0), (2.0e12, 5.0e9, 0.004, 40.0), (8e14, 9e11, 1e-5, 16.0)]
TABLE1 = [((1, 1, ()), 10.5), ((1, 2, CROSS), 6.6), ((2, 1, ()), 7.0), ((4, 1, ()), 7.2), ((2, 2, CROSS), 4.8)]


def main():
    alex = load_network(CONFIGS / "alexnet.net")
    out = {}
    rows = []
    for pi, (d, m, c) in enumerate(PLANS):
        for batch in (128, 256, 512):
            for ki, prm in enumerate(PARAMS):
                cp = CM.CostParams(*prm, memory=180 * 10 ** 9)
                st = CM.step_time(ParallelPlan(d, m, c), alex, batch, cp)
                days = CM.predict_total(ParallelPlan(d, m, c), alex, batch, 90, CM.IMAGENET_TRAIN_SIZE, cp).days
                rows.append((pi, batch, ki, st.compute_seconds, st.comm_seconds, days))
    out["step_rows"] = np.array(rows, dtype=np.float64)
    fit = CM.calibrate([(ParallelPlan(d, m, c), days) for (d, m, c), days in TABLE1], alex)
    out["table1_fit"] = np.array([fit.throughput, fit.bandwidth, fit.latency, fit.b_half], dtype=np.float64)
    np.savez_compressed(OUT / "costmodel.npz", **out)
    print("wrote", OUT / "costmodel.npz", out["step_rows"].shape, out["table1_fit"])


if __name__ == "__main__":
    main()
