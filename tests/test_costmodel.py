"""Cost model: parity with the reference's model on golden vectors
(tests/golden/make_golden_costmodel.py), the reference's own behavioural checks
(`pkg/tests/test_costmodel.py`), and the B200 compute-term recalibration."""

import math
from pathlib import Path

import numpy as np
import pytest

from paper_1312_5853_b200 import costmodel as CM
from paper_1312_5853_b200.errors import CalibrationError, InfeasiblePlanError, ValidationError
from paper_1312_5853_b200.netdef import load_network
from paper_1312_5853_b200.plan import ParallelPlan

ROOT = Path(__file__).resolve().parents[1]
GOLD = np.load(ROOT / "tests" / "golden" / "costmodel.npz")
ALEX = load_network(ROOT / "configs" / "alexnet.net")
CROSS = (3, 6, 8, 10)
PLANS = [(1, 1, ()), (2, 1, ()), (4, 1, ()), (1, 2, CROSS), (2, 2, CROSS), (1, 2, (6,)), (4, 2, (6,))]
PARAMS = [(1e12, 4e9, 1e-3, 32.0), (2.0e12, 5.0e9, 0.004, 40.0), (8e14, 9e11, 1e-5, 16.0)]
TABLE1 = [(ParallelPlan(1, 1), 10.5), (ParallelPlan(1, 2, CROSS), 6.6), (ParallelPlan(2, 1), 7.0),
          (ParallelPlan(4, 1), 7.2), (ParallelPlan(2, 2, CROSS), 4.8)]


def test_step_time_matches_reference_golden():
    for pi, batch, ki, comp, comm, days in GOLD["step_rows"]:
        d, m, c = PLANS[int(pi)]
        cp = CM.CostParams(*PARAMS[int(ki)], memory=180 * 10 ** 9)
        st = CM.step_time(ParallelPlan(d, m, c), ALEX, int(batch), cp)
        assert st.compute_seconds == pytest.approx(comp, rel=1e-12)
        assert st.comm_seconds == pytest.approx(comm, rel=1e-12, abs=1e-15)
        got = CM.predict_total(ParallelPlan(d, m, c), ALEX, int(batch), 90, CM.IMAGENET_TRAIN_SIZE, cp).days
        assert got == pytest.approx(days, rel=1e-12)


@pytest.fixture(scope="module")
def table1_fit():
    return CM.calibrate(TABLE1, ALEX)


def test_calibrate_matches_reference_fit(table1_fit):
    got = [table1_fit.throughput, table1_fit.bandwidth, table1_fit.latency, table1_fit.b_half]
    np.testing.assert_allclose(got, GOLD["table1_fit"], rtol=1e-6)


def test_calibrate_reproduces_table1_within_10_percent(table1_fit):
    for plan, days in TABLE1:
        pred = CM.predict_total(plan, ALEX, 256, 100, CM.IMAGENET_TRAIN_SIZE, table1_fit).days
        assert abs(pred - days) / days < 0.10, (plan.describe(), pred, days)


def test_calibrate_needs_four_observations():
    with pytest.raises(CalibrationError):
        CM.calibrate(TABLE1[:3], ALEX)


def test_efficiency_curve():
    assert CM.efficiency(32, 32) == 0.5
    assert CM.efficiency(1e9, 1) > 0.999
    with pytest.raises(ValidationError):
        CM.efficiency(0, 1)


def test_memory_infeasible():
    with pytest.raises(InfeasiblePlanError):
        CM.step_time(ParallelPlan(1, 1), ALEX, 256, CM.CostParams(1e12, 1e9, 0.0, 1.0, memory=1024))


def test_cost_params_round_trip(tmp_path):
    cp = CM.CostParams(throughput=1.25e12, bandwidth=3.5e9, latency=0.00125, b_half=17.5, memory=123456)
    CM.save_cost_params(cp, tmp_path / "c.txt")
    assert CM.load_cost_params(tmp_path / "c.txt") == cp
    (tmp_path / "bad.txt").write_text("throughput 1\n")
    with pytest.raises(ValidationError):
        CM.load_cost_params(tmp_path / "bad.txt")


def test_b200_cost_file_loads_and_predicts_the_measured_step():
    """configs/b200.cost (written by tools/calibrate_b200.py from measured device
    steps) reproduces its own calibration rows within 10%."""
    path = ROOT / "configs" / "b200.cost"
    cp = CM.load_cost_params(path)
    assert cp.memory == CM.B200_MEMORY
    rows = [tuple(float(v) for v in ln.split()[2:4]) for ln in path.read_text().splitlines()
            if ln.startswith("# step")]
    assert len(rows) >= 2
    for b, sec in rows:
        pred = CM.step_time(ParallelPlan(1, 1), ALEX, int(b), cp).step_seconds
        assert abs(pred - sec) / sec < 0.10, (b, pred, sec)


def test_calibrate_compute_recovers_known_params():
    true = CM.CostParams(throughput=7.5e14, bandwidth=CM.B200_LINK_BANDWIDTH, latency=CM.B200_MESSAGE_LATENCY,
                         b_half=24.0, memory=CM.B200_MEMORY)
    rows = [(b, CM.step_time(ParallelPlan(1, 1), ALEX, b, true).step_seconds) for b in (32, 64, 128, 256)]
    fit = CM.calibrate_compute(rows, ALEX)
    assert fit.throughput == pytest.approx(true.throughput, rel=1e-3)
    assert fit.b_half == pytest.approx(true.b_half, rel=1e-3)
    with pytest.raises(CalibrationError):
        CM.calibrate_compute(rows[:1], ALEX)
