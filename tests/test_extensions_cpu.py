"""Extension layers (absent from the reference): LRN and dropout.
CPU checks of their float64 definition (oracle) and of the dropout stream
contract: LRN backward vs central differences; keep rate; masks identical
under every data/model-parallel plan (counter-based SplitMix64 over the dense
activation), so DP/MP/hybrid stay equivalent to the single-worker step."""

import numpy as np
import pytest

from conftest import CONFIGS


def test_lrn_backward_matches_central_differences():
    from oracle import ref_kernels as K
    rs = np.random.RandomState(0)
    x, g = rs.randn(2, 9, 3, 2), rs.randn(2, 9, 3, 2)
    args = (5, 2.0, 0.2, 0.75)
    gx = K.lrn_backward(x, g, *args)
    num = np.zeros_like(x)
    eps = 1e-6
    for idx in np.ndindex(x.shape):
        xp, xm = x.copy(), x.copy()
        xp[idx] += eps
        xm[idx] -= eps
        num[idx] = ((K.lrn_forward(xp, *args) - K.lrn_forward(xm, *args)) * g).sum() / (2 * eps)
    assert np.abs(num - gx).max() / np.abs(num).max() < 1e-7


def test_lrn_known_answer():
    from oracle import ref_kernels as K
    x = np.zeros((1, 3, 1, 1))
    x[0, :, 0, 0] = [1.0, 2.0, 3.0]
    y = K.lrn_forward(x, size=3, k=1.0, alpha=1.0, beta=1.0)
    assert np.allclose(y[0, :, 0, 0], [1 / (1 + 5), 2 / (1 + 14), 3 / (1 + 13)])


def test_dropout_stream_rate_and_determinism():
    from paper_1312_5853_b200 import rng
    idx = np.arange(200_000)
    k1 = rng.dropout_keep(7, 3, 9, idx, 0.5)
    assert abs(k1.mean() - 0.5) < 0.01
    assert np.array_equal(k1, rng.dropout_keep(7, 3, 9, idx, 0.5))
    assert not np.array_equal(k1, rng.dropout_keep(7, 4, 9, idx, 0.5))      # fresh mask each step
    assert not np.array_equal(k1, rng.dropout_keep(7, 3, 10, idx, 0.5))     # and each layer
    assert rng.dropout_keep(7, 3, 9, idx, 0.0).all()
    # counter-based: a slice draws the same as the full stream
    assert np.array_equal(rng.dropout_keep(7, 3, 9, idx[5000:7000], 0.5), k1[5000:7000])


def test_parse_extension_layers_and_errors():
    import paper_1312_5853_b200 as P
    net = P.load_network(CONFIGS / "tinynet_lrn_dropout.net")
    assert [type(layer).__name__ for layer in net.layers][:4] == ["Conv", "ReLU", "LRN", "MaxPool"]
    with pytest.raises(P.ValidationError):
        P.parse_network("input 3 8 8\nconv 4 3 1 1\nlrn 4 2 0.0001 0.75\nfc 10\nsoftmax 10\n")   # even size
    with pytest.raises(P.ValidationError):
        P.parse_network("input 3 8 8\nconv 4 3 1 1\ndropout 1.0\nfc 10\nsoftmax 10\n")
    with pytest.raises(P.ValidationError):
        P.parse_network("input 3 8 8\nfc 16\nlrn 5 2 0.0001 0.75\nfc 10\nsoftmax 10\n")           # lrn needs CxHxW
    assert P.shape_report(P.load_network(CONFIGS / "alexnet_lrn_dropout.net"), 1).total_flops == \
        P.shape_report(P.load_network(CONFIGS / "alexnet.net"), 1).total_flops


@pytest.mark.parametrize("d,m,cross", [(2, 1, ()), (4, 1, ()), (2, 2, (4,))])
def test_dropout_plans_match_single_worker(d, m, cross):
    """Oracle: every plan with dropout follows the dense single-worker trajectory."""
    import paper_1312_5853_b200 as P
    from oracle.ref_engine import OracleFabric
    net = P.load_network(CONFIGS / "tinynet_lrn_dropout.net")
    dense = P.init_dense_params(net, 0)
    rs = np.random.RandomState(1)
    x, y = rs.randn(8, 3, 16, 16), rs.randint(0, 10, 8)
    if m == 1:
        ref, alt = OracleFabric(net, P.ParallelPlan(1, 1), dense), OracleFabric(net, P.ParallelPlan(d, 1), dense)
        for _ in range(3):
            assert abs(ref.step(x, y) - alt.step(x, y)) < 1e-12
        for i in ref.params[0]:
            assert np.allclose(ref.params[0][i]["w"], alt.params[0][i]["w"], rtol=0, atol=1e-13)
    else:   # grouped columns: compare the hybrid with the single-replica two-column run
        one, hyb = OracleFabric(net, P.ParallelPlan(1, m, cross), dense), \
            OracleFabric(net, P.ParallelPlan(d, m, cross), dense)
        for _ in range(3):
            assert abs(one.step(x, y) - hyb.step(x, y)) < 1e-12
