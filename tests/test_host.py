"""Host logic of the drop-in (rng, data, netdef, plans) against reference KATs.
CPU only."""

import numpy as np
import pytest

from conftest import CONFIGS, GOLDEN
from paper_1312_5853_b200 import rng
from paper_1312_5853_b200.data import gen_synthetic
from paper_1312_5853_b200.errors import PartitionError, ValidationError
from paper_1312_5853_b200.netdef import (
    columnize, load_network, parse_network, shape_report, worker_footprint_bytes)
from paper_1312_5853_b200.plan import (
    ParallelPlan, comm_volume, init_dense_params, merge_params, pack_tree, parse_plan,
    plan_columnized, split_params, unpack_tree)

HOST = np.load(GOLDEN / "host.npz")


def test_splitmix_vigna_kat():
    # Vigna's reference C implementation, seed 1234567 (pkg/tests/test_rng.py:9-37)
    g = rng.SplitMix64(1234567)
    assert [g.next_u64() for _ in range(3)] == [6457827717110365317, 3203168211198807973,
                                                9817491932198370423]


@pytest.mark.parametrize("key", [k for k in HOST.files if k.startswith("derive_")])
def test_derive_streams_match_reference(key):
    _, seed, dom, idx = key.split("_")
    s = rng.derive(int(seed), int(dom), int(idx))
    assert [s.next_u64() for _ in range(4)] == [int(v) for v in HOST[key]]


def test_gauss_uniform_permutation_match_reference():
    assert np.array_equal(rng.derive(9, 1).gauss_array((3, 5), std=0.7), HOST["gauss"])
    assert np.array_equal(rng.derive(9, 3, 2).uniform_array(11, -1.0, 1.0), HOST["uniform"])
    assert np.array_equal(rng.permutation(0, 0, 1000), HOST["perm"])
    assert np.array_equal(rng.permutation(5, 3, 37), HOST["perm_e3"])
    n = rng.SplitMix64(5)
    arr = rng.SplitMix64(5).next_u64_array(10)
    assert [int(v) for v in arr] == [n.next_u64() for _ in range(10)]


def test_synthetic_matches_reference():
    tr, te = gen_synthetic(3, 2, (2, 4, 4), seed=11)
    assert np.array_equal(tr.images, HOST["syn_train_x"])
    assert np.array_equal(tr.labels, HOST["syn_train_y"])
    assert np.array_equal(te.images, HOST["syn_test_x"])


def test_plan_rows_match_reference():
    nets = {n: load_network(CONFIGS / f"{n}.net") for n in ("alexnet", "tinynet", "alexnet_small64")}
    plans = [("alexnet", (1, 1, ())), ("alexnet", (2, 1, ())), ("alexnet", (8, 1, ())),
             ("alexnet", (1, 2, (6,))), ("alexnet", (4, 2, (6,))), ("alexnet", (2, 2, (3, 6, 8, 10))),
             ("tinynet", (2, 2, (3,))), ("tinynet", (1, 4, (3,))), ("alexnet_small64", (1, 2, (6,)))]
    for row, (nname, (d, m, cross)) in zip(HOST["plan_rows"], plans):
        plan = ParallelPlan(d, m, cross)
        cv = comm_volume(plan, nets[nname], 256 * d if nname == "alexnet" else 8 * d)
        cs = plan_columnized(nets[nname], plan)
        got = [cv.bytes, cv.messages, cs.column_param_count, shape_report(cs, 256).total_flops,
               worker_footprint_bytes(cs, 32), len(cs.cross_layers)]
        assert got == [int(v) for v in row]


def test_alexnet_geometry_and_flops():
    net = load_network(CONFIGS / "alexnet.net")
    assert net.output_shapes()[-1] == (1000,)
    assert shape_report(net, 256).total_flops == 1_743_753_363_456
    cs = columnize(net, 2, (6,))
    assert cs.cross_layers == frozenset({6, 13, 15, 17})
    assert cs.column_param_count == 32_531_112


def test_parse_errors():
    with pytest.raises(ValidationError):
        parse_network("input 3 224 224\nconv 96 11 4 0\nsoftmax 10\n")
    with pytest.raises(ValidationError, match="unknown layer keyword"):
        parse_network("input 1 4 4\nbatchnorm 5\nsoftmax 16\n")   # lrn / dropout are extensions now
    with pytest.raises(ValidationError):
        parse_plan("gpus 4\n")
    assert parse_plan("data_shards 2\nmodel_columns 2\ncross_layers 3\n") == ParallelPlan(2, 2, (3,))
    with pytest.raises(PartitionError):
        columnize(load_network(CONFIGS / "tinynet.net"), 3)


def test_split_merge_pack_roundtrip():
    net = load_network(CONFIGS / "tinynet.net")
    dense = init_dense_params(net, 11)
    cs = columnize(net, 2, (3,))
    back = merge_params([split_params(dense, cs, j) for j in range(2)], cs)
    for i in dense:
        for k in ("w", "b"):
            assert np.array_equal(back[i][k], dense[i][k])
    with pytest.raises(ValidationError, match="grouped"):
        cs2 = columnize(net, 2, ())
        merge_params([split_params(dense, cs2, j) for j in range(2)], cs2)
    cs1 = columnize(net, 1)
    flat = pack_tree(dense, cs1)
    assert flat.size == cs1.column_param_count
    un = unpack_tree(flat, cs1)
    assert all(np.array_equal(un[i]["w"], dense[i]["w"]) for i in dense)
