"""Host-side logic of the drop-in API that needs no GPU (reference test_count.py:191-222,
test_graph.py, test_preprocess.py unzip cases)."""
from __future__ import annotations

import numpy as np
import pytest

import paper_1503_00576_b200 as tcb
from paper_1503_00576_b200.count import _resolve_workers
from paper_1503_00576_b200.graph import EdgeArray, OrientedGraph, validate_oriented_graph


def test_even_plan_bounds():
    plan = tcb.PartitionPlan.even(4, 10)
    assert plan.bounds[0] == 0 and plan.bounds[-1] == 10
    assert plan.pool_range(0)[0] == 0
    plan.check_covers(10)
    with pytest.raises(ValueError):
        tcb.PartitionPlan.even(0, 10)
    with pytest.raises(ValueError):
        tcb.PartitionPlan(2, (0, 4, 9)).check_covers(10)
    with pytest.raises(ValueError):
        tcb.PartitionPlan(2, (0, 6, 4)).check_covers(4)


def test_worker_validation():
    assert _resolve_workers(None) >= 1
    assert _resolve_workers(3) == 3
    with pytest.raises(ValueError):
        _resolve_workers(0)


def test_edge_array_contract():
    g = EdgeArray([(1, 0), (0, 1)])
    assert g.num_vertices == 2 and g.edges.dtype == np.uint32 and not g.edges.flags.writeable
    assert EdgeArray([]).num_vertices == 0
    with pytest.raises(ValueError):
        EdgeArray([(0, -1)])
    with pytest.raises(ValueError):
        EdgeArray([(0, 2**32)])
    with pytest.raises(ValueError):
        EdgeArray(np.zeros((3, 3), dtype=np.int64))
    with pytest.raises(ValueError):
        EdgeArray(np.zeros((2, 2), dtype=np.float64))
    assert g == EdgeArray(np.array([(1, 0), (0, 1)], dtype=np.int64))


def test_unzip():
    src, dst = tcb.unzip(np.array([(0, 1), (0, 2), (1, 2)], dtype=np.uint32))
    assert src.tolist() == [0, 0, 1] and dst.tolist() == [1, 2, 2]
    src, dst = tcb.unzip(np.zeros((0, 2), dtype=np.uint32))
    assert src.tolist() == [] and dst.tolist() == []
    src, dst = tcb.unzip(np.array([(5, 7)], dtype=np.uint32))
    assert (src.tolist(), dst.tolist()) == ([5], [7])
    assert src.flags.c_contiguous and dst.flags.c_contiguous


def test_validate_oriented_graph_on_golden(golden):
    for case in golden["small"]:
        og = OrientedGraph(case["edge_src"], case["edge_dst"], case["node_offsets"])
        validate_oriented_graph(og)
        assert og.m_dir == case["m"]
    bad = OrientedGraph([0, 0], [2, 1], [0, 2, 2, 2])
    with pytest.raises(ValueError):
        validate_oriented_graph(bad)


def test_max_out_degree_bound():
    assert tcb.max_out_degree_bound(0) == 0
    assert tcb.max_out_degree_bound(8) == 4
    assert tcb.max_out_degree_bound(9) == 5
