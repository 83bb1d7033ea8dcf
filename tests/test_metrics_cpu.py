"""CPU checks of the metric helpers and host-side ingest logic (reference test_metrics.py,
test_io.py).  No GPU: transitivity and the DegreeOrder wedge sum are host arithmetic."""
from __future__ import annotations

import json
import os

import numpy as np
import pytest

import oracle
from conftest import GOLDEN_DIR, sha

from paper_1503_00576_b200 import cli
from paper_1503_00576_b200 import io as gio
from paper_1503_00576_b200.graph import DegreeOrder, EdgeArray, degrees_of
from paper_1503_00576_b200.metrics import (CountOverflowError, InconsistentCountsError,
                                           transitivity, wedge_count)


def test_transitivity_cases():
    assert transitivity(1, 3) == 1.0
    assert transitivity(0, 3) == 0.0
    assert transitivity(1, 6) == 0.5
    assert transitivity(0, 0) == 0.0
    with pytest.raises(InconsistentCountsError):
        transitivity(2, 5)


def test_wedges_degree_order_golden():
    with open(os.path.join(GOLDEN_DIR, "golden_ingest.json")) as fh:
        gi = json.load(fh)
    rec = gi["wedges"]["rmat_10_8_7"]
    g = EdgeArray(oracle.symmetrize(oracle.rmat_pairs(10, 8, seed=7)))
    assert sha(g.edges) == rec["edges_sha256"]
    assert wedge_count(degrees_of(g)) == rec["wedges"]


def test_wedge_overflow_reported():
    assert wedge_count(DegreeOrder(np.array([2**32, 1]))) == 2**32 * (2**32 - 1) // 2
    with pytest.raises(CountOverflowError):
        wedge_count(DegreeOrder(np.full(3, 2**33)))


def test_line_message_rebuild(tmp_path):
    p = tmp_path / "x.txt"
    p.write_text("0 1\n1 2 3\n4 x\n-1 2\n")
    assert gio._line_message(p, 2) == "expected two fields, got 3"
    assert gio._line_message(p, 3) == "not an integer pair: '4 x'"
    assert gio._line_message(p, 4) == "vertex id out of unsigned 32-bit range: '-1 2'"


def test_cli_usage_errors():
    assert cli.main([]) == 2
    assert cli.main(["count"]) == 2
    assert cli.main(["count", "f", "--mode", "loose"]) == 2
    with pytest.raises(ValueError):
        gio.read_edge_list("whatever", mode="loose")
