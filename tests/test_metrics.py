"""Ground truth and error metrics (paper_1110_6220_b200/metrics.py, the
reference's metrics.cpp) -- SURVEY.md section 8(f) row 2.

Goldens (tests/golden/metrics.*, make_golden.py --metrics) hold the
reference's refine-4 ground truth and its method_metrics reports for the small
cases, computed on the reference's own fields.
"""
import json
import os

import numpy as np
import pytest

import paper_1110_6220_b200 as E
from tests.golden.make_golden import SMALL_CASES

HERE = os.path.join(os.path.dirname(__file__), "golden")


def _gold():
    with open(os.path.join(HERE, "metrics.json")) as f:
        return json.load(f), np.load(os.path.join(HERE, "metrics.npz")), \
            np.load(os.path.join(HERE, "small.npz"))


CASES = {cid: make for cid, make, _ in SMALL_CASES}


def test_refined_problem_maps_exits_like_ground_truth():
    # metrics.cpp:83-91: (i, j) -> (refine*i, refine*j), costs kept, order kept
    p = E.build_problem(E.Grid(7, 5, 0.25, -1.0, 0.5), E.speed_constant(),
                        E.ExitSpec.node_set([(1, 0), (6, 2), (3, 4)], [0.0, 0.5, 0.25]))
    f = E.refined_problem(p, 4)
    assert (f.grid.m, f.grid.n, f.grid.h, f.grid.x0, f.grid.y0) == (25, 17, 0.0625, -1.0, 0.5)
    want = sorted([(4 * j * 25 + 4 * i, c) for (i, j), c in
                   zip([(1, 0), (6, 2), (3, 4)], [0.0, 0.5, 0.25])])
    assert list(f.exit_nodes) == [w[0] for w in want]
    assert list(f.exit_cost) == [w[1] for w in want]
    with pytest.raises(ValueError):
        E.refined_problem(p, 0)


@pytest.mark.gpu
def test_device_metrics_equal_reference_reports():
    """Same fields in (the reference's method, exact and truth fields): maxima,
    counts and the X+ test exactly the reference's; the two sums within 1e-12."""
    gold, truth, fields = _gold()
    for key, want in gold.items():
        cid = key.split("/")[0]
        p = CASES[cid]()
        r = E.method_metrics(fields[key], fields[f"{cid}/fmm"], truth[f"{cid}/truth4"],
                             p.exit_nodes)
        assert (r.l_inf, r.max_error_ratio, r.ratio_of_max, r.m_plus, r.x_plus_empty) == \
            (want["l_inf"], want["max_error_ratio"], want["ratio_of_max"], want["m_plus"],
             want["x_plus_empty"]), key
        assert r.l_1 == pytest.approx(want["l_1"], rel=1e-12, abs=0.0), key
        assert r.avg_error_ratio == pytest.approx(want["avg_error_ratio"], rel=1e-12), key


@pytest.mark.gpu
def test_ground_truth_and_full_pipeline():
    """Our refine-4 ground truth (the device FMM row on the refined grid) is the
    reference's within 1e-10, and the whole pipeline -- our solves, our truth,
    device metrics -- reproduces the reference's reports."""
    gold, truth, _ = _gold()
    for cid, make, cells in SMALL_CASES:
        p = make()
        t = E.ground_truth(p, 4)
        assert float(np.max(np.abs(t - truth[f"{cid}/truth4"]))) <= 1e-10, cid
        exact = E.fmm_solve(p).values
        for key in [f"{cid}/fsm"] + [f"{cid}/{m}/{c}" for c in cells for m in ("hcm", "fhcm")]:
            parts = key.split("/")
            cl = E.build_cells(p.grid, int(parts[2]), int(parts[2])) if len(parts) == 3 else None
            u = E.solve(p, parts[1], cl).values
            r = E.method_metrics(u, exact, t, p.exit_nodes)
            w = gold[key]
            assert r.l_inf == pytest.approx(w["l_inf"], rel=1e-9), key
            assert r.l_1 == pytest.approx(w["l_1"], rel=1e-9), key
            assert abs(r.m_plus - w["m_plus"]) <= max(2, w["m_plus"] // 1000), key
