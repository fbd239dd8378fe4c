"""Field dumps and CSV rows in the reference's formats
(paper_1110_6220_b200/experiment_io.py; field_io.cpp, experiment.cpp:314-329)
-- SURVEY.md section 8(f) row 3.  CPU tests compare bytes with the reference's
own writers (oracle/_ref); the GPU test builds a row through the device
solvers and metrics."""
import json
import os

import numpy as np
import pytest

import paper_1110_6220_b200 as E
from paper_1110_6220_b200 import experiment_io as X
from oracle import oracle as O

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _field():
    rng = np.random.default_rng(7)
    u = rng.uniform(0, 3, size=(5, 7)) * 10.0 ** rng.integers(-20, 20, size=(5, 7))
    u[1, 2] = np.inf
    u[0, 0] = 0.0
    return u.reshape(-1), 7, 5, 0.0123456789012345678


@pytest.mark.parametrize("fmt", ["raw", "ascii"])
def test_dump_round_trip(tmp_path, fmt):
    u, m, n, h = _field()
    path = str(tmp_path / f"f.{fmt}")
    X.dump_field(u, m, n, h, path, fmt)
    v, m2, n2, h2 = X.load_field(path, fmt)
    assert (m2, n2) == (m, n) and np.array_equal(v, u)
    assert h2 == (h if fmt == "ascii" else 0.0)


@pytest.mark.skipif(not O.have_ref(), reason="oracle/_ref not built")
@pytest.mark.parametrize("fmt", ["raw", "ascii"])
def test_dump_bytes_equal_reference(tmp_path, fmt):
    u, m, n, h = _field()
    ours, ref = str(tmp_path / "ours"), str(tmp_path / "ref")
    X.dump_field(u, m, n, h, ours, fmt)
    O.ref_dump_field(u, m, n, h, ref, fmt == "ascii")
    assert open(ours, "rb").read() == open(ref, "rb").read()


@pytest.mark.skipif(not O.have_ref(), reason="oracle/_ref not built")
def test_csv_header_and_lines_equal_reference():
    assert X.csv_header() == O.ref_csv_header()
    rng = np.random.default_rng(3)
    for k in range(200):
        meth = X.METHODS[k % 6]
        d9 = [rng.uniform(0, 1e4), 10.0 ** rng.uniform(-12, 1), 10.0 ** rng.uniform(-12, 1),
              rng.uniform(0, 50), rng.uniform(0, 50), rng.uniform(0, 50), rng.uniform(0, 10),
              rng.uniform(0, 100), rng.uniform(0, 100)]
        if k % 17 == 0:
            d9[1] = np.inf
        c3 = [int(rng.integers(0, 1 << 40)) for _ in range(3)]
        row = X.ExperimentRow(f"p{k}", meth, int(rng.integers(2, 40000)), int(rng.integers(0, 512)),
                              *d9, *c3)
        assert X.csv_line(row) == O.ref_csv_line(row.problem, meth, row.grid_m, row.cells_x,
                                                 d9, c3)


@pytest.mark.gpu
def test_run_row_matches_reference_row(tmp_path):
    """A row through the device path: the reference's counters and metrics
    (small.json, metrics.json) in the reference's CSV schema."""
    from tests.golden.make_golden import SMALL_CASES
    with open(os.path.join(GOLD, "small.json")) as f:
        counters = json.load(f)
    with open(os.path.join(GOLD, "metrics.json")) as f:
        mets = json.load(f)
    cid, make, cells = SMALL_CASES[0]
    p = make()
    exact = E.fmm_solve(p).values
    truth = E.ground_truth(p, 4)
    E.set_hcm_mode("exact")  # the reference's counters need its exact heap order
    try:
        rows = [(meth, X.run_row(cid, p, meth, cells[0], exact, truth, dump_dir=str(tmp_path)))
                for meth in ("fhcm", "hcm", "fmsm")]
    finally:
        E.set_hcm_mode("band")
    for meth, r in rows:
        key = f"{cid}/{meth}/{cells[0]}"
        assert (r.sweeps, r.node_updates, r.heap_removals) == (
            counters[key]["sweeps"], counters[key]["node_updates"], counters[key]["heap_removals"])
        assert r.l_inf == pytest.approx(mets[key]["l_inf"], rel=1e-9)
        line = X.csv_line(r)
        assert line.split(",")[:4] == [cid, meth, str(p.grid.m), str(cells[0])]
        v, m, n, h = X.load_field(str(tmp_path / f"{cid}_{meth}_m{p.grid.m}_c{cells[0]}.txt"),
                                  "ascii")
        assert (m, n) == (p.grid.m, p.grid.n) and np.isfinite(v).all()
