"""Concurrent solves on one GPU (eik_plan_run_batch / eik_solve_batch).

Sharing the device changes only which SMs a solve's persistent kernel holds,
never its results: every solve of a batch must be bit-for-bit (values and
counters) the solve run alone, and the full C2 method matrix run as one batch
must reproduce the reference's golden fields.
"""
import hashlib
import json
import os

import numpy as np
import pytest

import paper_1110_6220_b200 as E
from paper_1110_6220_b200 import configs

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden")


def sha(u):
    return hashlib.sha256(np.ascontiguousarray(u, dtype=np.float64).tobytes()).hexdigest()


def bitwise(a, b):
    return np.array_equal(np.asarray(a).view(np.int64), np.asarray(b).view(np.int64))


def counters(o):
    return (o.sweeps, o.node_updates, o.heap_removals, o.hybrid.mon_checks, o.hybrid.mon_single)


def matrix(p, sizes):
    g = p.grid
    # the exact HCM replay: batch results are compared bit for bit with goldens
    rows = [("fmm", 0), ("fsm", 0)] + [(m, cs) for cs in sizes
                                       for m in ("fmsm", "hcm_exact", "fhcm")]
    return [(m, cs, E.build_cells(g, max(2, g.m // cs), max(2, g.m // cs)) if cs else None)
            for m, cs in rows]


def test_batch_equals_solo_c1_matrix():
    p = configs.config1().problem
    rows = matrix(p, (8, 16, 32))
    plans = [E.Plan(p, m, cells) for m, _, cells in rows]
    try:
        solo = []
        for pl in plans:
            u = np.empty(p.grid.size())
            solo.append((pl.run(u), u))
        for _ in range(2):  # repeated batches reuse the plans
            us = [np.empty(p.grid.size()) for _ in plans]
            outs, ms = E.run_batch(plans, us)
            assert ms > 0.0
            for (m, cs, _), (so, su), bo, bu in zip(rows, solo, outs, us):
                assert bitwise(bu, su), (m, cs)
                assert counters(bo) == counters(so), (m, cs)
                assert bo.ctas >= 1
    finally:
        for pl in plans:
            pl.close()


def test_batch_c2_matrix_golden():
    with open(os.path.join(GOLD, "big.json")) as f:
        big = json.load(f)
    p = configs.config2().problem
    rows = matrix(p, (8, 16, 32, 64))
    plans = [E.Plan(p, m, cells) for m, _, cells in rows]
    try:
        us = [np.empty(p.grid.size()) for _ in plans]
        outs, ms = E.run_batch(plans, us)
        fsm_u = us[1]
        for (m, cs, _), o, u in zip(rows, outs, us):
            key = f"c2/{m.replace('_exact', '')}" + (f"/{cs}" if cs else "")
            if m == "fmm":  # the FMM row is the exact fixed point: FSM's field
                assert bitwise(u, fsm_u)
                assert o.heap_removals == big[key]["heap_removals"]
                continue
            assert sha(u) == big[key]["sha256"], key
            assert (o.sweeps, o.node_updates, o.heap_removals) == \
                (big[key]["sweeps"], big[key]["node_updates"], big[key]["heap_removals"]), key
            if m in ("hcm_exact", "fhcm"):
                assert (o.hybrid.mon_checks, o.hybrid.mon_single) == \
                    (big[key]["mon_checks"], big[key]["mon_single"]), key
        # the step is concurrent: shorter than the solves' device times summed
        assert ms < sum(o.device_ms for o in outs)
    finally:
        for pl in plans:
            pl.close()


def test_solve_batch_equals_solve():
    p = configs.config1().problem
    rows = matrix(p, (16,))
    jobs = [(p, m, cells, None) for m, _, cells in rows]
    outs, ms = E.solve_batch(jobs)
    for (m, cs, cells), bo in zip(rows, outs):
        so = E.solve(p, m, cells)
        assert bitwise(bo.values, so.values), m
        assert counters(bo) == counters(so), m


def test_ctas_cap_and_capacity():
    p = configs.config1().problem
    cells = E.build_cells(p.grid, 16, 16)
    hc = E.Plan(p, "fhcm", cells)
    fs = E.Plan(p, "fsm")
    try:
        dev, fixed = hc.capacity()
        assert dev >= 1 and fixed == 0
        dev_f, fixed_f = fs.capacity()
        nstrips = -(-p.grid.n // 32)  # one warp per 32-row strip, 4 warps per CTA
        assert fixed_f == -(-nstrips // 4) and dev_f >= fixed_f
        full = hc.run(np.empty(p.grid.size()))
        hc.set_ctas(1)  # the committer alone: the serial exact replay
        u1 = np.empty(p.grid.size())
        alone = hc.run(u1)
        assert alone.ctas == 1 and alone.spec[0] == 0
        assert counters(alone) == counters(full)
        assert bitwise(u1, full.values)
        hc.set_ctas(0)
        assert hc.run().ctas == full.ctas
        with pytest.raises(E.ConfigError):
            hc.set_ctas(-1)
    finally:
        hc.close()
        fs.close()


def test_batch_rejects_duplicates_and_empty():
    p = configs.config1().problem
    pl = E.Plan(p, "fsm")
    try:
        with pytest.raises(ValueError):
            E.run_batch([pl, pl])
        outs, ms = E.run_batch([])
        assert outs == [] and ms == 0.0
    finally:
        pl.close()


def test_solve_batch_device_speed_equals_solve():
    """eik_solve_batch with the speed field already on the device
    (speed_on_device = 1): each plan's run copies it device to device before
    its solve (the deferred upload), results bit-identical to solve()."""
    import ctypes as C

    import torch

    from paper_1110_6220_b200 import _native as N
    from paper_1110_6220_b200 import solvers as S

    p = configs.config1().problem
    rows = matrix(p, (16,))
    Fd = torch.from_numpy(np.ascontiguousarray(p.sampled_speed())).cuda()
    torch.cuda.synchronize()
    n = len(rows)
    keep, pp, cc = [], (C.POINTER(N.eik_problem) * n)(), (C.POINTER(N.eik_cells) * n)()
    meth = (C.c_int32 * n)()
    res = (N.eik_output * n)()
    us = []
    for k, (m, _, cells) in enumerate(rows):
        cp, kp = S._c_problem(p, p.sampled_speed())
        cp.speed = C.cast(C.c_void_p(Fd.data_ptr()), C.POINTER(C.c_double))
        cp.speed_on_device = 1
        tables = S.cell_tables(p, cells) if cells is not None else None
        c, kc = S._c_cells(cells, tables)
        keep += [cp, kp, c, kc]
        pp[k] = C.pointer(cp)
        cc[k] = C.pointer(c) if c is not None else C.POINTER(N.eik_cells)()
        meth[k] = N.METHOD_NAMES[m]
        u = np.empty(p.grid.size())
        us.append(u)
        res[k].u = N.dptr(u)
        res[k].u_on_device = 0
    ms = C.c_double()
    N.raise_for(N.lib.eik_solve_batch(pp, cc, meth, n, res, C.byref(ms)))
    for k, (m, cs, cells) in enumerate(rows):
        so = E.solve(p, m, cells)
        assert bitwise(us[k], so.values), m
        assert res[k].sweeps == so.sweeps and res[k].heap_removals == so.heap_removals, m
