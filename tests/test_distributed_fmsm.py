"""FMSM sharded by row strips of cells, run by levels of the cell DAG
(paper_1110_6220_b200/distributed.py fmsm_solve_strips).

CPU: the schedule's levels are a valid layering of the reference's rank-order
pass; one strip and gloo worlds of 2 and 3 ranks -- with the strip's cells
processed by a pure-Python restatement of fmsm.cpp:176-222 (test
infrastructure, small grids only) -- equal the oracle's fmsm_solve bit for
bit, counters included.  GPU: the same through the device strip plan
(eik_plan_create_fmsm_strip / eik_plan_fmsm_level_async), one strip, two
ranks on one device over gloo (levels are host-synchronised: no kernel waits
on another rank), and the NCCL stream-ordered path with one rank.
"""
import math
import os
import socket
import tempfile

import numpy as np
import pytest

import paper_1110_6220_b200 as E
from paper_1110_6220_b200.distributed import fmsm_schedule, fmsm_solve_strips
from oracle import oracle as O

SW, NW, NE, SE = 0, 1, 2, 3  # SweepDir (local_update.hpp:23)


def _quad(ua, ub, f, h):  # local_update.hpp:30-43
    c = h / f
    if math.isfinite(ua) and math.isfinite(ub):
        diff = ua - ub
        if abs(diff) <= c:
            return 0.5 * (ua + ub) + 0.5 * math.sqrt(2.0 * c * c - diff * diff)
    return c + (ub if ub < ua else ua)


class CpuFmsmStrip:
    """A strip of a sharded FMSM on the CPU, the reference's cell pass
    (fmsm.cpp:176-222) restated in Python: the checker for the sharding
    logic.  Mirrors DeviceFmsmStrip's interface."""

    def __init__(self, local, cells_x, cells_y, base_y, row0, row_end):
        g = local.grid
        self.m, self.n, self.h = g.m, g.n, g.h
        self.F = local.sampled_speed().reshape(self.n, self.m)
        self.exit = np.zeros((self.n, self.m), dtype=bool)
        self.exit.reshape(-1)[np.asarray(local.exit_nodes)] = True
        self.u0 = np.full((self.n, self.m), np.inf)
        self.u0.reshape(-1)[np.asarray(local.exit_nodes)] = local.exit_cost
        self.cx, self.cy, self.base_y, self.row0, self.row_end = cells_x, cells_y, base_y, row0, \
            row_end
        self.base_x = g.m // cells_x
        self.sweeps = self.updates = 0

    def _rect(self, cell):
        x, y = cell % self.cx, cell // self.cx
        ib = x * self.base_x
        ie = self.m if x == self.cx - 1 else ib + self.base_x
        jb = self.row0 + y * self.base_y
        je = self.row_end if y == self.cy - 1 else jb + self.base_y
        return ib, ie, jb, je

    def levels(self, cells_by_level, level_off, flags):
        self.cells, self.off, self.flags = list(cells_by_level), list(level_off), list(flags)
        self.u = self.u0.copy()
        self.sweeps = self.updates = 0

    def _sweep(self, r, d, directional):
        ib, ie, jb, je = r
        iasc, jasc = d in (SW, NW), d in (SW, SE)
        u, F, h = self.u, self.F, self.h
        changed = False
        for i in (range(ib, ie) if iasc else range(ie - 1, ib - 1, -1)):
            for j in (range(jb, je) if jasc else range(je - 1, jb - 1, -1)):
                if self.exit[j, i]:
                    continue
                self.updates += 1
                e = u[j, i + 1] if i + 1 < self.m else math.inf
                w = u[j, i - 1] if i > 0 else math.inf
                nn = u[j + 1, i] if j + 1 < self.n else math.inf
                s = u[j - 1, i] if j > 0 else math.inf
                if directional:
                    a, b = {NE: (e, nn), NW: (w, nn), SE: (e, s), SW: (w, s)}[d]
                else:
                    a, b = (w if w < e else e), (s if s < nn else nn)
                cand = _quad(a, b, float(F[j, i]), h)
                if cand < u[j, i]:
                    u[j, i] = cand
                    changed = True
        return changed

    def run_level(self, L, stream=0):
        for cell in self.cells[self.off[L]:self.off[L + 1]]:
            r = self._rect(cell)
            fl = self.flags[cell]
            if fl & 16:  # Q-cell: FSM to convergence, halo frozen (fmsm.cpp:200-210)
                k = 0
                while True:
                    ch = self._sweep(r, k % 4, False)
                    k += 1
                    if not ch:
                        break
                self.sweeps += k
            else:  # one directional sweep per chosen direction, NE NW SE SW
                for d in (NE, NW, SE, SW):
                    if fl & (1 << d):
                        self._sweep(r, d, True)
                        self.sweeps += 1

    def get_rows(self, row0, nrows, out):
        out[:] = self.u[row0:row0 + nrows].reshape(-1)

    def set_rows(self, row0, nrows, src):
        self.u[row0:row0 + nrows] = np.asarray(src).reshape(nrows, self.m)

    def counters(self):
        return self.sweeps, self.updates


def _case(kind="sin"):
    if kind == "sin":
        g = E.Grid(41, 37, 1.0 / 40, 0.0, 0.0)
        p = E.build_problem(g, E.speed_sinusoid(0.5, 3), E.ExitSpec.point_source((0.31, 0.52)))
        return p, E.build_cells(g, 8, 7)
    g = E.Grid(45, 43, 1.0 / 44, -0.5, -0.5)
    p = E.build_problem(g, E.speed_checkerboard(5),
                        E.ExitSpec.node_set([(3, 5), (40, 38), (20, 21)], [0.0, 0.03, 0.01]))
    return p, E.build_cells(g, 6, 9)


def test_schedule_levels_layer_the_rank_order():
    for kind in ("sin", "chk"):
        p, cells = _case(kind)
        s = fmsm_schedule(p, cells)
        cx, cy = cells.cells_x, cells.cells_y
        assert np.array_equal(s.order[s.rank], np.arange(cx * cy))
        for c in range(cx * cy):
            x, y = c % cx, c // cx
            nbs = [c - 1 if x > 0 else -1, c + 1 if x + 1 < cx else -1,
                   c - cx if y > 0 else -1, c + cx if y + 1 < cy else -1]
            early = [s.level[b] for b in nbs if b >= 0 and s.rank[b] < s.rank[c]]
            assert s.level[c] == (max(early) + 1 if early else 0)
            for b in nbs:  # adjacent cells never share a level
                assert b < 0 or s.level[b] != s.level[c]
        ref = O.oracle_solve(p, "fmsm", cells)
        assert s.coarse_pops == ref.heap_removals


@pytest.mark.parametrize("kind", ["sin", "chk"])
def test_single_strip_cpu_is_fmsm_bitwise(kind):
    p, cells = _case(kind)
    r = fmsm_solve_strips(p, cells, strip_factory=CpuFmsmStrip)
    ref = O.oracle_solve(p, "fmsm", cells)
    assert np.array_equal(r.values, ref.u)
    assert (r.sweeps, r.node_updates, r.heap_removals) == (ref.sweeps, ref.node_updates,
                                                           ref.heap_removals)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, outdir, use_device, kind):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        p, cells = _case(kind)
        r = fmsm_solve_strips(p, cells, strip_factory=None if use_device else CpuFmsmStrip)
        np.save(os.path.join(outdir, f"u{rank}.npy"), r.values)
        np.save(os.path.join(outdir, f"k{rank}.npy"),
                np.array([r.sweeps, r.node_updates, r.heap_removals, r.exchanges]))
    finally:
        dist.destroy_process_group()


def _run_world(world, use_device, kind):
    import torch.multiprocessing as mp
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_worker, args=(world, _free_port(), d, use_device, kind), nprocs=world, join=True)
        us = [np.load(os.path.join(d, f"u{r}.npy")) for r in range(world)]
        ks = [np.load(os.path.join(d, f"k{r}.npy")) for r in range(world)]
    return us, ks


@pytest.mark.parametrize("world,kind", [(2, "sin"), (3, "chk")])
def test_gloo_strips_cpu_are_fmsm_bitwise(world, kind):
    p, cells = _case(kind)
    us, ks = _run_world(world, False, kind)
    ref = O.oracle_solve(p, "fmsm", cells)
    for r in range(world):
        assert np.array_equal(us[r], ref.u)
        assert tuple(ks[r][:3]) == (ref.sweeps, ref.node_updates, ref.heap_removals)
        assert ks[r][3] > 0  # edge rows were exchanged


@pytest.mark.gpu
@pytest.mark.parametrize("kind", ["sin", "chk"])
def test_device_single_strip_is_fmsm_bitwise(kind):
    p, cells = _case(kind)
    r = fmsm_solve_strips(p, cells)
    ref = O.oracle_solve(p, "fmsm", cells)
    assert np.array_equal(r.values, ref.u)
    assert (r.sweeps, r.node_updates, r.heap_removals) == (ref.sweeps, ref.node_updates,
                                                           ref.heap_removals)


@pytest.mark.gpu
def test_device_strip_larger_grid_bitwise():
    g = E.Grid.centered(257)
    p = E.build_problem(g, E.speed_sinusoid(0.5, 20), E.ExitSpec.point_source((0.1, -0.2)))
    cells = E.build_cells(g, 16, 16)
    r = fmsm_solve_strips(p, cells)
    ref = O.oracle_solve(p, "fmsm", cells)
    assert np.array_equal(r.values, ref.u) and r.sweeps == ref.sweeps
    assert r.levels > 1


@pytest.mark.gpu
@pytest.mark.parametrize("world,kind", [(2, "sin"), (2, "chk"), (3, "chk")])
def test_device_strips_ranks_bitwise(world, kind):
    """Two / three ranks on one GPU over gloo (the levels are host-synchronised:
    no kernel waits on another rank's)."""
    p, cells = _case(kind)
    us, ks = _run_world(world, True, kind)
    ref = O.oracle_solve(p, "fmsm", cells)
    for r in range(world):
        assert np.array_equal(us[r], ref.u)
        assert tuple(ks[r][:3]) == (ref.sweeps, ref.node_updates, ref.heap_removals)


def _nccl_single(_index, outdir, port):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1)
    try:
        p, cells = _case("chk")
        r = fmsm_solve_strips(p, cells, gather="rank0")
        np.save(os.path.join(outdir, "u.npy"), r.values)
        np.save(os.path.join(outdir, "k.npy"), np.array([r.sweeps, r.node_updates]))
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
def test_device_stream_ordered_levels_single_rank():
    import torch.multiprocessing as mp
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_nccl_single, args=(d, _free_port()), nprocs=1, join=True)
        u = np.load(os.path.join(d, "u.npy"))
        k = np.load(os.path.join(d, "k.npy"))
    p, cells = _case("chk")
    ref = O.oracle_solve(p, "fmsm", cells)
    assert np.array_equal(u, ref.u) and k[0] == ref.sweeps and k[1] == ref.node_updates


def _random_problem(rng, k):
    m = int(rng.integers(9, 70))
    n = int(rng.integers(9, 70))
    g = E.Grid(m, n, 1.0 / (m - 1), -0.3, 0.2)
    kind = k % 5
    if kind == 4:  # speed ratio 1e6: past the bucket ring, the heap path
        sp = E.speed_checkerboard(3, 1e-6, 1.0)
    elif kind == 0:
        sp = E.speed_sinusoid(0.5, int(rng.integers(1, 6)))
    elif kind == 1:
        sp = E.speed_checkerboard(int(rng.integers(0, 4)) * 2 + 1, 1.0, float(rng.uniform(1.5, 80)))
    elif kind == 2:
        sp = E.speed_constant()
    else:
        sp = E.speed_checkerboard(3, 0.01, 1.0)
    if k % 3 == 0:
        ex = E.ExitSpec.point_source((g.x0 + float(rng.uniform(0, m - 1)) * g.h,
                                      g.y0 + float(rng.uniform(0, n - 1)) * g.h))
    else:
        cnt = int(rng.integers(1, 6))
        nodes = sorted({(int(rng.integers(0, m)), int(rng.integers(0, n))) for _ in range(cnt)})
        costs = [float(rng.uniform(0, 50.0 if k % 5 == 0 else 0.05)) for _ in nodes]
        ex = E.ExitSpec.node_set(nodes, costs)
    p = E.build_problem(g, sp, ex)
    cx = int(rng.integers(2, max(3, m // 2)))
    cy = int(rng.integers(2, max(3, n // 2)))
    return p, E.build_cells(g, cx, cy)


def test_schedule_order_equals_the_oracle_on_random_problems():
    """eik_fmsm_schedule (the product's Part I: bucketed exact queue, heap
    fallback for extreme speed ratios / cost spreads, insertion-sorted
    quantised order) equals the oracle's Part I -- order, coarse removals and
    coarse updates -- on random problems (CPU, no device)."""
    rng = np.random.default_rng(11)
    for k in range(120):
        p, cells = _random_problem(rng, k)
        s = fmsm_schedule(p, cells)
        order, pops, upd = O.oracle_fmsm_order(p, cells)
        assert np.array_equal(s.order, order), k
        assert (s.coarse_pops, s.coarse_updates) == (pops, upd), k
