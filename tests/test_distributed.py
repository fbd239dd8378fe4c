"""Strip-Jacobi FSM across ranks (paper_1110_6220_b200/distributed.py,
SURVEY.md section 8(e) option A).

CPU (gloo, world size 2, the oracle's sweep plugged in as the strip sweeper):
the distributed run must equal a serial emulation of the same rounds bit for
bit, with the same round count, and the reference's fixed point within 1e-10.
GPU: one strip is fsm_solve bit for bit (identical sweeps); two ranks on one
device (gloo exchange, no kernel waits on another rank) equal the emulation.
"""
import os
import socket
import tempfile

import numpy as np
import pytest

import paper_1110_6220_b200 as E
from paper_1110_6220_b200.distributed import strip_bounds, strip_problem
from oracle import oracle as O


def _problem(m=61, n=57, kind="sin"):
    g = E.Grid(m, n, 1.0 / (m - 1), 0.0, 0.0)
    sp = E.speed_sinusoid(0.5, 3) if kind == "sin" else E.speed_checkerboard(5)
    ex = E.ExitSpec.node_set([(5, 7), (m - 9, n - 4), (m // 2, n // 2)], [0.0, 0.02, 0.01])
    return E.build_problem(g, sp, ex)


class OracleStripSweeper:
    """The strip on the CPU through the oracle's sweep (test infrastructure):
    mirrors eik_plan_prepare (u = +inf, exits = cost) and eik_plan_sweep."""

    def __init__(self, local):
        g = local.grid
        self.m, self.nl, self.h = g.m, g.n, g.h
        self.F = np.ascontiguousarray(local.sampled_speed(), dtype=np.float64)
        self.frozen = np.zeros(g.m * g.n, dtype=np.uint8)
        self.frozen[local.exit_nodes] = 1
        self.u = np.full(g.m * g.n, np.inf)
        self.u[local.exit_nodes] = local.exit_cost

    def sweep(self, k):
        return O.oracle_fsm_sweep(self.m, self.nl, self.h, self.F, self.frozen, self.u, k & 3)

    def get_rows(self, r, nrows, out):
        out[:] = self.u[r * self.m:(r + nrows) * self.m]

    def set_rows(self, r, nrows, src):
        self.u[r * self.m:(r + nrows) * self.m] = np.asarray(src)


def emulate(problem, world, factory=OracleStripSweeper, bounds=None):
    """The same rounds in one process: every strip sweeps, then edges swap.
    `bounds` overrides the balanced row split with explicit [r0, r1) strips."""
    m, n = problem.grid.m, problem.grid.n
    strips = bounds or [strip_bounds(n, world, r) for r in range(world)]
    world = len(strips)
    sws = [factory(strip_problem(problem, a, b)) for a, b in strips]
    for s in sws:
        s.set_rows(0, 1, np.full(m, np.inf))
        s.set_rows(s.nl - 1, 1, np.full(m, np.inf))
    k = 0
    while True:
        changed = [s.sweep(k) for s in sws]
        k += 1
        lo = [np.empty(m) for _ in sws]
        hi = [np.empty(m) for _ in sws]
        for r, s in enumerate(sws):
            s.get_rows(1, 1, lo[r])
            s.get_rows(s.nl - 2, 1, hi[r])
        for r, s in enumerate(sws):
            if r > 0:
                s.set_rows(0, 1, hi[r - 1])
            if r < world - 1:
                s.set_rows(s.nl - 1, 1, lo[r + 1])
        if not any(changed):
            break
    u = np.empty(m * n)
    for (a, b), s in zip(strips, sws):
        s.get_rows(1, b - a, u[a * m:b * m])
    return u, k


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
        p = _problem(kind=kind)
        fac = None if use_device else OracleStripSweeper
        r = E.fsm_solve_strips(p, sweeper_factory=fac)
        np.save(os.path.join(outdir, f"u{rank}.npy"), r.values)
        np.save(os.path.join(outdir, f"k{rank}.npy"), np.array([r.sweeps, r.node_updates]))
    finally:
        dist.destroy_process_group()


def _run_world(world, use_device, kind="sin"):
    import torch.multiprocessing as mp
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_worker, args=(world, _free_port(), d, use_device, kind), nprocs=world, join=True)
        us = [np.load(os.path.join(d, f"u{r}.npy")) for r in range(world)]
        ks = [np.load(os.path.join(d, f"k{r}.npy")) for r in range(world)]
    return us, ks


def test_strip_bounds_cover_rows():
    for n, world in [(10, 1), (10, 3), (2049, 8), (57, 2)]:
        b = [strip_bounds(n, world, r) for r in range(world)]
        assert b[0][0] == 0 and b[-1][1] == n
        assert all(b[r][1] == b[r + 1][0] and b[r][1] > b[r][0] for r in range(world - 1))
    with pytest.raises(E.ConfigError):
        strip_bounds(3, 4, 0)


def test_strip_problem_maps_rows_and_exits():
    p = _problem()
    m = p.grid.m
    loc = strip_problem(p, 20, 40)
    assert (loc.grid.m, loc.grid.n) == (m, 22)
    F = p.sampled_speed().reshape(p.grid.n, m)
    assert np.array_equal(loc.sampled_speed().reshape(22, m)[1:-1], F[20:40])
    own = [(e % m, e // m) for e in p.exit_nodes if 20 <= e // m < 40]
    lex = set(int(e) for e in loc.exit_nodes)
    assert all((j - 19) * m + i in lex for i, j in own)
    assert all(i in lex and (21 * m + i) in lex for i in range(m))  # ghost rows frozen
    assert np.all(np.diff(loc.exit_nodes) > 0)


def test_single_strip_is_fsm_bitwise():
    p = _problem()
    u, k = emulate(p, 1)
    ref = O.oracle_solve(p, "fsm")
    assert np.array_equal(u, ref.u) and k == ref.sweeps


@pytest.mark.parametrize("world", [2, 3, 5])
def test_emulated_strips_reach_the_fixed_point(world):
    p = _problem(kind="chk")
    u, k = emulate(p, world)
    ref = O.oracle_solve(p, "fsm")
    assert float(np.max(np.abs(u - ref.u))) <= 1e-10
    assert k >= ref.sweeps


def test_gloo_world2_equals_emulation():
    p = _problem()
    us, ks = _run_world(2, use_device=False)
    u, k = emulate(p, 2)
    for r in range(2):
        assert np.array_equal(us[r], u)
        assert ks[r][0] == k
        assert ks[r][1] == k * (p.grid.size() - len(p.exit_nodes))
    assert float(np.max(np.abs(u - O.oracle_solve(p, "fsm").u))) <= 1e-10


@pytest.mark.gpu
def test_device_single_strip_is_fsm_bitwise():
    p = _problem()
    r = E.fsm_solve_strips(p)
    ref = O.oracle_solve(p, "fsm")
    assert np.array_equal(r.values, ref.u)
    assert r.sweeps == ref.sweeps and r.node_updates == ref.node_updates


@pytest.mark.gpu
def test_device_strips_two_ranks_equal_emulation():
    p = _problem(kind="chk")
    us, ks = _run_world(2, use_device=True, kind="chk")
    u, k = emulate(p, 2)
    for r in range(2):
        assert np.array_equal(us[r], u) and ks[r][0] == k


@pytest.mark.gpu
@pytest.mark.parametrize("part_rows,kind", [(32, "chk"), (64, "sin"), (96, "chk")])
def test_device_partitions_equal_emulation(part_rows, kind):
    """eik_plan_set_partitions: the strip-Jacobi rounds inside one launch
    (parts of part_rows rows, edge rows read from the previous sweep) equal
    the serial emulation of the same rounds bit for bit, sweep count included."""
    p = _problem(m=61, n=203, kind=kind)
    n = p.grid.n
    bounds = [(a, min(a + part_rows, n)) for a in range(0, n, part_rows)]
    u, k = emulate(p, len(bounds), bounds=bounds)
    plan = E.Plan(p, "fsm")
    plan.set_partitions(part_rows)
    got = np.empty(p.grid.size())
    o = plan.run(u_host=got)
    assert np.array_equal(got, u)
    assert o.sweeps == k
    plan.set_partitions(0)  # back to the exact wavefront: fsm_solve bit for bit
    o = plan.run(u_host=got)
    ref = O.oracle_solve(p, "fsm")
    assert np.array_equal(got, ref.u) and o.sweeps == ref.sweeps
    plan.close()
    with pytest.raises(E.ConfigError):
        E.Plan(p, "fsm").set_partitions(48)


def test_strip_speed_is_the_whole_grid_sampling():
    """A rank samples only its rows, with the GLOBAL coordinates: bit for bit
    the rows of the whole grid's sampling (SpeedField and plain callables)."""
    from paper_1110_6220_b200.configs import config5
    from paper_1110_6220_b200.distributed import strip_speed
    p = config5(257).problem  # the 16-sinusoid field (tabulated sampling)
    q = _problem()
    for prob in (p, q):
        F = prob.sampled_speed().reshape(prob.grid.n, prob.grid.m)
        fresh = E.Problem(prob.grid, prob.speed, prob.exit_nodes, prob.exit_cost)
        for a, b in [(0, 17), (40, 41), (prob.grid.n - 9, prob.grid.n)]:
            assert np.array_equal(strip_speed(fresh, a, b), F[a:b])
    g = q.grid
    call = E.Problem(g, lambda x, y: 1.0 + 0.25 * np.sin(3 * x) * np.cos(2 * y), q.exit_nodes,
                     q.exit_cost)
    F = call.sampled_speed().reshape(g.n, g.m)
    fresh = E.Problem(g, call.speed, q.exit_nodes, q.exit_cost)
    assert np.array_equal(strip_speed(fresh, 5, 30), F[5:30])


def _nccl_single(_index, outdir, port):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1)
    try:
        p = _problem(kind="chk")
        r = E.fsm_solve_strips(p, gather="rank0")
        np.save(os.path.join(outdir, "u.npy"), r.values)
        np.save(os.path.join(outdir, "k.npy"), np.array([r.sweeps, r.node_updates]))
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
def test_device_stream_ordered_rounds_single_rank():
    """The NCCL path (rounds enqueued on the stream, the change flag read two
    rounds behind) with one rank is fsm_solve: same bits, same sweep count."""
    import torch.multiprocessing as mp
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_nccl_single, args=(d, _free_port()), nprocs=1, join=True)
        u = np.load(os.path.join(d, "u.npy"))
        k = np.load(os.path.join(d, "k.npy"))
    ref = O.oracle_solve(_problem(kind="chk"), "fsm")
    assert np.array_equal(u, ref.u) and k[0] == ref.sweeps and k[1] == ref.node_updates


@pytest.mark.gpu
@pytest.mark.parametrize("devices,kind", [([0, 0], "chk"), ([0, 0, 0], "sin"),
                                          ([0, 0, 0, 0, 0], "chk")])
def test_solve_multi_equals_emulation(devices, kind):
    """eik_solve_multi: strips on the listed devices (here several strips on
    one GPU; the rounds' kernels never wait on each other), edge rows by peer
    copy -- the serial emulation of the same rounds bit for bit."""
    p = _problem(m=73, n=131, kind=kind)
    out = E.solve_multi(p, "fsm", devices)
    u, k = emulate(p, len(devices))
    assert np.array_equal(out.values, u) and out.sweeps == k == out.rounds
    assert float(np.max(np.abs(out.values - O.oracle_solve(p, "fsm").u))) <= 1e-10
    fmm = E.solve_multi(p, "fmm", devices)
    ref = O.oracle_solve(p, "fmm")
    assert np.array_equal(fmm.values, u)
    assert (fmm.sweeps, fmm.node_updates, fmm.heap_removals) == (0, ref.node_updates,
                                                                ref.heap_removals)


@pytest.mark.gpu
def test_solve_multi_one_device_is_fsm():
    p = _problem()
    a = E.solve_multi(p, "fsm", [0])
    b = O.oracle_solve(p, "fsm")
    assert np.array_equal(a.values, b.u) and a.sweeps == b.sweeps
