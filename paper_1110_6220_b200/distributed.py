"""Strip-Jacobi FSM across ranks (option A).

fsm_solve (classic_solvers.cpp:128-158) on one grid, split into row strips:
rank r owns rows [n*r/P, n*(r+1)/P) and holds one frozen ghost row on each
side.  Round k:

  1. every rank runs one Gauss-Seidel sweep in direction k mod 4 over its
     strip (the device wavefront kernel, bit-exact within the strip); the
     ghost rows are read as fixed neighbours (+inf at the domain edge, the
     off-grid value of gather_neighbors, local_update.hpp:67-74);
  2. the ranks exchange edge rows (ghost rows <- the neighbours' edge rows)
     with point-to-point send/recv, and all-reduce the change flag (MAX).

The loop stops after the first round in which no strip changed anything: that
round read ghost rows equal to the post-round state, so the field satisfies
every node's update equation with its true neighbours -- the discrete fixed
point fsm_solve converges to (parity <= 1e-10; SURVEY A.11 measured 6e-16).
The round count exceeds the single-domain sweep count (22 -> 29 at P = 2..8,
SURVEY A.11); with P = 1 it is the reference's, and the field is bit-exact.
node_updates follows the reference's accounting: sweeps x (M - |Q|).

One process per GPU over torch.distributed: NCCL (CUDA tensors, exchange
device to device) on GPUs; gloo (CPU tensors) for the multi-process CPU tests,
where tests/ plug in the oracle's sweep instead of the device plan.
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass
from typing import Callable, Optional

import numpy as np

from . import _native as N
from .problem import Grid, Problem


def strip_bounds(n: int, world: int, rank: int):
    """Rows [r0, r1) owned by `rank` (balanced, every strip non-empty)."""
    if world < 1 or world > n:
        raise N.ConfigError(f"cannot split {n} rows over {world} ranks")
    return n * rank // world, n * (rank + 1) // world


def strip_speed(problem: Problem, r0: int, r1: int) -> np.ndarray:
    """F on rows [r0, r1) only, at the GLOBAL node coordinates (bit-identical
    to the whole grid's sampling): a rank never materialises the full field."""
    from .problem import SpeedField
    g = problem.grid
    if problem._F is not None:  # already sampled (e.g. a caller-provided array)
        return problem._F.reshape(g.n, g.m)[r0:r1]
    out = np.empty((r1 - r0) * g.m, dtype=np.float64)
    if isinstance(problem.speed, SpeedField):
        import os
        gc = g.c()
        N.raise_for(N.lib.eik_field_sample_rows(C.byref(problem.speed.cfield), C.byref(gc), r0,
                                                r1 - r0, N.dptr(out), min(32, os.cpu_count() or 1)))
    else:
        xs = g.x0 + np.arange(g.m, dtype=np.float64) * g.h
        ys = g.y0 + np.arange(r0, r1, dtype=np.float64) * g.h  # Grid::y(j) = y0 + j*h
        X, Y = np.meshgrid(xs, ys)
        out[:] = np.asarray(problem.speed(X, Y), dtype=np.float64).reshape(-1)
    return out.reshape(r1 - r0, g.m)


def strip_problem(problem: Problem, r0: int, r1: int) -> Problem:
    """The strip's own problem: rows [r0-1, r1] of the grid (local rows 0 and
    nl-1 are the ghost rows), exits = the strip's exits plus every ghost node
    (frozen; their values are set after prepare and after each exchange).
    Only the strip's rows of F are sampled (memory ~1/P of the grid)."""
    g = problem.grid
    m = g.m
    nl = r1 - r0 + 2
    Fl = np.ones((nl, m), dtype=np.float64)  # ghost rows: any positive speed
    Fl[1:-1] = strip_speed(problem, r0, r1)
    ex = np.asarray(problem.exit_nodes, dtype=np.int64)
    ec = np.asarray(problem.exit_cost, dtype=np.float64)
    rows = ex // m
    sel = (rows >= r0) & (rows < r1)
    own = ex[sel] - (r0 - 1) * m
    nodes = np.concatenate([np.arange(m, dtype=np.int64), own,
                            (nl - 1) * m + np.arange(m, dtype=np.int64)])
    cost = np.concatenate([np.zeros(m), ec[sel], np.zeros(m)])
    lg = Grid(m, nl, g.h, g.x0, g.y0 + (r0 - 1) * g.h)
    return Problem(lg, None, nodes, cost, _F=np.ascontiguousarray(Fl.reshape(-1)))


class DeviceStripSweeper:
    """The strip on the device: an FSM plan driven sweep by sweep
    (eik_plan_prepare / eik_plan_sweep / eik_plan_get_rows / _set_rows)."""

    def __init__(self, local: Problem):
        from .solvers import Plan
        try:
            import torch
            if torch.cuda.is_available() and torch.cuda.is_initialized():
                N.raise_for(N.lib.eik_set_device(torch.cuda.current_device()))
        except ImportError:
            pass
        self.plan = Plan(local, "fsm")
        self.m, self.nl = local.grid.m, local.grid.n
        N.raise_for(N.lib.eik_plan_prepare(self.plan._h))

    def sweep(self, k: int) -> bool:
        ch = (C.c_int32 * 1)()
        N.raise_for(N.lib.eik_plan_sweep(self.plan._h, k, 1, ch))
        return bool(ch[0])

    # stream-ordered variants (no host synchronisation): the round runs on the
    # caller's CUDA stream, the change flag lands in a device int32 tensor
    def sweep_async(self, k: int, flag, stream: int) -> None:
        N.raise_for(N.lib.eik_plan_sweep_async(self.plan._h, k, 1, C.c_void_p(flag.data_ptr()),
                                               C.c_void_p(stream)))

    def rows_async(self, row0: int, nrows: int, buf, to_plan: bool, stream: int) -> None:
        N.raise_for(N.lib.eik_plan_rows_async(self.plan._h, row0, nrows,
                                              C.c_void_p(buf.data_ptr()), 1 if to_plan else 0,
                                              C.c_void_p(stream)))

    @staticmethod
    def _ptr(buf):
        if isinstance(buf, np.ndarray):
            return buf.ctypes.data, 0
        return buf.data_ptr(), int(buf.is_cuda)

    def get_rows(self, row0: int, nrows: int, out) -> None:
        p, dev = self._ptr(out)
        N.raise_for(N.lib.eik_plan_get_rows(self.plan._h, row0, nrows, C.c_void_p(p), dev))

    def set_rows(self, row0: int, nrows: int, src) -> None:
        p, dev = self._ptr(src)
        N.raise_for(N.lib.eik_plan_set_rows(self.plan._h, row0, nrows, C.c_void_p(p), dev))

    def close(self):
        self.plan.close()


@dataclass
class StripSolve:
    values: Optional[np.ndarray]  # the m*n field (gather="all", or rank 0 with "rank0"),
                                  # this rank's rows (gather="none"), else None
    sweeps: int             # rounds, including the final unchanged one
    node_updates: int       # sweeps * (M - |Q|), the reference's accounting
    rows: tuple             # this rank's [r0, r1)
    device_ms: float = 0.0  # the rounds (max over ranks on GPUs), CUDA events


LOOKAHEAD = 2  # rounds enqueued beyond the last one whose change flag was read


def fsm_solve_strips(problem: Problem, group=None,
                     sweeper_factory: Optional[Callable[[Problem], object]] = None,
                     max_rounds: Optional[int] = None, gather: str = "all") -> StripSolve:
    """fsm_solve over the ranks of `group` (torch.distributed), strip-Jacobi.
    Without an initialised process group it runs as a single strip.

    On GPUs (NCCL) a round is enqueued on the current CUDA stream with no host
    synchronisation -- sweep (eik_plan_sweep_async), edge rows into send
    buffers, NCCL send/recv, ghost rows back, all-reduce(MAX) of the change
    flag, its copy into pinned memory -- and the host reads the flag of the
    round LOOKAHEAD behind, so the device never idles on the host; rounds
    enqueued past the first unchanged one change nothing (a fixed point stays
    fixed) and the count reported is the first unchanged round's.
    gather: "all" (every rank gets the field), "rank0", or "none" (each rank
    keeps its own rows)."""
    import torch
    import torch.distributed as dist

    if dist.is_available() and dist.is_initialized():
        rank, world = dist.get_rank(group), dist.get_world_size(group)
        on_gpu = dist.get_backend(group) == "nccl"
    else:
        rank, world, on_gpu = 0, 1, False
    g = problem.grid
    m, n = g.m, g.n
    r0, r1 = strip_bounds(n, world, rank)
    local = strip_problem(problem, r0, r1)
    nl = local.grid.n
    sw = (sweeper_factory or DeviceStripSweeper)(local)
    dev = torch.device("cuda", torch.cuda.current_device()) if on_gpu else torch.device("cpu")
    row = lambda: torch.empty(m, dtype=torch.float64, device=dev)  # noqa: E731
    inf_row = torch.full((m,), math.inf, dtype=torch.float64, device=dev)

    def put(r, t):
        sw.set_rows(r, 1, t if on_gpu else t.numpy())

    def take(r, t):
        sw.get_rows(r, 1, t if on_gpu else t.numpy())

    put(0, inf_row)        # below row 0 / above row n-1 the field is off-grid
    put(nl - 1, inf_row)
    send_lo, send_hi, recv_lo, recv_hi = row(), row(), row(), row()
    limit = max_rounds if max_rounds is not None else 4 * (m + n) + 16
    k = 0
    dev_ms = 0.0
    if on_gpu and hasattr(sw, "sweep_async"):
        k, dev_ms = _rounds_async(sw, rank, world, group, nl, limit, send_lo, send_hi, recv_lo,
                                  recv_hi, dev)
    else:
        while True:
            if k >= limit:
                raise N.BudgetError("strip-Jacobi FSM did not converge within the round budget")
            changed = sw.sweep(k)
            k += 1
            if world > 1:
                ops = []
                if rank > 0:
                    take(1, send_lo)
                    ops += [dist.P2POp(dist.isend, send_lo, rank - 1, group),
                            dist.P2POp(dist.irecv, recv_lo, rank - 1, group)]
                if rank < world - 1:
                    take(nl - 2, send_hi)
                    ops += [dist.P2POp(dist.isend, send_hi, rank + 1, group),
                            dist.P2POp(dist.irecv, recv_hi, rank + 1, group)]
                for w in dist.batch_isend_irecv(ops):
                    w.wait()
                if on_gpu:
                    torch.cuda.current_stream().synchronize()
                if rank > 0:
                    put(0, recv_lo)
                if rank < world - 1:
                    put(nl - 1, recv_hi)
                flag = torch.tensor([1 if changed else 0], dtype=torch.int32, device=dev)
                dist.all_reduce(flag, op=dist.ReduceOp.MAX, group=group)
                changed = bool(flag.item())
            if not changed:
                break
    # the field: every rank ("all"), rank 0 ("rank0") or each its own rows
    own = np.empty((r1 - r0) * m, dtype=np.float64)
    sw.get_rows(1, r1 - r0, own)
    u = own
    if world > 1 and gather != "none":
        rows_max = max(strip_bounds(n, world, r)[1] - strip_bounds(n, world, r)[0]
                       for r in range(world))
        buf = torch.full((rows_max * m,), math.inf, dtype=torch.float64, device=dev)
        buf[: own.size] = torch.from_numpy(own).to(dev)
        if gather == "all":
            parts = [torch.empty_like(buf) for _ in range(world)]
            dist.all_gather(parts, buf, group=group)
        else:
            parts = [torch.empty_like(buf) for _ in range(world)] if rank == 0 else None
            dist.gather(buf, parts, dst=0, group=group)
        if parts is not None:
            u = np.empty(n * m, dtype=np.float64)
            for r in range(world):
                a, b = strip_bounds(n, world, r)
                u[a * m:b * m] = parts[r][: (b - a) * m].cpu().numpy()
        else:
            u = None
    close = getattr(sw, "close", None)
    if close:
        close()
    return StripSolve(u, k, k * (m * n - len(problem.exit_nodes)), (r0, r1), dev_ms)


def _rounds_async(sw, rank, world, group, nl, limit, send_lo, send_hi, recv_lo, recv_hi, dev):
    """The rounds on the device, stream-ordered (see fsm_solve_strips);
    returns (rounds, device ms of the rounds, max over ranks)."""
    import torch
    import torch.distributed as dist

    # a stream of our own: the default stream's handle is 0, which the ABI
    # reads as "the plan's stream" (not ordered with torch's work)
    stream = torch.cuda.Stream(dev)
    stream.wait_stream(torch.cuda.current_stream(dev))
    with torch.cuda.stream(stream):
        out = _rounds_on(stream, sw, rank, world, group, nl, limit, send_lo, send_hi, recv_lo,
                         recv_hi, dev)
    torch.cuda.current_stream(dev).wait_stream(stream)
    return out


def _rounds_on(stream, sw, rank, world, group, nl, limit, send_lo, send_hi, recv_lo, recv_hi,
               dev):
    import torch
    import torch.distributed as dist

    sh = stream.cuda_stream
    ring = 8
    flags = torch.zeros(ring, dtype=torch.int32, device=dev)
    host = torch.zeros(limit + 1, dtype=torch.int32, pin_memory=True)
    events = [None] * ring
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    k = 0
    done_at = None
    while done_at is None:
        if k >= limit:
            raise N.BudgetError("strip-Jacobi FSM did not converge within the round budget")
        slot = k % ring
        if events[slot] is not None:
            events[slot].synchronize()  # ring slot free (LOOKAHEAD < ring, so already done)
        f = flags[slot:slot + 1]
        sw.sweep_async(k, f, sh)
        if world > 1:
            ops = []
            if rank > 0:
                sw.rows_async(1, 1, send_lo, False, sh)
                ops += [dist.P2POp(dist.isend, send_lo, rank - 1, group),
                        dist.P2POp(dist.irecv, recv_lo, rank - 1, group)]
            if rank < world - 1:
                sw.rows_async(nl - 2, 1, send_hi, False, sh)
                ops += [dist.P2POp(dist.isend, send_hi, rank + 1, group),
                        dist.P2POp(dist.irecv, recv_hi, rank + 1, group)]
            for w in dist.batch_isend_irecv(ops):
                w.wait()  # NCCL: the current stream waits; the host does not
            if rank > 0:
                sw.rows_async(0, 1, recv_lo, True, sh)
            if rank < world - 1:
                sw.rows_async(nl - 1, 1, recv_hi, True, sh)
            dist.all_reduce(f, op=dist.ReduceOp.MAX, group=group)
        host[k:k + 1].copy_(f, non_blocking=True)
        ev = torch.cuda.Event()
        ev.record(stream)
        events[slot] = ev
        j = k - LOOKAHEAD
        if j >= 0:
            events[j % ring].synchronize()
            if int(host[j]) == 0:
                done_at = j
        k += 1
    # rounds j+1 .. k-1 were enqueued past the fixed point: harmless
    e1.record(stream)
    e1.synchronize()
    ms = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(ms, op=dist.ReduceOp.MAX, group=group)
    return done_at + 1, float(ms.item())


# ---- FMSM sharded by row strips of cells --------------------
#
# fmsm_solve (fmsm.cpp:126-226): Part I (the coarse Fast March and its
# quantised order) is computed by every rank identically on the host; Part II
# -- one pass over the cells in rank order, a cell reading only its nodes and
# its cross halo -- runs by LEVELS of the cell DAG: level(c) = 0 without an
# earlier-ranked neighbour, else 1 + the largest level among them
# (eik_fmsm_schedule).  A cell's earlier-ranked neighbours lie in earlier
# levels and its later-ranked ones in later levels, so when level L runs, each
# of its cells sees exactly the inputs it sees in the reference's pass; the
# cells of one level are pairwise non-adjacent and run at once.  Rank r owns
# the cell rows [cy0, cy1) (their node rows plus a ghost row on each side);
# after a level that processed cells of its first / last cell row, it sends
# that edge row to the neighbour, which knows from the same schedule when to
# receive it.  The field, sweeps and node updates are fmsm_solve's bit for bit.


@dataclass
class FmsmSchedule:
    order: np.ndarray   # cells in coarse order
    rank: np.ndarray    # inverse of order
    flags: np.ndarray   # per cell: bit d = SweepDir d chosen, 16 = Q-cell
    level: np.ndarray   # per cell: DAG level
    coarse_pops: int
    coarse_updates: int


def fmsm_schedule(problem: Problem, cells, tables=None) -> FmsmSchedule:
    """Part I on the host through the C-ABI (eik_fmsm_schedule)."""
    from .problem import _eval_speed
    from .solvers import _c_problem
    # Part I reads neither F nor the border probes: only F at the cell
    # centres (fmsm.cpp:18-30), sampled here for the J centres alone
    F = problem._F if problem._F is not None else np.ones(1)
    p, keep_p = _c_problem(problem, F)
    J = cells.cells_x * cells.cells_y
    if tables is not None:
        centre = np.ascontiguousarray(tables.center, dtype=np.float64)
    else:
        g = problem.grid.c()
        cxy = np.empty((J, 2), dtype=np.float64)
        N.lib.eik_cell_centers(C.byref(g), cells.cells_x, cells.cells_y, N.dptr(cxy))
        centre = np.ascontiguousarray(_eval_speed(problem.speed, cxy), dtype=np.float64)
    c = N.eik_cells()
    c.cells_x, c.cells_y = cells.cells_x, cells.cells_y
    c.center_speed = N.dptr(centre)
    order = np.empty(J, dtype=np.int32)
    rank = np.empty(J, dtype=np.int32)
    flags = np.empty(J, dtype=np.uint8)
    level = np.empty(J, dtype=np.int32)
    cnt = np.zeros(2, dtype=np.int64)
    N.raise_for(N.lib.eik_fmsm_schedule(C.byref(p), C.byref(c), order.ctypes.data,
                                        rank.ctypes.data, flags.ctypes.data, level.ctypes.data,
                                        cnt.ctypes.data))
    return FmsmSchedule(order, rank, flags, level, int(cnt[0]), int(cnt[1]))


class DeviceFmsmStrip:
    """A strip of a sharded FMSM on the device (eik_plan_create_fmsm_strip):
    the strip's cells run level by level (eik_plan_fmsm_level_async)."""

    def __init__(self, local: Problem, cells_x: int, cells_y: int, base_y: int, row0: int,
                 row_end: int):
        from .solvers import _c_problem
        try:
            import torch
            if torch.cuda.is_available() and torch.cuda.is_initialized():
                N.raise_for(N.lib.eik_set_device(torch.cuda.current_device()))
        except ImportError:
            pass
        self._F = local.sampled_speed()
        p, self._keep = _c_problem(local, self._F)
        self._h = N.lib.eik_plan_create_fmsm_strip(C.byref(p), cells_x, cells_y, base_y, row0,
                                                   row_end)
        if not self._h:
            N.raise_for(N.lib.eik_last_status() or N.EIK_ERR_CUDA)

    def levels(self, cells_by_level: np.ndarray, level_off: np.ndarray, flags: np.ndarray):
        self._lv = (np.ascontiguousarray(cells_by_level, dtype=np.int32),
                    np.ascontiguousarray(level_off, dtype=np.int32),
                    np.ascontiguousarray(flags, dtype=np.uint8))
        N.raise_for(N.lib.eik_plan_fmsm_levels(self._h, self._lv[0].ctypes.data,
                                               self._lv[1].ctypes.data, len(level_off) - 1,
                                               self._lv[2].ctypes.data))

    def run_level(self, L: int, stream: int = 0) -> None:
        N.raise_for(N.lib.eik_plan_fmsm_level_async(self._h, int(L), C.c_void_p(stream)))

    def rows_async(self, row0: int, nrows: int, buf, to_plan: bool, stream: int) -> None:
        N.raise_for(N.lib.eik_plan_rows_async(self._h, row0, nrows, C.c_void_p(buf.data_ptr()),
                                              1 if to_plan else 0, C.c_void_p(stream)))

    def get_rows(self, row0: int, nrows: int, out) -> None:
        p, dev = DeviceStripSweeper._ptr(out)
        N.raise_for(N.lib.eik_plan_get_rows(self._h, row0, nrows, C.c_void_p(p), dev))

    def set_rows(self, row0: int, nrows: int, src) -> None:
        p, dev = DeviceStripSweeper._ptr(src)
        N.raise_for(N.lib.eik_plan_set_rows(self._h, row0, nrows, C.c_void_p(p), dev))

    def counters(self):
        out = np.zeros(2, dtype=np.int64)
        N.raise_for(N.lib.eik_plan_fmsm_counters(self._h, out.ctypes.data))
        return int(out[0]), int(out[1])

    def close(self):
        lib = getattr(N, "lib", None)
        if self._h and lib is not None:
            lib.eik_plan_destroy(self._h)
            self._h = None

    def __del__(self):
        self.close()


@dataclass
class FmsmStripSolve:
    values: Optional[np.ndarray]  # as StripSolve.values
    sweeps: int                   # fine-pass cell sweeps (fmsm.cpp:208,222)
    node_updates: int             # coarse + fine node updates (fmsm.cpp:173-174,183)
    heap_removals: int            # coarse Fast March removals (fmsm.cpp:173)
    levels: int                   # DAG levels of the fine pass
    exchanges: int                # edge rows this rank sent
    rows: tuple                   # this rank's node rows [r0, r1)
    device_ms: float = 0.0


def fmsm_solve_strips(problem: Problem, cells, tables=None, group=None,
                      strip_factory: Optional[Callable] = None,
                      gather: str = "all") -> FmsmStripSolve:
    """fmsm_solve over the ranks of `group`, row strips of cells, by levels of
    the cell DAG (see above).  Without a process group: one strip.  On GPUs
    (NCCL) the levels, edge-row copies and sends are enqueued on one CUDA
    stream with no host synchronisation."""
    import torch
    import torch.distributed as dist

    if dist.is_available() and dist.is_initialized():
        rank, world = dist.get_rank(group), dist.get_world_size(group)
        on_gpu = dist.get_backend(group) == "nccl"
    else:
        rank, world, on_gpu = 0, 1, False
    g = problem.grid
    m, n = g.m, g.n
    cx, cy = cells.cells_x, cells.cells_y
    sch = fmsm_schedule(problem, cells, tables)
    cy0, cy1 = strip_bounds(cy, world, rank)
    base_y = n // cy
    jb = lambda c: c * base_y  # noqa: E731  (cells.cpp:7-19: remainder to the last)
    je = lambda c: n if c == cy - 1 else (c + 1) * base_y  # noqa: E731
    r0, r1 = jb(cy0), je(cy1 - 1)
    local = strip_problem(problem, r0, r1)
    nl = local.grid.n
    sp = (strip_factory or DeviceFmsmStrip)(local, cx, cy1 - cy0, base_y, 1, 1 + r1 - r0)
    # the strip's cells grouped by level, by rank within a level
    lv = sch.level.reshape(cy, cx)
    mine = np.arange(cy0 * cx, cy1 * cx, dtype=np.int64)
    nlev = int(sch.level.max()) + 1
    key = sch.level[mine].astype(np.int64) * (cx * cy) + sch.rank[mine]
    srt = mine[np.argsort(key, kind="stable")]
    counts = np.bincount(sch.level[mine], minlength=nlev)
    off = np.zeros(nlev + 1, dtype=np.int32)
    off[1:] = np.cumsum(counts)
    sp.levels((srt - cy0 * cx).astype(np.int32), off, sch.flags[mine])
    # when an edge row changes: the levels of the cells in my first / last cell
    # row (sent) and in the neighbours' adjacent rows (received)
    send_lo = set(lv[cy0].tolist()) if rank > 0 else set()
    send_hi = set(lv[cy1 - 1].tolist()) if rank < world - 1 else set()
    recv_lo = set(lv[cy0 - 1].tolist()) if rank > 0 else set()
    recv_hi = set(lv[cy1].tolist()) if rank < world - 1 else set()
    dev = torch.device("cuda", torch.cuda.current_device()) if on_gpu else torch.device("cpu")
    bufs = [torch.empty(m, dtype=torch.float64, device=dev) for _ in range(4)]
    inf_row = torch.full((m,), math.inf, dtype=torch.float64, device=dev)

    def swap(do_send_lo, do_send_hi, do_recv_lo, do_recv_hi, stream):
        ops = []
        if do_send_lo:
            take(1, bufs[0], stream)
            ops.append(dist.P2POp(dist.isend, bufs[0], rank - 1, group))
        if do_recv_lo:
            ops.append(dist.P2POp(dist.irecv, bufs[1], rank - 1, group))
        if do_send_hi:
            take(nl - 2, bufs[2], stream)
            ops.append(dist.P2POp(dist.isend, bufs[2], rank + 1, group))
        if do_recv_hi:
            ops.append(dist.P2POp(dist.irecv, bufs[3], rank + 1, group))
        if ops:
            for w in dist.batch_isend_irecv(ops):
                w.wait()
        if do_recv_lo:
            put(0, bufs[1], stream)
        if do_recv_hi:
            put(nl - 1, bufs[3], stream)
        return int(do_send_lo) + int(do_send_hi)

    def take(r, t, stream):
        if on_gpu:
            sp.rows_async(r, 1, t, False, stream)
        else:
            sp.get_rows(r, 1, t.numpy())

    def put(r, t, stream):
        if on_gpu:
            sp.rows_async(r, 1, t, True, stream)
        else:
            sp.set_rows(r, 1, t.numpy())

    sent = 0
    dev_ms = 0.0

    def levels_loop(stream):
        nonlocal sent
        sh = stream.cuda_stream if stream is not None else 0
        # ghost rows: +inf past the grid, else the neighbour's prepared edge row
        put(0, inf_row, sh)
        put(nl - 1, inf_row, sh)
        sent += swap(rank > 0, rank < world - 1, rank > 0, rank < world - 1, sh)
        for L in range(nlev):
            if off[L + 1] > off[L]:
                sp.run_level(L, sh)
            if world > 1:
                sent += swap(L in send_lo, L in send_hi, L in recv_lo, L in recv_hi, sh)

    if on_gpu:
        stream = torch.cuda.Stream(dev)
        stream.wait_stream(torch.cuda.current_stream(dev))
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(stream):
            e0.record(stream)
            levels_loop(stream)
            e1.record(stream)
        e1.synchronize()
        torch.cuda.current_stream(dev).wait_stream(stream)
        ms = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(ms, op=dist.ReduceOp.MAX, group=group)
        dev_ms = float(ms.item())
    else:
        levels_loop(None)
    sweeps, updates = sp.counters()
    if world > 1:
        t = torch.tensor([sweeps, updates], dtype=torch.int64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
        sweeps, updates = int(t[0]), int(t[1])
    own = np.empty((r1 - r0) * m, dtype=np.float64)
    sp.get_rows(1, r1 - r0, own)
    u = own
    if world > 1 and gather != "none":
        bounds = [(jb(strip_bounds(cy, world, r)[0]), je(strip_bounds(cy, world, r)[1] - 1))
                  for r in range(world)]
        rows_max = max(b - a for a, b in bounds)
        buf = torch.full((rows_max * m,), math.inf, dtype=torch.float64, device=dev)
        buf[: own.size] = torch.from_numpy(own).to(dev)
        if gather == "all":
            parts = [torch.empty_like(buf) for _ in range(world)]
            dist.all_gather(parts, buf, group=group)
        else:
            parts = [torch.empty_like(buf) for _ in range(world)] if rank == 0 else None
            dist.gather(buf, parts, dst=0, group=group)
        if parts is not None:
            u = np.empty(n * m, dtype=np.float64)
            for r, (a, b) in enumerate(bounds):
                u[a * m:b * m] = parts[r][: (b - a) * m].cpu().numpy()
        else:
            u = None
    close = getattr(sp, "close", None)
    if close:
        close()
    return FmsmStripSolve(u, sweeps, sch.coarse_updates + updates, sch.coarse_pops, nlev, sent,
                          (r0, r1), dev_ms)
