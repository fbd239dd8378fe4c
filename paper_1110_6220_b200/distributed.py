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


def strip_problem(problem: Problem, r0: int, r1: int) -> Problem:
    """The strip's own problem: rows [r0-1, r1] of the grid (local rows 0 and
    nl-1 are the ghost rows), exits = the strip's exits plus every ghost node
    (frozen; their values are set after prepare and after each exchange)."""
    g = problem.grid
    m = g.m
    nl = r1 - r0 + 2
    F = problem.sampled_speed().reshape(g.n, m)
    Fl = np.ones((nl, m), dtype=np.float64)  # ghost rows: any positive speed
    Fl[1:-1] = F[r0:r1]
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
    values: np.ndarray      # the full m*n field (every rank)
    sweeps: int             # rounds, including the final unchanged one
    node_updates: int       # sweeps * (M - |Q|), the reference's accounting
    rows: tuple             # this rank's [r0, r1)


def fsm_solve_strips(problem: Problem, group=None,
                     sweeper_factory: Optional[Callable[[Problem], object]] = None,
                     max_rounds: Optional[int] = None) -> StripSolve:
    """fsm_solve over the ranks of `group` (torch.distributed), strip-Jacobi.
    Without an initialised process group it runs as a single strip."""
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
    # assemble the full field on every rank (strips padded to the largest)
    own = np.empty((r1 - r0) * m, dtype=np.float64)
    sw.get_rows(1, r1 - r0, own)
    if world > 1:
        rows_max = max(strip_bounds(n, world, r)[1] - strip_bounds(n, world, r)[0]
                       for r in range(world))
        buf = torch.full((rows_max * m,), math.inf, dtype=torch.float64, device=dev)
        buf[: own.size] = torch.from_numpy(own).to(dev)
        parts = [torch.empty_like(buf) for _ in range(world)]
        dist.all_gather(parts, buf, group=group)
        u = np.empty(n * m, dtype=np.float64)
        for r in range(world):
            a, b = strip_bounds(n, world, r)
            u[a * m:b * m] = parts[r][: (b - a) * m].cpu().numpy()
    else:
        u = own
    close = getattr(sw, "close", None)
    if close:
        close()
    return StripSolve(u, k, k * (m * n - len(problem.exit_nodes)), (r0, r1))
