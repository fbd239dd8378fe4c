"""Host-side problem types: a Python mirror of the reference's L0 types.

Mirrors /root/reference/proj/include/eikonal/grid.hpp (Grid, Problem,
ExitSpec, build_problem, snap_point_to_node), cells.hpp (build_cells) and the
speed-field layer.  Speed functions are either native fields (evaluated in C
with the reference's libm, so sampled F is bit-identical to what the
reference's on-demand SpeedFn returns) or any Python callable f(x, y) that
accepts float64 arrays.
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field
from typing import Callable, List, Optional, Sequence, Tuple, Union

import numpy as np

from . import _native as N
from ._native import ConfigError

INF = math.inf


@dataclass(frozen=True)
class Grid:
    """Uniform node lattice (grid.hpp:36-58): node (i,j) at (x0+i*h, y0+j*h)."""
    m: int
    n: int
    h: float
    x0: float = 0.0
    y0: float = 0.0

    def __post_init__(self):
        if self.m < 2 or self.n < 2:
            raise ConfigError("grid needs at least 2 nodes per axis")
        if not (self.h > 0.0):
            raise ConfigError("grid spacing must be positive")

    @staticmethod
    def unit_square(m: int) -> "Grid":
        if m < 2:
            raise ConfigError("grid needs at least 2 nodes per axis")
        return Grid(m, m, 1.0 / (m - 1))

    @staticmethod
    def centered(m: int) -> "Grid":
        """[-1,1]^2 with m nodes per axis: Grid(m, m, 2/(m-1), -1, -1)."""
        return Grid(m, m, 2.0 / (m - 1), -1.0, -1.0)

    def size(self) -> int:
        return self.m * self.n

    def index(self, i: int, j: int) -> int:
        return j * self.m + i

    def node(self, linear: int) -> Tuple[int, int]:
        return linear % self.m, linear // self.m

    def x(self, i) -> float:
        return self.x0 + i * self.h

    def y(self, j) -> float:
        return self.y0 + j * self.h

    def contains(self, i: int, j: int) -> bool:
        return 0 <= i < self.m and 0 <= j < self.n

    def c(self) -> N.eik_grid:
        return N.eik_grid(self.m, self.n, self.h, self.x0, self.y0)


def _snap_axis(t: float, count: int) -> int:
    lo = int(math.floor(t))
    lo = min(max(lo, 0), count - 1)
    hi = min(lo + 1, count - 1)
    idx = hi if (t - lo > 0.5) else lo  # t - lo == 0.5 resolves to lo
    return min(max(idx, 0), count - 1)


def snap_point_to_node(grid: Grid, p: Tuple[float, float]) -> Tuple[int, int]:
    """grid.cpp:22-41; raises ValueError (std::domain_error) outside the box."""
    eps = 1e-12 * grid.h
    x, y = p
    if (x < grid.x0 - eps or x > grid.x(grid.m - 1) + eps or
            y < grid.y0 - eps or y > grid.y(grid.n - 1) + eps):
        raise ValueError("point outside grid bounding box")
    return (_snap_axis((x - grid.x0) / grid.h, grid.m),
            _snap_axis((y - grid.y0) / grid.h, grid.n))


# ---- speed fields -------------------------------------------------------

class SpeedField:
    """Native speed field (include/eikonal_b200.h eik_field).  Keeps the
    numpy tables it points into alive."""

    def __init__(self, cfield: N.eik_field, keep=(), name: str = ""):
        self.cfield = cfield
        self._keep = keep
        self.name = name

    def __call__(self, x, y):
        x = np.asarray(x, dtype=np.float64)
        y = np.asarray(y, dtype=np.float64)
        xb, yb = np.broadcast_arrays(x, y)
        xy = np.ascontiguousarray(np.stack([xb.ravel(), yb.ravel()], axis=1))
        out = np.empty(xb.size, dtype=np.float64)
        N.raise_for(N.lib.eik_field_eval_points(C.byref(self.cfield), N.dptr(xy), xb.size,
                                                N.dptr(out)))
        return out.reshape(xb.shape) if xb.shape else float(out[0])

    def sample(self, grid: Grid, threads: int = 0) -> np.ndarray:
        import os
        out = np.empty(grid.size(), dtype=np.float64)
        g = grid.c()
        th = threads or min(32, os.cpu_count() or 1)
        N.raise_for(N.lib.eik_field_sample(C.byref(self.cfield), C.byref(g), N.dptr(out), th))
        return out


def speed_constant(value: float = 1.0) -> SpeedField:
    return SpeedField(N.eik_field(kind=N.EIK_FIELD_CONSTANT, value=value), name="constant")


def speed_sinusoid(amplitude: float, freq: int) -> SpeedField:
    """1 + a sin(freq pi x) sin(freq pi y) (speed_fields.cpp:27-29, :76-83)."""
    if not abs(amplitude) < 1.0:
        raise ConfigError("sinusoid amplitude must satisfy |a| < 1")
    return SpeedField(N.eik_field(kind=N.EIK_FIELD_SINUSOID, amp=amplitude, freq=freq),
                      name=f"sinusoid({amplitude},{freq})")


def speed_checkerboard(k: int, slow: float = 1.0, fast: float = 2.0) -> SpeedField:
    """Unit-square k x k checkerboard (speed_fields.cpp:23-26, :62-74)."""
    if k < 1 or k % 2 == 0:
        raise ConfigError("checkerboard needs an odd checker count")
    if not (slow > 0.0 and fast > 0.0):
        raise ConfigError("checkerboard speeds must be positive")
    return SpeedField(N.eik_field(kind=N.EIK_FIELD_CHECKER, checkers=k, slow=slow, fast=fast),
                      name=f"checker{k}")


def speed_comb_maze(n_barriers: int, barrier_speed: float = 0.01,
                    barrier_width: float = 1.0 / 11.0,
                    gap_fraction: float = 1.0 / 11.0) -> SpeedField:
    """speed_fields.cpp:30-41, :85-100."""
    if n_barriers < 1:
        raise ConfigError("comb maze needs >= 1 barrier")
    if not barrier_speed > 0.0:
        raise ConfigError("barrier speed must be positive")
    if barrier_width >= 1.0 / (n_barriers + 1):
        raise ConfigError("comb barriers overlap")
    if gap_fraction <= 0.0 or gap_fraction >= 1.0:
        raise ConfigError("gap fraction must lie in (0,1)")
    return SpeedField(N.eik_field(kind=N.EIK_FIELD_COMB, n_barriers=n_barriers,
                                  barrier_speed=barrier_speed, barrier_width=barrier_width,
                                  gap_fraction=gap_fraction), name=f"comb{n_barriers}")


def speed_blocks(block_speed: np.ndarray, x0: float, y0: float, scale: float) -> SpeedField:
    """nb x nb piecewise-constant blocks: b = clamp(floor((x-x0)*scale), 0, nb-1)."""
    bs = np.ascontiguousarray(block_speed, dtype=np.float64)
    nb = bs.shape[0]
    if bs.shape != (nb, nb) or not np.all(bs > 0):
        raise ConfigError("block speeds must be a positive nb x nb table")
    f = N.eik_field(kind=N.EIK_FIELD_BLOCKS, nb=nb, bx0=x0, by0=y0, bscale=scale,
                    block_speed=N.dptr(bs))
    return SpeedField(f, keep=(bs,), name=f"blocks{nb}")


def speed_nodemask(grid: Grid, mask: np.ndarray, slow: float, fast: float) -> SpeedField:
    """F = slow where the nearest mask node is set, fast elsewhere."""
    mk = np.ascontiguousarray(mask, dtype=np.uint8).ravel()
    if mk.size != grid.size():
        raise ConfigError("mask must have m*n entries")
    f = N.eik_field(kind=N.EIK_FIELD_NODEMASK, slow=slow, fast=fast, mask_grid=grid.c(),
                    mask=mk.ctypes.data_as(C.POINTER(C.c_uint8)))
    return SpeedField(f, keep=(mk,), name="nodemask")


def speed_sinsum(p: np.ndarray, q: np.ndarray, phi: np.ndarray) -> SpeedField:
    """1 + 0.5*S/K, S = sum_k sin(pi*(p_k x + q_k y) + phi_k), separable form."""
    p = np.ascontiguousarray(p, dtype=np.float64)
    q = np.ascontiguousarray(q, dtype=np.float64)
    phi = np.ascontiguousarray(phi, dtype=np.float64)
    f = N.eik_field(kind=N.EIK_FIELD_SINSUM, K=len(p), kp=N.dptr(p), kq=N.dptr(q),
                    kphi=N.dptr(phi))
    return SpeedField(f, keep=(p, q, phi), name=f"sinsum{len(p)}")


SpeedFn = Union[SpeedField, Callable]


def _eval_speed(speed: SpeedFn, xy: np.ndarray) -> np.ndarray:
    if isinstance(speed, SpeedField):
        out = np.empty(xy.shape[0], dtype=np.float64)
        N.raise_for(N.lib.eik_field_eval_points(C.byref(speed.cfield), N.dptr(xy),
                                                xy.shape[0], N.dptr(out)))
        return out
    return np.asarray(speed(xy[:, 0], xy[:, 1]), dtype=np.float64).reshape(-1)


# ---- exits and problems ---------------------------------------------------

@dataclass
class ExitSpec:
    """grid.hpp:84-108."""
    kind: str = "point"  # point | boundary | nodes
    point: Tuple[float, float] = (0.5, 0.5)
    point_cost: float = 0.0
    nodes: Sequence[Tuple[int, int]] = ()
    node_costs: Sequence[float] = ()

    @staticmethod
    def point_source(p, q: float = 0.0) -> "ExitSpec":
        return ExitSpec(kind="point", point=tuple(p), point_cost=q)

    @staticmethod
    def full_boundary() -> "ExitSpec":
        return ExitSpec(kind="boundary")

    @staticmethod
    def node_set(nodes, costs=()) -> "ExitSpec":
        return ExitSpec(kind="nodes", nodes=list(nodes), node_costs=list(costs))


@dataclass
class Problem:
    """grid.hpp:69-80."""
    grid: Grid
    speed: SpeedFn
    exit_nodes: np.ndarray  # int64, strictly ascending
    exit_cost: np.ndarray   # float64
    exit_points: np.ndarray = field(default_factory=lambda: np.zeros((0, 2)))
    exit_point_cost: np.ndarray = field(default_factory=lambda: np.zeros(0))
    _F: Optional[np.ndarray] = None

    def speed_at(self, i: int, j: int) -> float:
        return float(_eval_speed(self.speed, np.array([[self.grid.x(i), self.grid.y(j)]])) [0])

    def sampled_speed(self) -> np.ndarray:
        """F at every node, bit-identical to speed(x0+i*h, y0+j*h); cached."""
        if self._F is None:
            if isinstance(self.speed, SpeedField):
                self._F = self.speed.sample(self.grid)
            else:
                g = self.grid
                xs = g.x0 + np.arange(g.m, dtype=np.float64) * g.h
                ys = g.y0 + np.arange(g.n, dtype=np.float64) * g.h
                X, Y = np.meshgrid(xs, ys)
                self._F = np.ascontiguousarray(
                    np.asarray(self.speed(X, Y), dtype=np.float64).reshape(-1))
        return self._F


def build_problem(grid: Grid, speed: SpeedFn, exits: ExitSpec) -> Problem:
    """grid.cpp:43-90: snap / mark, sort, duplicates keep the smaller cost."""
    marked: List[Tuple[int, float]] = []
    pts = np.zeros((0, 2))
    pcost = np.zeros(0)
    if exits.kind == "point":
        i, j = snap_point_to_node(grid, exits.point)
        marked.append((grid.index(i, j), float(exits.point_cost)))
        pts = np.array([exits.point], dtype=np.float64)
        pcost = np.array([exits.point_cost], dtype=np.float64)
    elif exits.kind == "boundary":
        for j in range(grid.n):
            for i in range(grid.m):
                if i == 0 or i == grid.m - 1 or j == 0 or j == grid.n - 1:
                    marked.append((grid.index(i, j), 0.0))
    elif exits.kind == "nodes":
        for k, (i, j) in enumerate(exits.nodes):
            if not grid.contains(i, j):
                raise ConfigError("exit node outside grid")
            q = float(exits.node_costs[k]) if len(exits.node_costs) else 0.0
            if not math.isfinite(q):
                raise ConfigError("exit cost must be finite")
            marked.append((grid.index(i, j), q))
    else:
        raise ConfigError(f"unknown exit kind '{exits.kind}'")
    if not marked:
        raise ConfigError("exit set is empty")
    marked.sort()
    nodes: List[int] = []
    costs: List[float] = []
    for idx, q in marked:
        if nodes and nodes[-1] == idx:
            costs[-1] = min(costs[-1], q)
        else:
            nodes.append(idx)
            costs.append(q)
    return Problem(grid, speed, np.array(nodes, dtype=np.int64),
                   np.array(costs, dtype=np.float64), pts, pcost)


# ---- cell decomposition ------------------------------------------------------

def _split_axis(nodes: int, cells: int):
    base = nodes // cells
    b, e, at = [], [], 0
    for c in range(cells):
        b.append(at)
        at += base
        if c == cells - 1:
            at = nodes
        e.append(at)
    return b, e


@dataclass
class CellDecomposition:
    """cells.hpp:27-75 (build_cells, cells.cpp:32-47)."""
    grid: Grid
    cells_x: int
    cells_y: int
    hc_x: float
    hc_y: float
    i_begin: List[int]
    i_end: List[int]
    j_begin: List[int]
    j_end: List[int]

    def cell_count(self) -> int:
        return self.cells_x * self.cells_y

    def cell_index(self, cx: int, cy: int) -> int:
        return cy * self.cells_x + cx


def build_cells(grid: Grid, cells_x: int, cells_y: int) -> CellDecomposition:
    if cells_x < 1 or cells_y < 1:
        raise ConfigError("cell counts must be positive")
    if cells_x > grid.m or cells_y > grid.n:
        raise ConfigError("more cells than grid nodes along an axis")
    ib, ie = _split_axis(grid.m, cells_x)
    jb, je = _split_axis(grid.n, cells_y)
    return CellDecomposition(grid, cells_x, cells_y, (grid.m // cells_x) * grid.h,
                             (grid.n // cells_y) * grid.h, ib, ie, jb, je)


@dataclass
class CellTables:
    """Host-sampled speed tables the two-scale methods evaluate off-grid."""
    probe_w: np.ndarray
    probe_e: np.ndarray
    probe_s: np.ndarray
    probe_n: np.ndarray
    center: np.ndarray


def cell_tables(problem: Problem, cells: CellDecomposition) -> CellTables:
    g = problem.grid.c()
    tabs = []
    for side in range(4):
        cnt = N.lib.eik_cell_probe_points(C.byref(g), cells.cells_x, cells.cells_y, side, N.dptr(None))
        if cnt < 0:
            raise ConfigError("bad cell decomposition")
        xy = np.empty((cnt, 2), dtype=np.float64)
        N.lib.eik_cell_probe_points(C.byref(g), cells.cells_x, cells.cells_y, side, N.dptr(xy))
        tabs.append(_eval_speed(problem.speed, xy))
    J = cells.cell_count()
    cxy = np.empty((J, 2), dtype=np.float64)
    N.lib.eik_cell_centers(C.byref(g), cells.cells_x, cells.cells_y, N.dptr(cxy))
    return CellTables(*tabs, _eval_speed(problem.speed, cxy))
