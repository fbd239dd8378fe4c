"""BASELINE.json configurations as seeded synthetic problems.

All grids are Grid(m, m, 2/(m-1), -1, -1) on [-1,1]^2;
with m-1 a power of two every node coordinate is an exact binary fraction.
No public dataset is involved; every input is generated here from a seed.
"""
from __future__ import annotations

import math
from dataclasses import dataclass
from typing import List, Optional

import numpy as np

from .problem import (ExitSpec, Grid, Problem, build_problem, speed_blocks, speed_constant,
                      speed_nodemask, speed_sinsum, speed_sinusoid)


@dataclass
class Config:
    name: str
    problem: Problem
    methods: List[str]
    cell_sizes: List[int]  # points per cell side; cells per axis = m // size

    def cells_for(self, size: int) -> int:
        return max(1, self.problem.grid.m // size)


def config1(m: int = 257) -> Config:
    """C1: F = 1, centre point source; exact solution |x| (PR1 oracle)."""
    g = Grid.centered(m)
    p = build_problem(g, speed_constant(), ExitSpec.point_source((0.0, 0.0)))
    return Config("c1_constant", p, ["fmm", "fsm", "fmsm"], [16])


def config2(m: int = 2049) -> Config:
    """C2: F = 1 + 0.5 sin(20 pi x) sin(20 pi y), centre source."""
    g = Grid.centered(m)
    p = build_problem(g, speed_sinusoid(0.5, 20), ExitSpec.point_source((0.0, 0.0)))
    return Config("c2_sinusoid", p, ["fmm", "fsm", "fmsm", "hcm", "fhcm"], [8, 16, 32, 64])


def config3(m: int = 4097, seed: Optional[int] = None) -> Config:
    """C3: 8x8 blocks, F = 1 / 2 alternating (or iid {0.5,1,2} from `seed`)."""
    g = Grid.centered(m)
    bx, by = np.meshgrid(np.arange(8), np.arange(8))
    if seed is None:
        bs = np.where((bx + by) % 2 == 0, 1.0, 2.0)
    else:
        rng = np.random.default_rng(seed)
        bs = rng.choice(np.array([0.5, 1.0, 2.0]), size=(8, 8))
    # b = clamp(floor((x+1)*4), 0, 7)
    p = build_problem(g, speed_blocks(bs, -1.0, -1.0, 4.0), ExitSpec.point_source((0.0, 0.0)))
    return Config("c3_checker", p, ["fmm", "fsm", "fmsm", "hcm", "fhcm"], [16, 32, 64, 24, 48])


def maze_mask(m: int, seed: int = 4, area_frac: float = 0.05, thick: int = 4) -> np.ndarray:
    """Seeded axis-aligned wall segments `thick` nodes thick, each with at
    least one gap, until walls cover ~area_frac of the nodes; the corner
    source region is kept clear."""
    rng = np.random.default_rng(seed)
    mask = np.zeros((m, m), dtype=np.uint8)
    target = area_frac * m * m
    while mask.sum(dtype=np.int64) < target:
        horiz = rng.random() < 0.5
        length = int(rng.integers(m // 8, m // 2))
        a = int(rng.integers(0, m - thick))          # position across the wall
        s = int(rng.integers(0, max(1, m - length)))  # start along the wall
        gap_w = int(rng.integers(max(8, m // 128), max(9, m // 32)))
        ngap = int(rng.integers(1, 4))
        seg = np.ones(length, dtype=bool)
        for _ in range(ngap):
            gpos = int(rng.integers(0, max(1, length - gap_w)))
            seg[gpos:gpos + gap_w] = False
        if horiz:
            mask[a:a + thick, s:s + length] |= seg[None, :]
        else:
            mask[s:s + length, a:a + thick] |= seg[:, None]
    clear = max(8, m // 64)
    mask[:clear, :clear] = 0  # source at the (0,0) corner is never in a wall
    return mask


def config4(m: int = 4097, seed: int = 4) -> Config:
    """C4: maze, walls F = 0.01 (5% of the area), F = 1 elsewhere, corner source."""
    g = Grid.centered(m)
    mask = maze_mask(m, seed)
    p = build_problem(g, speed_nodemask(g, mask, 0.01, 1.0), ExitSpec.point_source((-1.0, -1.0)))
    return Config("c4_maze", p, ["fmm", "fsm", "fmsm", "hcm", "fhcm"], [16, 32])


def sinsum_coeffs(seed: int = 5, K: int = 16):
    rng = np.random.default_rng(seed)
    p = np.zeros(K)
    q = np.zeros(K)
    for k in range(K):
        while True:
            a, b = rng.integers(-32, 33, size=2)
            if 1 <= max(abs(a), abs(b)) <= 32:
                break
        p[k], q[k] = a, b
    phi = rng.uniform(0.0, 2.0 * math.pi, size=K)
    return p, q, phi


def config5(m: int = 32769, seed: int = 5, n_sources: int = 64) -> Config:
    """C5: F = 1 + 0.5*S/16 (16 random-phase sinusoids, wavenumbers 1..32),
    64 random point-node sources; row strips across GPUs."""
    g = Grid.centered(m)
    p, q, phi = sinsum_coeffs(seed)
    rng = np.random.default_rng(seed + 1000)
    flat = rng.choice(m * m, size=n_sources, replace=False)
    nodes = [(int(k % m), int(k // m)) for k in flat]
    prob = build_problem(g, speed_sinsum(p, q, phi), ExitSpec.node_set(nodes))
    return Config("c5_sinsum", prob, ["fsm", "fhcm"], [16, 32])


CONFIGS = {"c1": config1, "c2": config2, "c3": config3, "c4": config4, "c5": config5}
