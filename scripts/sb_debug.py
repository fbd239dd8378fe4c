"""Find where super-block skipping (EIK_FSM_SB) diverges from the plain
wavefront: per-sweep changed flags and the field after K sweeps, same launch.
usage: python scripts/sb_debug.py SEED"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1110_6220_b200 as E  # noqa: E402
from paper_1110_6220_b200.distributed import DeviceStripSweeper  # noqa: E402

seed = int(sys.argv[1]) if len(sys.argv) > 1 else 2
rng = np.random.default_rng(seed)
m, n = int(rng.integers(20, 300)), int(rng.integers(20, 300))
g = E.Grid(m, n, float(rng.uniform(0.001, 0.1)), 0.0, 0.0)
k = int(rng.integers(1, 12))
nodes = [(int(rng.integers(0, m)), int(rng.integers(0, n))) for _ in range(k)]
costs = list(rng.uniform(0, 0.5, size=k))
F = rng.uniform(0.05, 3.0, size=(n, m))
mask = rng.random((n, m)) < 0.1
F[mask] = 0.01
sp = lambda x, y, F=F, g=g: F[np.rint((y - g.y0) / g.h).astype(int),  # noqa: E731
                              np.rint((x - g.x0) / g.h).astype(int)]
p = E.build_problem(g, sp, E.ExitSpec.node_set(nodes, costs))
print("m", m, "n", n, "strips", (n + 31) // 32)


def run(sb, K):
    os.environ["EIK_FSM_SB"] = str(sb)
    E.lib.eik_debug_reload_knobs()
    s = DeviceStripSweeper(p)
    flags = s.plan.sweep(0, K)
    out = np.zeros((n, m))
    s.get_rows(0, n, out)
    s.close()
    return flags, out


K = 45
f1, _ = run(1, K)
f0, _ = run(0, K)
print("sb=1", "".join("1" if x else "0" for x in f1))
print("sb=0", "".join("1" if x else "0" for x in f0))
for K in range(1, 45):
    _, u1 = run(1, K)
    _, u0 = run(0, K)
    d = np.argwhere(u1.view(np.int64) != u0.view(np.int64))
    if len(d):
        print("first field difference after", K, "sweeps (sweep index", K - 1, "dir", (K - 1) & 3, "):", len(d), "nodes")
        for (j, i) in d[:12]:
            print("  row", j, "(strip", j // 32, "lane", j % 32, ") col", i, "sb", u1[j, i], "plain", u0[j, i])
        break
