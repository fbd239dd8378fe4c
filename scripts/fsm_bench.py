"""FSM wavefront timing per config (development aid).
usage: python scripts/fsm_bench.py [c1 c2 c3 c4 c5 ...]   (EIK_FSM_NOSKIP=1: no clean-step skip)
Prints device ms (best of 3 resident runs), sweeps, algorithmic GB/s (24 B/node/sweep)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1110_6220_b200 as E  # noqa: E402
from paper_1110_6220_b200 import configs  # noqa: E402

for name in sys.argv[1:] or ["c1", "c2", "c3", "c4"]:
    t0 = time.time()
    p = configs.CONFIGS[name]().problem
    plan = E.Plan(p, "fsm")
    best = None
    for _ in range(3 if name != "c5" else 2):
        o = plan.run()
        best = o if best is None or o.device_ms < best.device_ms else best
    M = p.grid.m * p.grid.n
    gbs = 24.0 * M * best.sweeps / (best.device_ms * 1e-3) / 1e9
    print(f"{name} fsm m={p.grid.m} device_ms={best.device_ms:.3f} sweeps={best.sweeps} "
          f"algGB/s={gbs:.1f} Mpts/s={M / best.device_ms / 1e3:.1f} (setup {time.time() - t0:.1f}s)",
          flush=True)
    del plan
