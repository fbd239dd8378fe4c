"""Sharded FMSM (distributed.fmsm_solve_strips) on config 5 with ONE NCCL rank:
the level-by-level pass's device time and level count next to the single-GPU
dataflow (eik_plan_run).  Development aid.  usage: python scripts/fmsm_strips_c5.py [m] [cs]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_1110_6220_b200 as E  # noqa: E402
from paper_1110_6220_b200 import configs  # noqa: E402
from paper_1110_6220_b200.distributed import fmsm_schedule, fmsm_solve_strips  # noqa: E402

m = int(sys.argv[1]) if len(sys.argv) > 1 else 32769
cs = int(sys.argv[2]) if len(sys.argv) > 2 else 32
os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
os.environ.setdefault("MASTER_PORT", "29533")
torch.cuda.set_device(0)
dist.init_process_group("nccl", rank=0, world_size=1)
cfg = configs.config5(m)
p = cfg.problem
cells = E.build_cells(p.grid, cfg.cells_for(cs), cfg.cells_for(cs))
t0 = time.perf_counter()
s = fmsm_schedule(p, cells)
t1 = time.perf_counter()
print(f"schedule: {1e3 * (t1 - t0):.1f} ms host, levels {int(s.level.max()) + 1}, J {s.level.size}",
      flush=True)
for rep in range(2):
    r = fmsm_solve_strips(p, cells, gather="rank0")
    print(f"strips(1 rank): device {r.device_ms:.1f} ms, levels {r.levels}, sweeps {r.sweeps}",
          flush=True)
plan = E.Plan(p, "fmsm", cells)
u = np.empty(p.grid.size())
for rep in range(2):
    o = plan.run(u_host=u)
    print(f"dataflow: device {o.device_ms:.1f} ms + host {o.host_ms:.1f} ms, sweeps {o.sweeps}",
          flush=True)
print("bitwise equal:", bool(np.array_equal(u, r.values)), flush=True)
dist.destroy_process_group()
