"""Every BASELINE config with reference goldens (C2, C3, C4, C5 at 2049^2):
device time of each method alone on the GPU (resident plan, best of 2) next to
the unmodified reference's single-core time on the survey host (goldens'
`ms`), with the field's sha256 checked against the golden (parity).
Prints a markdown table.  usage: python scripts/config_table.py"""
import hashlib
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1110_6220_b200 as E  # noqa: E402
from paper_1110_6220_b200 import configs  # noqa: E402

gold = {}
for f in ("big.json", "c34.json", "c5.json"):
    with open(os.path.join(ROOT, "tests", "golden", f)) as fh:
        gold.update(json.load(fh))
builders = {"c2": lambda: configs.config2().problem, "c3": lambda: configs.config3().problem,
            "c4": lambda: configs.config4().problem, "c5_2049": lambda: configs.config5(2049).problem}
print("| case | points | B200 ms | reference ms (1 core) | speed-up | bit-exact |")
print("|---|---|---|---|---|---|")
for name, build in builders.items():
    keys = sorted(k for k in gold if k.startswith(name + "/") and "ms" in gold[k])
    if not keys:
        continue
    p = build()
    M = p.grid.m * p.grid.n
    u = np.empty(M)
    for key in keys:
        want = gold[key]
        parts = key.split("/")
        meth = parts[1]
        cells = E.build_cells(p.grid, want["cells"], want["cells"]) if len(parts) > 2 else None
        plan = E.Plan(p, meth, cells)
        best = None
        for _ in range(2):
            o = plan.run(u_host=u)
            t = o.device_ms + o.host_ms
            best = t if best is None or t < best else best
        plan.close()
        same = "—"
        if "sha256" in want:
            same = "yes" if hashlib.sha256(u.tobytes()).hexdigest() == want["sha256"] else "NO"
        print(f"| {key} | {M} | {best:.1f} | {want['ms']:.0f} | {want['ms'] / best:.0f}x | {same} |",
              flush=True)
