"""Run the FSM wavefront with on-device tracing and summarise the timeline."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1110_6220_b200 as E  # noqa: E402
from paper_1110_6220_b200 import configs  # noqa: E402

out_dir = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out"
cases = [("n64", E.build_problem(E.Grid(4096, 64, 1 / 64, 0, 0), E.speed_constant(),
                                 E.ExitSpec.node_set([(0, 0)]))),
         ("n256", E.build_problem(E.Grid(4096, 256, 1 / 64, 0, 0), E.speed_constant(),
                                  E.ExitSpec.node_set([(0, 0)]))),
         ("c2", configs.config2().problem)]
only = sys.argv[2:] if len(sys.argv) > 2 else None
if only and "c5" in only:
    cases.append(("c5", configs.config5().problem))
for name, p in cases:
    if only and name not in only:
        continue
    plan = E.Plan(p, "fsm")
    plan.run()
    path = os.path.join(out_dir, f"trace_{name}.txt")
    os.environ["EIK_TRACE_FSM"] = path
    E.lib.eik_debug_reload_knobs()  # knobs are read once per process
    o = plan.run()
    del os.environ["EIK_TRACE_FSM"]
    E.lib.eik_debug_reload_knobs()
    rows = [tuple(int(x) for x in line.split()) for line in open(path)]
    t0 = min(r[2] for r in rows)
    print(f"== {name}: sweeps={o.sweeps} dev_ms={o.device_ms:.3f}")
    nstr = max(r[1] for r in rows) + 1
    for k in sorted(set(r[0] for r in rows)):
        rk = sorted([r for r in rows if r[0] == k], key=lambda r: r[1])
        pick = rk if nstr <= 8 else [rk[0], rk[1], rk[len(rk) // 2], rk[-2], rk[-1]]
        s = "  ".join(f"b{r[1]}:[{(r[2]-t0)/1e3:.1f} w{(r[3]-r[2])/1e3:.1f} "
                      f"body{(r[4]-r[3])/1e3:.1f} p{r[5]} c{r[6]}]" for r in pick)
        print(f" k={k:2d} {s}")
    plan.close()
