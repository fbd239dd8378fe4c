"""Per-sweep summary of an FSM trace file (scripts/fsm_trace.py output):
strip start spread (the fill), body durations, computed steps, polls.
usage: python scripts/fsm_trace_summary.py gpurun_out/trace_c2.txt"""
import collections
import sys

rows = [tuple(int(x) for x in line.split()) for line in open(sys.argv[1])]
t0 = min(r[2] for r in rows)
byk = collections.defaultdict(list)
for r in rows:
    byk[r[0]].append(r)
for k in sorted(byk):
    rk = sorted(byk[k], key=lambda r: r[1])
    n = len(rk)
    st = [(r[3] - t0) / 1e3 for r in rk]
    en = [(r[4] - t0) / 1e3 for r in rk]
    body = sorted((r[4] - r[3]) / 1e3 for r in rk)
    comp = sorted(r[6] for r in rk)
    polls = sorted(r[5] for r in rk)
    skips = sorted((r[7] if len(r) > 7 else 0) for r in rk)
    tnorm = sorted((r[8] / 1e3 if len(r) > 8 else 0) for r in rk)
    nnorm = sorted((r[9] if len(r) > 9 else 0) for r in rk)
    # lag between consecutive strips' body starts, in the sweep's strip order
    order = sorted(range(n), key=lambda i: st[i])
    lags = sorted(st[order[i + 1]] - st[order[i]] for i in range(n - 1))
    print(f"k={k:2d} starts {min(st):9.1f}..{max(st):9.1f} (fill {max(st) - min(st):7.1f} us, "
          f"lag med {lags[len(lags) // 2]:5.1f}) ends {min(en):9.1f}..{max(en):9.1f} | body med "
          f"{body[n // 2]:7.1f} | computed med {comp[n // 2]:5d} polls med {polls[n // 2]:5d} skipped super-blocks med {skips[n // 2]:4d} | computed runs: med {tnorm[n // 2]:7.1f} us over {nnorm[n // 2]:4d} blocks")
