"""Generate the golden fixtures in tests/golden/ from the UNMODIFIED reference.

Run here (where /root/reference exists and oracle/_ref/libeikref.so is
built):  python tests/golden/make_golden.py [--big]

  kat.json      known-answer values of the reference's own unit tests
                (test_local_update.cpp:31-46,64-70,125-133; cells/metrics),
                recomputed by the reference functions, stored as float.hex.
  small.npz     full value fields of small problems for every method, plus
  small.json    their counters (sweeps, node_updates, heap pops, Mon checks).
  big.json      BASELINE configs: sha256 of the reference's u bytes and its
                counters (C1 257^2, C2 2049^2 all methods/cell sizes, and the
                acceptance sweep counts of acceptance.cpp:133-146).
  c34.json      (--c34) configs 3 and 4 at 4097^2.
  c5.json       (--c5) config 5's field family at 2049^2.
  metrics.*     (--metrics) metrics.cpp ground truth and reports, small cases.
"""
from __future__ import annotations

import argparse
import hashlib
import json
import math
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import paper_1110_6220_b200 as E  # noqa: E402
from paper_1110_6220_b200 import configs  # noqa: E402
from oracle import oracle as O  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
INF = math.inf


def sha(u: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(u, dtype=np.float64).tobytes()).hexdigest()


def counters(r) -> dict:
    return {"sweeps": r.sweeps, "node_updates": r.node_updates, "heap_removals": r.heap_removals,
            "mon_checks": r.mon_checks, "mon_single": r.mon_single}


def kat() -> dict:
    R = O.rlib
    q = R.ref_quadrant_update
    nbp = lambda v: (np.array(v, dtype=np.float64)).ctypes.data_as(O._dp)  # noqa: E731
    out = {"quadrant": [], "node": [], "directional": []}
    for a, b, f, h in [(0.0, 0.0, 1.0, 1.0), (0.0, INF, 2.0, 0.1), (0.0, 10.0, 1.0, 1.0),
                       (INF, INF, 1.0, 1.0), (1.0, 2.0, 1.0, 2.0)]:
        out["quadrant"].append([a, b, f, h, q(a, b, f, h).hex()])
    for nb, f, h in [([0.05, INF, INF, INF], 1.0, 0.1), ([0.0, 3.0, 0.0, 2.0], 1.0, 1.0),
                     ([INF, INF, INF, INF], 1.0, 1.0)]:
        out["node"].append([nb, f, h, R.ref_node_update(nbp(nb), f, h).hex()])
    for nb, d, f, h in [([0.0, -5.0, 0.0, -5.0], 2, 1.0, 1.0), ([INF, 0.0, INF, 0.0], 2, 1.0, 1.0),
                        ([0.0, INF, 10.0, INF], 2, 1.0, 1.0), ([1.0, 2.0, 3.0, 4.0], 0, 1.0, 1.0),
                        ([1.0, 2.0, 3.0, 4.0], 1, 1.0, 1.0), ([1.0, 2.0, 3.0, 4.0], 3, 1.0, 1.0)]:
        out["directional"].append([nb, d, f, h, R.ref_directional_update(nbp(nb), d, f, h).hex()])
    # 1e5 seeded random draws (test_local_update.cpp:72-85 style), hashed
    rng = np.random.default_rng(42)
    n = 100000
    vals = np.where(rng.random((n, 4)) < 0.15, INF, 10.0 * rng.random((n, 4)) - 2.0)
    fs = 0.05 + 3.0 * rng.random(n)
    hs = 0.01 + rng.random(n)
    res = np.array([R.ref_node_update(nbp(vals[k]), fs[k], hs[k]) for k in range(n)])
    out["random_node_update"] = {"seed": 42, "n": n, "sha256": sha(res)}
    return out


SMALL_CASES = [
    # (case id, problem factory, cell counts)
    ("sinB45", lambda: E.build_problem(E.Grid.unit_square(45), E.speed_sinusoid(0.99, 2),
                                       E.ExitSpec.point_source((0.5, 0.5))), [4, 7]),
    ("comb4_44", lambda: E.build_problem(E.Grid.unit_square(44), E.speed_comb_maze(4),
                                         E.ExitSpec.point_source((0.0, 0.0))), [4, 11]),
    ("chk11_33_boundary", lambda: E.build_problem(E.Grid.unit_square(33), E.speed_checkerboard(11),
                                                  E.ExitSpec.full_boundary()), [4]),
    ("c2_65", lambda: configs.config2(65).problem, [4, 8]),
]


def small():
    arrays, meta = {}, {}
    for cid, make, cells in SMALL_CASES:
        p = make()
        for method in ("fmm", "fsm", "lsm"):
            r = O.ref_solve(p, method)
            arrays[f"{cid}/{method}"] = r.u
            meta[f"{cid}/{method}"] = counters(r)
        for c in cells:
            for method in ("hcm", "fhcm", "fmsm"):
                r = O.ref_solve(p, method, c, c)
                arrays[f"{cid}/{method}/{c}"] = r.u
                meta[f"{cid}/{method}/{c}"] = counters(r)
    np.savez_compressed(os.path.join(HERE, "small.npz"), **arrays)
    with open(os.path.join(HERE, "small.json"), "w") as f:
        json.dump(meta, f, indent=1, sort_keys=True)


def big():
    out = {}
    c1 = configs.config1()
    p = c1.problem
    g = p.grid
    xs = g.x0 + np.arange(g.m) * g.h
    X, Y = np.meshgrid(xs, xs)
    exact = np.hypot(X, Y).reshape(-1)
    for method, cs in [("fmm", 0), ("fsm", 0), ("fmsm", 16)]:
        cx = g.m // cs if cs else 0
        r = O.ref_solve(p, method, cx, cx)
        err = np.abs(r.u - exact)
        out[f"c1/{method}" + (f"/{cs}" if cs else "")] = dict(
            sha256=sha(r.u), linf_vs_abs=float(err.max()), l1_vs_abs=float(err.mean()),
            ms=r.elapsed_ms, **counters(r))
    c2 = configs.config2()
    p = c2.problem
    for method in ("fsm", "fmm"):
        t = time.time()
        r = O.ref_solve(p, method)
        out[f"c2/{method}"] = dict(sha256=sha(r.u), ms=r.elapsed_ms, **counters(r))
        print(method, time.time() - t, flush=True)
    for cs in (8, 16, 32, 64):
        cx = p.grid.m // cs
        for method in ("fmsm", "hcm", "fhcm"):
            r = O.ref_solve(p, method, cx, cx)
            out[f"c2/{method}/{cs}"] = dict(sha256=sha(r.u), cells=cx, ms=r.elapsed_ms, **counters(r))
            print(method, cs, r.elapsed_ms, flush=True)
    # acceptance.cpp:133-146 published FSM sweep counts
    acc = {}
    for name, m, expect in [("constant", 1408, 5), ("constant", 176, 5), ("checker11", 176, 16),
                            ("checker41", 164, 44)]:
        sp = {"constant": E.speed_constant(), "checker11": E.speed_checkerboard(11),
              "checker41": E.speed_checkerboard(41)}[name]
        pr = E.build_problem(E.Grid.unit_square(m), sp, E.ExitSpec.point_source((0.5, 0.5)))
        r = O.ref_solve(pr, "fsm")
        acc[f"{name}/{m}"] = {"sweeps": r.sweeps, "published": expect, "sha256": sha(r.u)}
    out["acceptance_fsm_sweeps"] = acc
    with open(os.path.join(HERE, "big.json"), "w") as f:
        json.dump(out, f, indent=1, sort_keys=True)


C34_CELLS = {"c3": [16, 32, 64, 24, 48], "c4": [16, 32]}


def c34():
    """BASELINE configs 3 (4097^2 8x8 checkerboard; cell sizes aligned with
    the 512-node blocks and misaligned) and 4 (4097^2 seeded maze, corner
    source): sha256 + counters of the reference for every method."""
    out = {}
    for name, make in (("c3", configs.config3), ("c4", configs.config4)):
        p = make().problem
        for method in ("fsm", "fmm"):
            t = time.time()
            r = O.ref_solve(p, method)
            out[f"{name}/{method}"] = dict(sha256=sha(r.u), ms=r.elapsed_ms, **counters(r))
            print(name, method, round(time.time() - t, 1), flush=True)
        for cs in C34_CELLS[name]:
            cx = p.grid.m // cs
            for method in ("fmsm", "hcm", "fhcm"):
                r = O.ref_solve(p, method, cx, cx)
                out[f"{name}/{method}/{cs}"] = dict(sha256=sha(r.u), cells=cx, ms=r.elapsed_ms,
                                                    **counters(r))
                print(name, method, cs, round(r.elapsed_ms), flush=True)
    with open(os.path.join(HERE, "c34.json"), "w") as f:
        json.dump(out, f, indent=1, sort_keys=True)


def extra():
    """Round-2 fixtures (extra.json):
    * lsm: the reference's lsm_solve on C1, C2, C3, C4 and config 5's 2049^2
      member -- sha256 + counters (its field and sweeps are fsm_solve's; only
      node_updates differs);
    * fmm_vs_fsm: L-inf between the reference's FMM and FSM fields on C2, C3,
      C4 -- the GPU FMM row is bitwise the reference FSM (pinned by sha256),
      so this is exactly its distance to the reference FMM;
    * c3r: BASELINE config 3's seeded random-block variant (block speeds iid
      from {0.5, 1, 2}, seed 7), every method and cell size as c34.json."""
    out = {"lsm": {}, "fmm_vs_fsm": {}}
    cases = [("c1", configs.config1()), ("c2", configs.config2()), ("c3", configs.config3()),
             ("c4", configs.config4()), ("c5_2049", configs.config5(2049))]
    for name, cfg in cases:
        p = cfg.problem
        t = time.time()
        r = O.ref_solve(p, "lsm")
        out["lsm"][name] = dict(sha256=sha(r.u), ms=r.elapsed_ms, **counters(r))
        print(name, "lsm", round(time.time() - t, 1), flush=True)
        if name in ("c2", "c3", "c4"):
            a = O.ref_solve(p, "fmm")
            b = O.ref_solve(p, "fsm")
            out["fmm_vs_fsm"][name] = dict(linf=float(np.max(np.abs(a.u - b.u))),
                                           fmm_sha256=sha(a.u), fsm_sha256=sha(b.u),
                                           fmm=counters(a))
            print(name, "fmm vs fsm", out["fmm_vs_fsm"][name]["linf"], flush=True)
    p = configs.config3(seed=7).problem
    c3r = {}
    for method in ("fsm", "fmm"):
        r = O.ref_solve(p, method)
        c3r[method] = dict(sha256=sha(r.u), ms=r.elapsed_ms, **counters(r))
    for cs in C34_CELLS["c3"]:
        cx = p.grid.m // cs
        for method in ("fmsm", "hcm", "fhcm"):
            r = O.ref_solve(p, method, cx, cx)
            c3r[f"{method}/{cs}"] = dict(sha256=sha(r.u), cells=cx, ms=r.elapsed_ms,
                                         **counters(r))
            print("c3r", method, cs, round(r.elapsed_ms), flush=True)
    out["c3r"] = c3r
    with open(os.path.join(HERE, "extra.json"), "w") as f:
        json.dump(out, f, indent=1, sort_keys=True)


def metrics():
    """metrics.cpp on the small cases: the reference's refine-4 ground truth
    (metrics.npz, its FMM on the refined grid, subsampled) and its
    method_metrics report for every method against it (metrics.json), with
    u_method / u_exact taken from small.npz (the reference's own fields)."""
    fields = np.load(os.path.join(HERE, "small.npz"))
    arrays, meta = {}, {}
    for cid, make, cells in SMALL_CASES:
        p = make()
        fine = E.refined_problem(p, 4)
        rt = O.ref_solve(fine, "fmm").u.reshape(fine.grid.n, fine.grid.m)[::4, ::4]
        arrays[f"{cid}/truth4"] = np.ascontiguousarray(rt).reshape(-1)
        exact = fields[f"{cid}/fmm"]
        keys = [f"{cid}/fsm"] + [f"{cid}/{meth}/{c}" for c in cells for meth in ("hcm", "fhcm", "fmsm")]
        for k in keys:
            r = O.ref_metrics(p, fields[k], exact, 4)
            meta[k] = {"l_inf": r[0], "l_1": r[1], "max_error_ratio": r[2],
                       "avg_error_ratio": r[3], "ratio_of_max": r[4], "m_plus": int(r[5]),
                       "x_plus_empty": bool(r[6])}
    np.savez_compressed(os.path.join(HERE, "metrics.npz"), **arrays)
    with open(os.path.join(HERE, "metrics.json"), "w") as f:
        json.dump(meta, f, indent=1, sort_keys=True)


def c5():
    """BASELINE config 5's field family (16 random-phase sinusoids, 64 random
    node sources) at 2049^2, where the reference runs here: sha256 + counters
    of FSM and FHCM at 16/32-node cells (c5.json)."""
    out = {}
    p = configs.config5(2049).problem
    t = time.time()
    r = O.ref_solve(p, "fsm")
    out["c5_2049/fsm"] = dict(sha256=sha(r.u), ms=r.elapsed_ms, **counters(r))
    print("fsm", round(time.time() - t, 1), flush=True)
    for cs in (16, 32):
        cx = p.grid.m // cs
        for method in ("fhcm", "hcm", "fmsm"):
            r = O.ref_solve(p, method, cx, cx)
            out[f"c5_2049/{method}/{cs}"] = dict(sha256=sha(r.u), cells=cx, ms=r.elapsed_ms,
                                                 **counters(r))
            print(method, cs, round(r.elapsed_ms), flush=True)
    with open(os.path.join(HERE, "c5.json"), "w") as f:
        json.dump(out, f, indent=1, sort_keys=True)


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--big", action="store_true")
    ap.add_argument("--c34", action="store_true")
    ap.add_argument("--c5", action="store_true")
    ap.add_argument("--metrics", action="store_true")
    ap.add_argument("--extra", action="store_true")
    a = ap.parse_args()
    if not O.have_ref():
        sys.exit("oracle/_ref/libeikref.so missing: run make -C oracle here")
    if a.c34:
        c34()
        sys.exit(0)
    if a.c5:
        c5()
        sys.exit(0)
    if a.metrics:
        metrics()
        sys.exit(0)
    if a.extra:
        extra()
        sys.exit(0)
    with open(os.path.join(HERE, "kat.json"), "w") as f:
        json.dump(kat(), f, indent=1)
    small()
    if a.big:
        big()
