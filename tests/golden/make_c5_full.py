"""Golden fixtures for BASELINE config 5 at FULL size (32769^2, 1.07e9 nodes).

TEST INFRASTRUCTURE ONLY (run here, where /root/reference and oracle/_ref
exist; the GPU box only reads the JSON this writes).

The UNMODIFIED reference solvers (oracle/_ref/libeikref.so, built by
oracle/Makefile from /root/reference/proj/src) run on config 5 with an
array-backed SpeedFn (oracle/ref_shim.cpp `ref_solve_array`; SURVEY.md 8(d),
BASELINE.md 3): on-node F comes from the sampled array, off-grid probes are
evaluated in closed form -- the same bits as the on-demand SpeedFn.
`--check` first proves that on config 5's 2049^2 member against c5.json
(generated with the on-demand SpeedFn).

Each method writes tests/golden/c5_full/<key>.json as soon as it finishes:
sha256 of the whole field, sha256 of every 1024-row block (so a mismatch can
be located), every counter, and the reference's own solve time.  `--merge`
collects them into tests/golden/c5_full.json.

    python tests/golden/make_c5_full.py --check
    python tests/golden/make_c5_full.py fsm            # ~1.5-3 h on one core
    python tests/golden/make_c5_full.py fhcm/32 fhcm/16 hcm/32 fmsm/32
    python tests/golden/make_c5_full.py --merge
"""
from __future__ import annotations

import argparse
import ctypes as C
import hashlib
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle import oracle as O  # noqa: E402
from paper_1110_6220_b200 import _native as N  # noqa: E402
from paper_1110_6220_b200 import configs  # noqa: E402

PARTS = os.path.join(HERE, "c5_full")
BLOCK_ROWS = 1024
_METHOD = {"fmm": 0, "fsm": 1, "lsm": 2, "hcm": 3, "fhcm": 4, "fmsm": 5}

_dp = C.POINTER(C.c_double)
_i64p = C.POINTER(C.c_int64)
lib = O.rlib
lib.ref_solve_array.argtypes = [C.c_int, C.POINTER(N.eik_grid), C.POINTER(N.eik_field), _dp,
                                _i64p, _dp, C.c_int64, C.c_int, C.c_int, C.POINTER(O.ref_stats)]
lib.ref_solve_array.restype = C.c_void_p
lib.ref_result_values.argtypes = [C.c_void_p]
lib.ref_result_values.restype = _dp
lib.ref_result_free.argtypes = [C.c_void_p]


def field_digest(u: np.ndarray, m: int) -> dict:
    """sha256 of the field (same bytes as tests' sha(u)) + per-block shas."""
    whole = hashlib.sha256()
    blocks = []
    rows = u.size // m
    for r0 in range(0, rows, BLOCK_ROWS):
        b = memoryview(u[r0 * m:min(rows, r0 + BLOCK_ROWS) * m])
        whole.update(b)
        blocks.append(hashlib.sha256(b).hexdigest())
    fin = np.isfinite(u)
    return dict(sha256=whole.hexdigest(), block_rows=BLOCK_ROWS, block_sha256=blocks,
                u_max=float(u[fin].max()), u_sum=float(u[fin].sum(dtype=np.float64)),
                n_inf=int(u.size - fin.sum()))


def run(p, key: str) -> dict:
    method, _, cs = key.partition("/")
    g = p.grid
    cx = g.m // int(cs) if cs else 0
    F = p.sampled_speed()
    en = np.ascontiguousarray(p.exit_nodes, dtype=np.int64)
    ec = np.ascontiguousarray(p.exit_cost, dtype=np.float64)
    st = O.ref_stats()
    cg = g.c()
    h = lib.ref_solve_array(_METHOD[method], C.byref(cg), C.byref(p.speed.cfield),
                            F.ctypes.data_as(_dp), en.ctypes.data_as(_i64p),
                            ec.ctypes.data_as(_dp), len(en), cx, cx, C.byref(st))
    if not h:
        raise RuntimeError(lib.ref_last_error().decode())
    try:
        ptr = lib.ref_result_values(h)
        u = np.ctypeslib.as_array(ptr, shape=(g.size(),))
        d = field_digest(u, g.m)
    finally:
        lib.ref_result_free(h)
    d.update(method=method, cells=cx, m=g.m, ms=st.elapsed_ms, sweeps=st.sweeps,
             node_updates=st.node_updates, heap_removals=st.heap_removals,
             cell_removals=st.cell_removals, cell_sweeps=st.cell_sweeps,
             mon_checks=st.mon_checks, mon_single=st.mon_single, avhr=st.avhr, avs=st.avs,
             mon_pct=st.mon_pct, speed_fn="array-backed (on-node F[j*m+i], closed form off-grid)")
    return d


def check() -> None:
    """The array-backed SpeedFn reproduces c5.json (on-demand SpeedFn) at 2049^2."""
    with open(os.path.join(HERE, "c5.json")) as f:
        want = json.load(f)
    p = configs.config5(2049).problem
    for key in ("fsm", "fhcm/32", "hcm/16", "fmsm/16"):
        d = run(p, key)
        w = want["c5_2049/" + key]
        ok = d["sha256"] == w["sha256"] and all(d[c] == w[c] for c in
                                                 ("sweeps", "node_updates", "heap_removals",
                                                  "mon_checks", "mon_single"))
        print(key, "OK" if ok else "MISMATCH", round(d["ms"]), "ms", flush=True)
        if not ok:
            sys.exit(1)


def merge() -> None:
    out = {}
    for fn in sorted(os.listdir(PARTS)):
        if fn.endswith(".json"):
            with open(os.path.join(PARTS, fn)) as f:
                d = json.load(f)
            out["c5_full/" + fn[:-5].replace("_", "/")] = d
    with open(os.path.join(HERE, "c5_full.json"), "w") as f:
        json.dump(out, f, indent=1, sort_keys=True)
    print(sorted(out))


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("keys", nargs="*", help="fsm, fhcm/32, hcm/16, fmsm/32, ...")
    ap.add_argument("--check", action="store_true")
    ap.add_argument("--merge", action="store_true")
    a = ap.parse_args()
    if a.check:
        check()
    if a.keys:
        os.makedirs(PARTS, exist_ok=True)
        t = time.time()
        p = configs.config5().problem
        p.sampled_speed()
        print("sampled F in", round(time.time() - t, 1), "s", flush=True)
        for key in a.keys:
            t = time.time()
            d = run(p, key)
            with open(os.path.join(PARTS, key.replace("/", "_") + ".json"), "w") as f:
                json.dump(d, f, indent=1, sort_keys=True)
            print(key, "done in", round(time.time() - t, 1), "s; sweeps", d["sweeps"],
                  "pops", d["heap_removals"], flush=True)
    if a.merge:
        merge()
