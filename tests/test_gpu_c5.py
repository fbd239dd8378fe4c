"""BASELINE config 5: the 16-term random sinusoid speed with 64 random node
sources.

* At 2049^2, where the unmodified reference runs in this container, FSM and
  HCM/FHCM/FMSM at 16/32-node cells reproduce its field bit for bit with
  identical counters (tests/golden/c5.json, make_golden.py --c5).
* At the full 32769^2 (1.07e9 points) against the reference's own run of the
  same problem (tests/golden/c5_full.json, make_c5_full.py): FSM, HCM, FHCM
  and FMSM at 16/32-node cells bit for bit with identical counters.
"""
import hashlib
import json
import os

import numpy as np
import pytest

import paper_1110_6220_b200 as E
from paper_1110_6220_b200 import configs

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden", "c5.json")


def sha(u):
    return hashlib.sha256(np.ascontiguousarray(u, dtype=np.float64).tobytes()).hexdigest()


_P = {}


def _problem(m):
    if m not in _P:
        _P[m] = configs.config5(m).problem
    return _P[m]


CASES = [("fsm", 0)] + [(meth, cs) for cs in (16, 32) for meth in ("fmsm", "hcm", "fhcm")]


@pytest.mark.parametrize("method,cs", CASES, ids=[f"{a}-{b}" for a, b in CASES])
def test_c5_family_bitwise_2049(method, cs):
    with open(GOLD) as f:
        want = json.load(f)["c5_2049/" + method + (f"/{cs}" if cs else "")]
    p = _problem(2049)
    cells = E.build_cells(p.grid, want["cells"], want["cells"]) if cs else None
    out = E.solve(p, "hcm_exact" if method == "hcm" else method, cells)
    assert sha(out.values) == want["sha256"]
    assert (out.sweeps, out.node_updates, out.heap_removals, out.hybrid.mon_checks,
            out.hybrid.mon_single) == (want["sweeps"], want["node_updates"],
                                       want["heap_removals"], want["mon_checks"],
                                       want["mon_single"])


FULL = os.path.join(os.path.dirname(__file__), "golden", "c5_full.json")


def _full_keys():
    if not os.path.exists(FULL):
        return []
    with open(FULL) as f:
        return sorted(json.load(f))


_FULL = {}


def _c5_full():
    if "cfg" not in _FULL:
        _FULL["cfg"] = configs.config5()
        _FULL["u"] = np.empty(_FULL["cfg"].problem.grid.size())
    return _FULL["cfg"], _FULL["u"]


@pytest.mark.slow
@pytest.mark.parametrize("key", _full_keys())
def test_c5_full_size_bitwise_against_reference(key):
    """Config 5 at its full 32769^2 (1.07e9 nodes): the unmodified reference
    solved it on the CPU (array-backed SpeedFn, tests/golden/make_c5_full.py;
    FSM ~1-2 h, the cell methods minutes) and its field hash, per-1024-row
    block hashes and counters are in c5_full.json.  The device must reproduce
    them bit for bit."""
    with open(FULL) as f:
        want = json.load(f)[key]
    cfg, u = _c5_full()
    p = cfg.problem
    method = want["method"]
    cells = E.build_cells(p.grid, want["cells"], want["cells"]) if want["cells"] else None
    plan = E.Plan(p, "hcm_exact" if method == "hcm" else method, cells)
    try:
        out = plan.run(u)
    finally:
        plan.close()
    got = (out.sweeps, out.node_updates, out.heap_removals, out.hybrid.mon_checks,
           out.hybrid.mon_single)
    ref = (want["sweeps"], want["node_updates"], want["heap_removals"], want["mon_checks"],
           want["mon_single"])
    m, br = p.grid.m, want["block_rows"]
    if sha(u) != want["sha256"]:
        bad = [b for b, h in enumerate(want["block_sha256"])
               if hashlib.sha256(memoryview(u[b * br * m:min(m, (b + 1) * br) * m])).hexdigest() != h]
        raise AssertionError(f"{key}: field differs in row blocks {bad[:20]} ({len(bad)} of "
                             f"{len(want['block_sha256'])}); counters {got} vs {ref}")
    assert got == ref, key
