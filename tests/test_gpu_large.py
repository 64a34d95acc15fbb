"""Full-size BASELINE configurations against reference-generated goldens.

tests/golden/large_*.json come from the UNMODIFIED reference solver
(tests/golden/gen_golden_large.py through oracle/_ref): the sha256 of the
whole reference table (opt int64 | DpArg kind | value, every cell), per
diagonal digests (to name the first differing diagonal), the top row, and
build_schedule_rec / solve_chain results.  The device tables come through the
C ABI (rkr_table_download), so every cell is compared bit-exactly:

  config 3   96/32/16384 (bench.py's chain): every fill kernel, both widths,
             the fused fill + walk, schedules and their replayed peaks
  config 4   all 1024 sweep instances (4 chains x 256 budgets, units=500)
             through rkr_sweep_chains and rkr_sweep
  config 5   the twin 256/64/4096 (bench.py's N=1 sharded chain) as one table
             and as 1/2/4 budget shards; the chain length L=1024 (B=64) at M=64
"""
import json
import os

import numpy as np
import pytest

from helpers import ops_digest, table_digest, tri_row
from paper_2307_01236_b200 import rotor
from paper_2307_01236_b200.menu import synthetic_menu

pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _load(name):
    with open(os.path.join(GOLDEN, f"large_{name}.json")) as f:
        return json.load(f)


@pytest.fixture(scope="module", autouse=True)
def _device():
    assert rotor.lib().rkr_device_ok(0) == 1, "no sm_100 device visible"


def diag_digests(o, k, v, L):
    out = []
    for d in range(L):
        idx = np.array([tri_row(L, s, s + d) for s in range(L - d)], np.int64)
        out.append(table_digest(o[idx], k[idx], v[idx])[:16])
    return out


def check_table(o, k, v, g):
    """Whole-table digest against the reference; on a mismatch name the first
    differing diagonal (and the top row) instead of just failing."""
    L = g["L"]
    if table_digest(o, k, v) == g["digest"]:
        return
    dd = diag_digests(o, k, v, L)
    bad = [d for d in range(L) if dd[d] != g["diag_digests"][d]]
    r = tri_row(L, 0, L - 1)
    top_ok = o[r].tolist() == g["top"] and k[r].tolist() == g["top_kind"]
    pytest.fail(f"table differs from the reference: diagonals {bad[:8]} (of {len(bad)}), "
                f"top row {'equal' if top_ok else 'differs'}")


def check_walks(t, menu, g, orc):
    L = g["L"]
    for w in g["walks"]:
        s, tt, m = w["s"], w["t"], w["m"]
        if w["status"] == 0:
            ops = t.backtrack(s, tt, m)
            assert (len(ops), ops_digest(ops)) == (w["n_ops"], w["ops_digest"]), (s, tt, m)
            assert t.opt(s, tt, m) == w["opt"]
            if w["replay_peak"] is not None:  # simulated peak must be exact
                assert orc.atomic_replay(menu, ops) == (w["replay_peak"], w["replay_time"])
                assert w["replay_time"] == w["opt"]
        else:
            with pytest.raises(rotor.InfeasibleBudget):
                t.backtrack(s, tt, m)
    if g["first_feasible"] >= 0:
        assert t.first_feasible(0, L - 1) == g["first_feasible"]


# ---------------------------------------------------------------------------
# config 3: 96 blocks x 32 options x 16384 budget slots
# ---------------------------------------------------------------------------
@pytest.fixture(scope="module")
def cfg3():
    return _load("cfg3")


@pytest.mark.parametrize("kernel,width", [("persistent", "auto"), ("queue", "auto"),
                                          ("queue", "64"), ("diagonal", "auto")])
def test_config3_full_table_vs_reference(cfg3, orc, kernel, width):
    g = cfg3
    L, M = g["L"], g["M"]
    menu = synthetic_menu(L, g["B"], M, g["seed"])
    with rotor.DpTable(menu, 1, M, width=width, kernel=kernel) as t:
        if kernel == "persistent":
            assert t.kernel() == "tiles"
        assert t.max_candidates_per_cell == g["max_cands"]
        o, k, v = t.download()
        check_table(o, k, v, g)
        del o, k, v
        t._host = None
        check_walks(t, menu, g, orc)


def test_config3_fused_fill_walk_vs_reference(cfg3):
    """bench.py's step (refill + walk from the top cell, one launch) repeated:
    the schedule and the table stay the reference's."""
    g = cfg3
    L, M = g["L"], g["M"]
    menu = synthetic_menu(L, g["B"], M, g["seed"])
    top = [w for w in g["walks"] if (w["s"], w["t"], w["m"]) == (0, L - 1, M)][0]
    with rotor.DpTable(menu, 1, M) as t:
        for _ in range(3):
            t.refill_walk(0, L - 1, M)
            ops = t.backtrack_fetch()
            assert ops_digest(ops) == top["ops_digest"]
        check_table(*t.download(), g)


def test_config3_solve_chain_vs_reference(cfg3):
    """rkr_solve_chain as bench.py's e2e leg calls it (budget = M + a_0 bytes,
    units = budget: unit 1, m_top = M)."""
    g = cfg3
    L, M = g["L"], g["M"]
    menu = synthetic_menu(L, g["B"], M, g["seed"])
    top = [w for w in g["walks"] if (w["s"], w["t"], w["m"]) == (0, L - 1, M)][0]
    budget = M + int(menu.act_sizes[0])
    sol = rotor.solve_chain(rotor.Chain.skeleton(L), menu, budget, budget)
    assert (sol.opt_time, sol.unit, sol.m_top) == (top["opt"], 1, M)
    assert ops_digest(sol.raw_ops) == top["ops_digest"]


# ---------------------------------------------------------------------------
# config 4: 4 chains x 256 budgets
# ---------------------------------------------------------------------------
def _check_sweep_rows(rows, inst, menus, orc):
    for r, e in zip(rows, inst):
        assert r.budget == e["budget"]
        if e["status"] == 0:
            assert r.feasible, e
            assert (r.opt_time, r.unit, r.m_top) == (e["opt_time"], e["unit"], e["m_top"]), e
            assert (len(r.ops), ops_digest(r.ops)) == (e["n_ops"], e["ops_digest"]), e
            assert orc.atomic_replay(menus[e["chain"]], r.ops) == (e["replay_peak"], e["replay_time"])
        else:
            assert not r.feasible and r.min_feasible == e["min_feasible"], e


def test_config4_sweep_chains_vs_reference(orc):
    from paper_2307_01236_b200.sweep import sweep_workload

    g = _load("cfg4")
    menus, inst = sweep_workload()
    assert [(x.chain, x.budget) for x in inst] == [(e["chain"], e["budget"]) for e in g["instances"]]
    per_chain = [[e for e in g["instances"] if e["chain"] == c] for c in range(len(menus))]
    # the workload exercises the min-feasible search (infeasible low budgets)
    assert sum(e["status"] == 2 for e in g["instances"]) > 0
    out = rotor.sweep_chains_raw(menus, [[e["budget"] for e in pc] for pc in per_chain], g["units"])
    for c in range(len(menus)):
        _check_sweep_rows(out[c], per_chain[c], menus, orc)


@pytest.mark.parametrize("chain", [0, 3])
def test_config4_sweep_per_chain_vs_reference(orc, chain):
    from paper_2307_01236_b200.sweep import sweep_workload

    g = _load("cfg4")
    menus, _ = sweep_workload()
    pc = [e for e in g["instances"] if e["chain"] == chain]
    rows = rotor.sweep_raw(menus[chain], [e["budget"] for e in pc], g["units"])
    _check_sweep_rows(rows, pc, menus, orc)


# ---------------------------------------------------------------------------
# config 5: the 256/64/4096 twin (single table and budget shards) and L = 1024
# ---------------------------------------------------------------------------
@pytest.fixture(scope="module")
def cfg5twin():
    return _load("cfg5twin")


def test_config5_twin_single_table_vs_reference(cfg5twin, orc):
    g = cfg5twin
    menu = synthetic_menu(g["L"], g["B"], g["M"], g["seed"])
    with rotor.DpTable(menu, 1, g["M"]) as t:
        check_table(*t.download(), g)
        t._host = None
        check_walks(t, menu, g, orc)


@pytest.mark.parametrize("n", [1, 2, 4])
def test_config5_twin_budget_shards_vs_reference(cfg5twin, n):
    g = cfg5twin
    L, M = g["L"], g["M"]
    menu = synthetic_menu(L, g["B"], M, g["seed"])
    with rotor.ShardedTable(menu, 1, M, n) as sh:
        check_table(*sh.download(), g)
        for w in g["walks"]:
            if w["s"] == 0 and w["t"] == L - 1 and w["status"] == 0:
                ops = sh.backtrack(0, L - 1, w["m"])
                assert ops_digest(ops) == w["ops_digest"]


@pytest.mark.parametrize("kernel", ["persistent", "queue"])
def test_chain_length_1024_vs_reference(orc, kernel):
    g = _load("l1024")
    menu = synthetic_menu(g["L"], g["B"], g["M"], g["seed"])
    with rotor.DpTable(menu, 1, g["M"], kernel=kernel) as t:
        check_table(*t.download(), g)
        t._host = None
        check_walks(t, menu, g, orc)


@pytest.mark.parametrize("kernel", ["persistent", "queue"])
def test_chain_length_1024_m256_vs_reference(orc, kernel):
    """The config-5 chain length (L=1024, B=64) at M=256 against the unmodified
    reference (20 min of its CPU; tests/golden/gen_golden_large.py l1024m256):
    whole table by diagonal digests, top row, walks and replayed peaks, on the
    budget-tile kernel (streamed programs) and on the row-segment queue -- the
    kernel a config-5 shard too large for 32-bit tile offsets runs."""
    g = _load("l1024m256")
    menu = synthetic_menu(g["L"], g["B"], g["M"], g["seed"])
    with rotor.DpTable(menu, 1, g["M"], kernel=kernel) as t:
        check_table(*t.download(), g)
        t._host = None
        check_walks(t, menu, g, orc)


@pytest.mark.parametrize("n", [2, 4])
def test_chain_length_1024_m256_budget_shards_vs_reference(n):
    """L=1024 split along the budget axis into n shards (halo pushed in the
    fill kernel): every shard's columns and the cross-shard walk against the
    reference."""
    g = _load("l1024m256")
    L, M = g["L"], g["M"]
    menu = synthetic_menu(L, g["B"], M, g["seed"])
    with rotor.ShardedTable(menu, 1, M, n) as sh:
        check_table(*sh.download(), g)
        for w in g["walks"]:
            if w["s"] == 0 and w["t"] == L - 1 and w["status"] == 0:
                assert ops_digest(sh.backtrack(0, L - 1, w["m"])) == w["ops_digest"]
