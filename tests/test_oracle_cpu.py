"""Pin the CPU oracle (oracle/rotor_oracle.c) to the reference's golden vectors.

The fixtures under tests/golden were produced by the unmodified reference
(tests/golden/gen_golden.py via oracle/_ref).  These tests run without a GPU.
"""
import numpy as np
import pytest

from helpers import ops_digest, table_digest, tri_row
from paper_2307_01236_b200.menu import Menu, synthetic_menu, tiny_chain_menu

INF = (2**63 - 1) // 4


def test_quantize_kats(orc, kat):
    # test_chain_dp.cpp:9-19 plus extra edge cases, as the reference answered them
    for b, u, st, unit, bu in kat["quantize"]:
        rst, runit, rbu = orc.quantize(b, u)
        assert rst == st
        if st == 0:
            assert (runit, rbu) == (unit, bu)


def test_tiny_chain_table(orc, kat):
    t = kat["tiny"]
    st, o, k, v, mc, wa = orc.fill(tiny_chain_menu(), 1, t["M"])
    assert st == 0
    assert o.tolist() == t["opt"] and k.tolist() == t["kind"] and v.tolist() == t["value"]
    assert (mc, wa) == (t["max_cands"], t["worst_allow"])
    # the literal values of test_chain_dp.cpp:41-54, 101-107
    r = tri_row(2, 0, 1)
    assert [o[r, m] for m in (64, 12, 11, 10)] == [39, 39, 49, 49]
    assert o[r, 9] >= INF
    assert (k[r, 10], v[r, 10]) == (2, 1)
    assert o[tri_row(2, 0, 0), 5] >= INF


def test_tiny_chain_schedules(orc, kat):
    menu = tiny_chain_menu()
    for M in (12, 10, 9):
        exp = kat["tiny"][f"schedule_M{M}"]
        st, o, k, v, _, _ = orc.fill(menu, 1, M)
        bst, ops = orc.build_schedule(menu, 1, M, (o, k, v), 0, 1, M)
        assert bst == exp["status"]
        assert [list(x) for x in ops] == exp["ops"]
    # test_chain_dp.cpp:68-75
    st, o, k, v, _, _ = orc.fill(menu, 1, 12)
    _, ops = orc.build_schedule(menu, 1, 12, (o, k, v), 0, 1, 12)
    assert ops == [(2, 0, 1), (2, 1, 1), (0, 1, -1), (3, 1, 1), (3, 0, 1)]


def test_solve_chain_kats(orc, kat):
    menu = tiny_chain_menu()
    for e in kat["solve"]:
        st, ops, ot, un, mt, mf = orc.solve_chain(menu, e["budget"], e["units"])
        assert st == e["status"], e
        assert mf == e["min_feasible"]
        if st == 0:
            assert (ot, un, mt) == (e["opt_time"], e["unit"], e["m_top"])
            assert [list(x) for x in ops] == e["ops"]
    # test_chain_dp.cpp:211-220
    assert orc.solve_chain(menu, 16, 16)[2] == 39
    assert orc.solve_chain(menu, 14, 14)[2] == 49
    assert orc.solve_chain(menu, 12, 12)[5] == 14


@pytest.mark.parametrize("suite", ["monotone", "ample", "symmetry", "enumeration", "work_bound",
                                   "relaxed"])
def test_random_menu_tables(orc, random_suites, suite):
    S = random_suites[suite]
    for e in S["menus"]:
        menu = Menu.from_json(e["menu"])
        st, o, k, v, mc, wa = orc.fill(menu, 1, S["M"])
        assert st == 0
        if "opt" in e:
            assert o.tolist() == e["opt"]
            assert k.tolist() == e["kind"]
            assert v.tolist() == e["value"]
        else:
            assert table_digest(o, k, v) == e["digest"]
        assert (mc, wa) == (e["max_cands"], e["worst_allow"])
        assert wa <= 0  # test_chain_dp.cpp:194-201


def test_enumeration_oracle_agreement(orc, random_suites):
    # test_chain_dp.cpp:156-174: DP == exhaustive enumeration (reference values)
    S = random_suites["enumeration"]
    for e in S["menus"]:
        menu = Menu.from_json(e["menu"])
        _, o, _, _, _, _ = orc.fill(menu, 1, 20)
        top = o[tri_row(menu.L, 0, menu.L - 1)]
        for i, m in enumerate(range(0, 21, 2)):
            ref = e["chain_oracle"][i]
            if top[m] >= INF:
                assert ref >= INF
            else:
                assert top[m] == ref


def test_relaxed_lower_bound(orc, random_suites):
    # test_chain_dp.cpp:176-192
    S = random_suites["relaxed"]
    for e in S["menus"]:
        menu = Menu.from_json(e["menu"])
        _, o, _, _, _, _ = orc.fill(menu, 1, 16)
        top = o[tri_row(menu.L, 0, menu.L - 1)]
        for i, m in enumerate(range(0, 17, 4)):
            if top[m] < INF:
                assert e["dijkstra"][i] <= top[m]


def test_synthetic_tables(orc, synthetic):
    for e in synthetic["tables"]:
        menu = synthetic_menu(e["L"], e["B"], e["M"], e["seed"], tie_stress=e["tie_stress"])
        st, o, k, v, mc, _ = orc.fill(menu, 1, e["M"])
        assert st == 0
        assert table_digest(o, k, v) == e["digest"], e["L"]
        assert mc == e["max_cands"]


def test_synthetic_solves_and_replay(orc, synthetic):
    for e in synthetic["solves"]:
        menu = synthetic_menu(e["L"], e["B"], e["M"], e["seed"], byte_scale=e["byte_scale"])
        st, ops, ot, un, mt, mf = orc.solve_chain(menu, e["budget"], e["units"])
        assert st == e["status"]
        assert mf == e["min_feasible"]
        if st == 0:
            assert (ot, un, mt) == (e["opt_time"], e["unit"], e["m_top"])
            assert ops_digest(ops) == e["ops_digest"]
            peak, tm = orc.atomic_replay(menu, ops)
            assert (peak, tm) == (e["replay_peak"], e["replay_time"])
            assert tm == ot  # reconstruction exactness (SPEC invariant)
            assert peak <= e["budget"]


def test_oracle_against_reference_directly(orc):
    """Where oracle/_ref is built, cross-check on fresh random draws too."""
    from oracle.pyoracle import HAVE_REF, Ref

    if not HAVE_REF:
        pytest.skip("oracle/_ref not built")
    ref = Ref()
    for menu in ref.random_menus(1234, 30, 5, 4):
        a = orc.fill(menu, 1, 40)
        b = ref.fill(menu, 1, 40)
        for x, y in zip(a[1:4], b[1:4]):
            np.testing.assert_array_equal(x, y)
    m = synthetic_menu(20, 6, 300, 99, tie_stress=True)
    a, b = orc.fill(m, 1, 300), ref.fill(m, 1, 300)
    for x, y in zip(a[1:4], b[1:4]):
        np.testing.assert_array_equal(x, y)


def test_oracle_matches_large_config4_goldens(orc):
    """The C restatement reproduces the reference's config-4 solve_chain results
    (tests/golden/large_cfg4.json) on a spread of the cheaper chains' budgets."""
    import json
    import os

    from helpers import ops_digest
    from paper_2307_01236_b200.sweep import sweep_workload

    g = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "large_cfg4.json")))
    menus, inst = sweep_workload()
    assert [(x.chain, x.budget) for x in inst] == [(e["chain"], e["budget"]) for e in g["instances"]]
    picks = [e for e in g["instances"] if e["chain"] < 2][::12]
    picks += [e for e in g["instances"] if e["status"] == 2][:6]
    for e in picks:
        st, ops, ot, un, mt, mf = orc.solve_chain(menus[e["chain"]], e["budget"], g["units"])
        assert st == e["status"]
        if st == 0:
            assert (ot, un, mt, ops_digest(ops)) == (e["opt_time"], e["unit"], e["m_top"],
                                                     e["ops_digest"])
        else:
            assert mf == e["min_feasible"]
