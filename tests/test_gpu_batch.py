"""Batched device solves (rkr_batch_*, rkr_sweep): every table of a batch and
every budget of a sweep bit-exact against the CPU oracle."""
import numpy as np
import pytest

from paper_2307_01236_b200 import rotor
from paper_2307_01236_b200.menu import BlockOption, Menu, synthetic_menu, tiny_chain_menu

pytestmark = pytest.mark.gpu


def _same(a, b):
    for x, y in zip(a, b):
        np.testing.assert_array_equal(x, y)


def _mixed_menus(random_suites):
    ms = [(tiny_chain_menu(), 1, 64)]
    for e in random_suites["enumeration"]["menus"][:12]:
        ms.append((Menu.from_json(e["menu"]), 1, 20))
    ms += [
        (synthetic_menu(17, 5, 300, 12), 1, 300),
        (synthetic_menu(40, 12, 700, 13, tie_stress=True), 1, 700),
        (synthetic_menu(24, 8, 500, 41, byte_scale=1024), 997, 480),
        (synthetic_menu(3, 2, 40, 5), 1, 0),
    ]
    return ms


@pytest.mark.parametrize("kernel", ["persistent", "queue"])
def test_batch_tables_match_oracle(orc, random_suites, kernel):
    items = _mixed_menus(random_suites)
    with rotor.Batch([m for m, _, _ in items], [u for _, u, _ in items],
                     [M for _, _, M in items], kernel=kernel) as b:
        assert len(b) == len(items)
        assert b.table(0).kernel() == ("tiles" if kernel == "persistent" else "queue")
        for rep in range(2):
            if rep:
                b.refill()
            for i, (m, u, M) in enumerate(items):
                st, *ref = orc.fill(m, u, M)
                assert st == 0
                t = b.table(i)
                _same(t.download(), ref[:3])
                top = ref[0][m.L - 1]  # row (0, L-1) in the s-major order
                fin = np.nonzero(top < rotor.K_INF_TIME)[0]
                if len(fin):
                    mm = int(fin[0])
                    _, ops = orc.build_schedule(m, u, M, tuple(ref[:3]), 0, m.L - 1, mm)
                    assert t.backtrack(0, m.L - 1, mm) == ops


def test_batch_falls_back_to_64bit_width(orc):
    big = 10**15
    wide = Menu.from_options([
        [BlockOption(0, big, None, 2, 5, 5, 0), BlockOption(1, big, big, 6, 7, 6, 8)],
        [BlockOption(0, big, None, 2, 5, 5, 0), BlockOption(1, big + 1, big, 5, 6, 6, 7)],
    ], [2, 2, 2])
    items = [(synthetic_menu(9, 3, 90, 3), 1, 90), (wide, 1, 30)]
    with rotor.Batch([m for m, _, _ in items], [1, 1], [90, 30]) as b:
        for i, (m, u, M) in enumerate(items):
            t = b.table(i)
            assert t.width() == 64
            _same(t.download(), orc.fill(m, u, M)[1:4])


def test_sweep_matches_solve_chain_per_budget(orc):
    menu = synthetic_menu(24, 8, 500, 41, byte_scale=1024)
    budgets = [1000, 20000, 70000, 71000, 80000, 90000, 120000, 200000, 512000, 2000000, 5]
    rows = rotor.sweep_raw(menu, budgets, 500)
    for r in rows:
        st, ops, ot, un, mt, mf = orc.solve_chain(menu, r.budget, 500)
        if st == 0:
            assert r.feasible
            assert (r.opt_time, r.unit, r.m_top) == (ot, un, mt)
            assert r.ops == ops
        else:
            assert st == 2 and not r.feasible
            assert r.min_feasible == mf


def test_sweep_helper_sorts_dedups_and_is_monotone():
    menu = synthetic_menu(33, 16, 4096, 44, byte_scale=64)
    lo, hi = 5000, 400000
    budgets = list(np.linspace(lo, hi, 40).astype(np.int64)) + [hi, lo]
    rows = rotor.sweep(menu, budgets, 500)
    assert [r.budget for r in rows] == sorted(set(int(b) for b in budgets))
    feas = [r.opt_time for r in rows if r.feasible]
    assert len(feas) > 10
    assert all(a >= b for a, b in zip(feas, feas[1:]))


def test_sweep_chains_equals_one_sweep_per_chain(orc):
    """rkr_sweep_chains (one batch over every chain's budgets) returns what
    one rkr_sweep call per chain returns, and both match solve_chain."""
    menus = [synthetic_menu(24, 8, 500, 41, byte_scale=1024),
             synthetic_menu(9, 3, 200, 7, byte_scale=256, tie_stress=True),
             synthetic_menu(33, 16, 4096, 44, byte_scale=64)]
    budgets = [[1000, 20000, 70000, 512000, 5],
               [300, 4000, 90000],
               [5000, 60000, 400000, 7]]
    multi = rotor.sweep_chains_raw(menus, budgets, 500)
    for menu, bs, rows in zip(menus, budgets, multi):
        single = rotor.sweep_raw(menu, bs, 500)
        assert len(rows) == len(single) == len(bs)
        for r, s in zip(rows, single):
            assert (r.budget, r.feasible, r.opt_time, r.unit, r.m_top, r.min_feasible, r.ops) == \
                   (s.budget, s.feasible, s.opt_time, s.unit, s.m_top, s.min_feasible, s.ops)
            st, ops, ot, un, mt, mf = orc.solve_chain(menu, r.budget, 500)
            assert r.feasible == (st == 0)
            if st == 0:
                assert (r.opt_time, r.ops) == (ot, ops)
            else:
                assert r.min_feasible == mf


@pytest.mark.parametrize("seed", [3, 11, 29])
def test_min_feasible_thresholds_equal_the_wide_table(orc, seed):
    """solve_chain's min-feasible search (chain_dp.hpp:265-288): the
    threshold recurrence on the budget's own table (default) and the
    reference's wide-table scan (RKR_TUNE_WIDE_SEARCH) give the same
    min_feasible_budget as the oracle, for every budget below and around it,
    single solves and batched sweeps."""
    rng = np.random.default_rng(seed)
    for L, B in ((3, 2), (9, 4), (17, 6)):
        menu = synthetic_menu(L, B, 300, int(rng.integers(1, 1 << 30)), tie_stress=bool(seed & 1))
        budgets = sorted({int(x) for x in rng.integers(1, int(menu.act_sizes.sum()) * 3, 24)})
        units = 37
        want = []
        for b in budgets:
            st, _, ot, un, mt, mf = orc.solve_chain(menu, b, units)
            want.append((st, mf))
        for flags in ((), ("wide_search",)):
            with rotor.tuning(*flags):
                rows = rotor.sweep_raw(menu, budgets, units)
                for b, r, (st, mf) in zip(budgets, rows, want):
                    assert r.feasible == (st == 0), (b, flags)
                    if st != 0:
                        assert r.min_feasible == mf, (b, flags)
                        with pytest.raises(rotor.InfeasibleBudget) as e:
                            rotor.solve_chain(rotor.Chain.skeleton(L), menu, b, units)
                        assert e.value.min_feasible_budget == mf, (b, flags)
