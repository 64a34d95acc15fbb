"""Randomised differential tests: arbitrary (including odd) menus, device vs
CPU oracle, every cell and a schedule per table.  Menus are drawn with an
explicit seeded generator so failures reproduce."""
import numpy as np
import pytest

from helpers import tri_row
from paper_2307_01236_b200 import rotor
from paper_2307_01236_b200.menu import BlockOption, Menu

pytestmark = pytest.mark.gpu


def odd_menu(rng):
    """Blocks with 0-5 saved options in random order (option 0 anywhere),
    duplicate ids, equal times (ties), zero sizes, peaks below the input."""
    L = int(rng.integers(1, 9))
    act = [int(x) for x in rng.integers(0, 7, L + 1)]
    blocks = []
    for i in range(L):
        a_in = act[i]
        opts = []
        tf0 = int(rng.integers(0, 6))
        pf0 = int(rng.integers(0, 12))
        opts.append(BlockOption(0, tf0, None, a_in, pf0, int(rng.integers(0, 12)), 0))
        for o in range(int(rng.integers(0, 6))):
            oid = int(rng.integers(1, 4))  # duplicates on purpose
            save = a_in + int(rng.integers(0, 8))
            opts.append(BlockOption(oid, int(rng.integers(0, 6)), int(rng.integers(0, 6)), save,
                                    int(rng.integers(0, 16)), int(rng.integers(0, 16)),
                                    int(rng.integers(0, 20))))
        order = rng.permutation(len(opts))
        blocks.append([opts[q] for q in order])
    return Menu.from_options(blocks, act)


@pytest.mark.parametrize("seed", range(6))
def test_random_odd_menus_vs_oracle(orc, seed):
    rng = np.random.default_rng(1000 + seed)
    for _ in range(25):
        menu = odd_menu(rng)
        unit = int(rng.integers(1, 4))
        M = int(rng.integers(0, 60))
        st, *ref = orc.fill(menu, unit, M)
        if st != 0:  # the oracle rejects it (e.g. no option 0 can't happen here)
            with pytest.raises(rotor.ValidationError):
                rotor.DpTable(menu, unit, M)
            continue
        for width in ("auto", "64"):
            for kernel in ("persistent", "diagonal"):
                with rotor.DpTable(menu, unit, M, width=width, kernel=kernel) as t:
                    o, k, v = t.download()
                    np.testing.assert_array_equal(o, ref[0])
                    np.testing.assert_array_equal(k, ref[1])
                    np.testing.assert_array_equal(v, ref[2])
                    assert t.max_candidates_per_cell == ref[3]
                    L = menu.L
                    m = int(rng.integers(-2, M + 3))
                    bst, bops = orc.build_schedule(menu, unit, M, tuple(ref[:3]), 0, L - 1, m)
                    if bst == 0:
                        assert t.backtrack(0, L - 1, m) == bops
                    elif bst == 2:
                        with pytest.raises(rotor.InfeasibleBudget):
                            t.backtrack(0, L - 1, m)


@pytest.mark.parametrize("seed", range(3))
def test_random_solve_chain_vs_oracle(orc, seed):
    rng = np.random.default_rng(2000 + seed)
    for _ in range(30):
        menu = odd_menu(rng)
        budget = int(rng.integers(0, 80))
        units = int(rng.integers(1, 40))
        st, ops, ot, un, mt, mf = orc.solve_chain(menu, budget, units)
        chain = rotor.Chain.skeleton(menu.L)
        if st == 0:
            sol = rotor.solve_chain(chain, menu, budget, units)
            assert (sol.opt_time, sol.unit, sol.m_top) == (ot, un, mt)
            assert sol.raw_ops == ops
        elif st == 2:
            with pytest.raises(rotor.InfeasibleBudget) as e:
                rotor.solve_chain(chain, menu, budget, units)
            assert e.value.min_feasible_budget == mf
        else:
            with pytest.raises(rotor.ValidationError):
                rotor.solve_chain(chain, menu, budget, units)


@pytest.mark.parametrize("seed", range(3))
def test_random_refill_walks_vs_oracle(orc, seed):
    """Odd menus, wider budgets, every persistent kernel: fill, then two
    refill + fused-walk rounds on the same table (the K1t kernel re-zeroes its
    own flags between launches) against the oracle's table and schedule."""
    rng = np.random.default_rng(3000 + seed)
    for _ in range(15):
        menu = odd_menu(rng)
        unit = int(rng.integers(1, 4))
        M = int(rng.integers(0, 300))
        st, *ref = orc.fill(menu, unit, M)
        if st != 0:
            continue
        L = menu.L
        for kernel in ("persistent", "tiles", "queue"):
            with rotor.DpTable(menu, unit, M, kernel=kernel) as t:
                for _rep in range(2):
                    m = int(rng.integers(-2, M + 3))
                    bst, bops = orc.build_schedule(menu, unit, M, tuple(ref[:3]), 0, L - 1, m)
                    if bst == 0:
                        t.refill_walk(0, L - 1, m)
                        assert t.backtrack_fetch() == bops
                    elif bst == 2:
                        t.refill_walk(0, L - 1, m)
                        with pytest.raises(rotor.InfeasibleBudget):
                            t.backtrack_fetch()
                    o, k, v = t.download()
                    np.testing.assert_array_equal(o, ref[0])
                    np.testing.assert_array_equal(k, ref[1])
                    np.testing.assert_array_equal(v, ref[2])


@pytest.mark.parametrize("scale", [1, 1000003])
@pytest.mark.parametrize("seed", range(3))
def test_random_menus_mixed_width_jobs(orc, seed, scale):
    """Odd menus through the mixed-width tile-job kernel, whose option batches
    run ungated when no threshold of the row is above the warp's smallest
    budget: rows on both sides of that test (budgets up to 300 slots, 32- and
    16-slot tiles), and sizes scaled past 2^29 (unit 1: thresholds far above
    and below the budgets, negative forward requirements)."""
    rng = np.random.default_rng(4000 + seed)
    for _ in range(12):
        menu = odd_menu(rng)
        if scale > 1:
            for f in ("save_mem", "peak_fwd", "peak_fwd_pre", "peak_bwd"):
                setattr(menu, f, getattr(menu, f) * scale)
            menu.act_sizes = menu.act_sizes * scale
        unit = 1 if scale > 1 else int(rng.integers(1, 4))
        M = int(rng.integers(40, 300))
        st, *ref = orc.fill(menu, unit, M)
        if st != 0:
            continue
        with rotor.tuning("jobs", "mixed", tile_rows=1), \
                rotor.DpTable(menu, unit, M, kernel="tiles") as t:
            o, k, v = t.download()
            np.testing.assert_array_equal(o, ref[0])
            np.testing.assert_array_equal(k, ref[1])
            np.testing.assert_array_equal(v, ref[2])
