"""Dominance pruning of open rows (K1t mixed-width tile jobs, the config-3
path): menus built to sit on both sides of its rules -- duplicate options
(equal pass time and pack shift: the earlier one must win), Pareto menus
with more undominated options than the per-block list holds (the block
falls back to the full scan), options equal in pass time but not in pack
shift -- every cell against the oracle, and pruned against unpruned tables."""
import numpy as np
import pytest

from paper_2307_01236_b200 import rotor
from paper_2307_01236_b200.menu import BlockOption, Menu, synthetic_menu

pytestmark = pytest.mark.gpu


def assert_same(got, ref):
    for g, r in zip(got, ref):
        np.testing.assert_array_equal(g, r)


def shaped_menu(L, B, M, seed, kind):
    """kind: 'pareto' (pass time falls as the pack shift grows: nothing is
    dominated), 'dup' (options repeated at other menu positions, ids
    shuffled), 'ties' (pass times from {100, 101}, pack shifts from 3
    values: many equal pairs)."""
    rng = np.random.default_rng(seed)
    a = max(1, M // (2 * L))
    act = [int(x) for x in rng.integers(a // 2 + 1, 3 * a // 2 + 2, L + 1)]
    blocks = []
    for i in range(L):
        a_in, a_out = act[i], act[i + 1]
        tf0 = int(rng.integers(50, 500))
        pf0 = a_in + a_out + int(rng.integers(0, a + 1))
        opts = [BlockOption(0, tf0, None, a_in, pf0, pf0, 0)]
        for o in range(1, B + 1):
            if kind == "pareto":
                save = a_in + a_out + o * max(1, a // 8)
                tb = 2000 - 37 * o
            elif kind == "ties":
                save = a_in + a_out + int(rng.integers(0, 3)) * a
                tb = int(rng.integers(0, 2))
            else:
                save = a_in + a_out + int(rng.integers(0, 3 * a + 1))
                tb = int(rng.integers(100, 1001))
            tf = tf0 + (0 if kind == "ties" else int(rng.integers(0, 5)))
            pf = max(save, pf0) + int(rng.integers(0, a + 1))
            pre = int(rng.integers(max(save, pf - a_out), pf + 1))
            pb = save + a_out + int(rng.integers(0, a + 1))
            opts.append(BlockOption(o, tf, tb + (100 if kind == "ties" else 0), save, pf, pre, pb))
        if kind == "dup":  # every saved option again, later in the menu
            extra = [BlockOption(int(rng.integers(1, B + 1)), x.time_fwd, x.time_bwd, x.save_mem,
                                 x.peak_fwd, x.peak_fwd_pre, x.peak_bwd) for x in opts[1:]]
            opts = opts + [extra[q] for q in rng.permutation(len(extra))]
        blocks.append(opts)
    return Menu.from_options(blocks, act)


@pytest.mark.parametrize("kind, B", [("pareto", 12), ("pareto", 24), ("dup", 8), ("ties", 16)])
@pytest.mark.parametrize("rows", [1, 2])
def test_pruned_rows_vs_oracle(orc, kind, B, rows):
    L, M = 20, 2500
    menu = shaped_menu(L, B, M, 90 + B, kind)
    st, o, k, v, _, _ = orc.fill(menu, 1, M)
    assert st == 0
    with rotor.tuning("jobs", "mixed", tile_rows=rows), rotor.DpTable(menu, 1, M, kernel="tiles") as t:
        assert_same(t.download(), (o, k, v))
        t.refill_walk(0, L - 1, M)
        bst, ref_ops = orc.build_schedule(menu, 1, M, (o, k, v), 0, L - 1, M)
        assert bst == 0 and t.backtrack_fetch() == ref_ops


@pytest.mark.parametrize("L, B, M, seed, tie", [(33, 16, 4096, 44, False), (48, 32, 3000, 5, True)])
def test_pruned_equals_unpruned(L, B, M, seed, tie):
    """The same table with and without pruning (config-2-sized; a tie-stress
    menu), bit for bit."""
    menu = synthetic_menu(L, B, M, seed, tie_stress=tie)
    with rotor.tuning("jobs", "mixed"), rotor.DpTable(menu, 1, M, kernel="tiles") as t:
        a = t.download()
    with rotor.tuning("jobs", "mixed", "no_prune"), rotor.DpTable(menu, 1, M, kernel="tiles") as t:
        b = t.download()
    assert_same(a, b)
