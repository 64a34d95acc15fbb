"""The dominance rule of the pruned open rows (rkr_tiles.cu, tile_job: the
one-table tile jobs, config 3), checked on the CPU against the reference's
own tables (oracle/_ref via the C restatement): in every cell (s < t, m)
where all options of block s are admissible, the first minimum of the option
scan (chain_dp.hpp:139-156: menu order, strict '<') over the block's
undominated options equals the one over all of them -- value and option.
Synthetic menus at unit 1 (sizes are budget units), tie-stress menus
included (equal pass times and shifts)."""
import numpy as np
import pytest

from helpers import tri_row
from paper_2307_01236_b200.menu import synthetic_menu

INF = (2**63 - 1) // 4


def undominated(tot, pack):
    """Indices kept by the kernel's rule: x is dropped if some y has pack <=
    x's and pass time <= x's (y before x) or < x's (y after x)."""
    keep = []
    for x in range(len(tot)):
        dom = False
        for y in range(len(tot)):
            if y != x and pack[y] <= pack[x] and (tot[y] <= tot[x] if y < x else tot[y] < tot[x]):
                dom = True
                break
        if not dom:
            keep.append(x)
    return keep


def first_min(idx, tot, sub_row, pack, m):
    best, arg = INF, -1
    for i in idx:
        sub = sub_row[m - pack[i]]
        if sub >= INF:
            continue
        v = tot[i] + sub
        if v < best:
            best, arg = v, i
    return best, arg


@pytest.mark.parametrize("L, B, M, seed, tie", [(10, 12, 300, 3, False), (12, 8, 250, 5, True),
                                              (8, 16, 200, 9, True), (14, 6, 400, 11, False)])
def test_pruned_option_scan_equals_full(orc, L, B, M, seed, tie):
    menu = synthetic_menu(L, B, M, seed, tie_stress=tie)
    st, o, _, _, _, _ = orc.fill(menu, 1, M)
    assert st == 0
    act = menu.act_sizes
    checked = 0
    for s in range(L - 1):
        lo, hi = int(menu.option_offsets[s]), int(menu.option_offsets[s + 1])
        saved = [q for q in range(lo, hi) if menu.has_bwd[q]]
        tot = [int(menu.time_fwd[q] + menu.time_bwd[q]) for q in saved]
        pack = [int(menu.save_mem[q] - act[s]) for q in saved]
        fwd = [int(menu.peak_fwd[q] - act[s]) for q in saved]
        bwd = [int(menu.peak_bwd[q] - act[s]) for q in saved]
        keep = undominated(tot, pack)
        assert len(keep) >= 1
        for t in range(s + 1, L):
            seed_t = 2 * int(act[t + 1]) if t < L - 1 else 0
            thx = max(max(f + seed_t for f in fwd), max(max(b, p) for b, p in zip(bwd, pack)))
            sub_row = o[tri_row(L, s + 1, t)]
            for m in range(max(thx, 0), M + 1):
                full = first_min(range(len(saved)), tot, sub_row, pack, m)
                pruned = first_min(keep, tot, sub_row, pack, m)
                assert full == pruned, (s, t, m, full, pruned)
                checked += 1
    assert checked > 1000, checked
