"""Budget-axis sharded tables (config 5 design) on one GPU: every shard's
halo arrives through the fused in-kernel exchange; the assembled table and the
cross-shard schedules are bit-exact against the CPU oracle and identical to
the unsharded table."""
import numpy as np
import pytest

from helpers import tri_row
from paper_2307_01236_b200 import rotor
from paper_2307_01236_b200.menu import synthetic_menu

pytestmark = pytest.mark.gpu


def _same(a, b):
    for x, y in zip(a, b):
        np.testing.assert_array_equal(x, y)


@pytest.mark.parametrize("L,B,M,seed,tie,n", [
    (12, 4, 600, 21, True, 2),
    (20, 6, 1500, 22, False, 3),
    (33, 8, 4096, 23, False, 4),
    (16, 5, 9000, 24, True, 2),     # R = 2 tiles
    (24, 6, 2100, 25, False, 5),
])
@pytest.mark.parametrize("width", ["auto", "64"])
def test_sharded_table_matches_oracle(orc, L, B, M, seed, tie, n, width):
    menu = synthetic_menu(L, B, M, seed, tie_stress=tie)
    st, *ref = orc.fill(menu, 1, M)
    assert st == 0
    with rotor.ShardedTable(menu, 1, M, n, width=width) as sh:
        # 32-bit shards run budget-tile jobs (K1t), 64-bit ones the queue (K1p)
        assert sh.shard(0).kernel() == ("queue" if width == "64" else "tiles")
        rg = sh.ranges()
        assert len(rg) == n and rg[0][0] == 0 and rg[-1][1] == M + 1
        for rep in range(2):
            if rep:
                sh.refill()
            _same(sh.download(), ref[:3])
        top = ref[0][tri_row(L, 0, L - 1)]
        fin = np.nonzero(top < rotor.K_INF_TIME)[0]
        ms = sorted(set([int(fin[0]) if len(fin) else 0, M // 3, M // 2, M, M + 9,
                         rg[-1][0], rg[-1][0] - 1, -1]))
        for m in ms:
            bst, bops = orc.build_schedule(menu, 1, M, tuple(ref[:3]), 0, L - 1, m)
            if bst == 0:
                assert sh.backtrack(0, L - 1, m) == bops
                assert sh.opt(0, L - 1, m) == (top[min(m, M)])
            else:
                with pytest.raises(rotor.InfeasibleBudget):
                    sh.backtrack(0, L - 1, m)


def test_sharded_equals_unsharded_config2_size():
    menu = synthetic_menu(33, 16, 4096, 44)
    with rotor.DpTable(menu, 1, 4096) as t, rotor.ShardedTable(menu, 1, 4096, 4) as sh:
        a = t.download()
        b = sh.download()
        _same(a, b)


def test_too_many_shards_is_rejected():
    menu = synthetic_menu(12, 4, 200, 3)
    with pytest.raises(rotor.ValidationError, match="too many shards"):
        rotor.ShardedTable(menu, 1, 200, 50)


@pytest.mark.parametrize("L,B,M,seed,n,kernel", [(16, 4, 900, 31, 3, "queue"),
                                                   (150, 8, 600, 32, 2, "persistent")])
def test_sharded_kernels_exact(orc, L, B, M, seed, n, kernel):
    """The row-segment queue (K1p) on request, and a long chain (streamed K1t
    shards): both bit-exact."""
    menu = synthetic_menu(L, B, M, seed, tie_stress=True)
    st, *ref = orc.fill(menu, 1, M)
    with rotor.ShardedTable(menu, 1, M, n, kernel=kernel) as sh:
        assert sh.shard(0).kernel() == ("queue" if kernel == "queue" else "tiles")
        _same(sh.download(), ref[:3])
        sh.refill()
        _same(sh.download(), ref[:3])
