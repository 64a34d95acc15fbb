"""Device parity: librkr (sm_100a) against the reference's golden vectors and
the CPU oracle, bit-exact on opt (int64), arg kind/value and schedules.

Every test here runs the CUDA kernels through the C ABI (include/rkr.h).
"""
import numpy as np
import pytest

from helpers import ops_digest, table_digest, tri_row
from paper_2307_01236_b200 import rotor
from paper_2307_01236_b200.menu import BlockOption, Menu, synthetic_menu, tiny_chain_menu

pytestmark = pytest.mark.gpu

INF = rotor.K_INF_TIME
WIDTHS = ["auto", "64"]
KERNELS = ["tiles", "queue", "diagonal"]


@pytest.fixture(scope="module", autouse=True)
def _device():
    assert rotor.lib().rkr_device_ok(0) == 1, "no sm_100 device visible"


def dev_tables(menu, unit, M, width="auto", kernel="persistent"):
    if kernel == "tiles" and width == "64":
        pytest.skip("the budget-tile fill (K1t) runs the 32-bit cost path only")
    with rotor.DpTable(menu, unit, M, width=width, kernel=kernel) as t:
        o, k, v = t.download()
        return o, k, v, t.width()


def assert_same(a, b):
    for x, y in zip(a, b):
        np.testing.assert_array_equal(x, y)


# ---------------------------------------------------------------------------
# Reference known-answer tests (test_chain_dp.cpp:21-107, :203-221)
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("width", WIDTHS)
def test_tiny_chain_kats(kat, width):
    menu = tiny_chain_menu()
    t = kat["tiny"]
    o, k, v, w = dev_tables(menu, 1, t["M"], width)
    assert w == (64 if width == "64" else 32)
    assert o.tolist() == t["opt"] and k.tolist() == t["kind"] and v.tolist() == t["value"]
    with rotor.DpTable(menu, 1, 64, width=width) as tb:
        assert [tb.opt(0, 1, m) for m in (64, 12, 11, 10)] == [39, 39, 49, 49]
        assert tb.opt(0, 1, 9) >= INF
        assert tb.arg(0, 1, 10) == rotor.DpArg(rotor.DpArg.CUT, 1)
        assert tb.opt(0, 0, 5) >= INF
        assert tb.opt(0, 1, -3) == INF and tb.arg(0, 1, -3) == rotor.DpArg()
        assert tb.opt(0, 1, 10**6) == 39  # clamp to m_max (chain_dp.hpp:105)
        assert tb.max_candidates_per_cell == t["max_cands"]
        assert tb.worst_cell_allowance == t["worst_allow"] == 0


def test_single_block_sum():
    menu = Menu.from_options(
        [[BlockOption(0, 10, None, 4, 8, 8, 0), BlockOption(1, 10, 12, 10, 10, 10, 14)]], [4, 4])
    with rotor.DpTable(menu, 1, 100) as t:
        assert t.opt(0, 0, 100) == 22


@pytest.mark.parametrize("width", WIDTHS)
def test_tiny_chain_schedules(kat, width):
    menu = tiny_chain_menu()
    for M in (12, 10, 9):
        exp = kat["tiny"][f"schedule_M{M}"]
        with rotor.DpTable(menu, 1, M, width=width) as t:
            if exp["status"] == 0:
                assert [list(x) for x in t.backtrack(0, 1, M)] == exp["ops"]
            else:
                with pytest.raises(rotor.InfeasibleBudget):
                    t.backtrack(0, 1, M)
    chain = rotor.Chain.skeleton(2)
    with rotor.DpTable(menu, 1, 12, width=width) as t:
        ops = rotor.build_schedule_rec(t, menu, chain, 0, 1, 12)
        assert ops[2] == rotor.ScheduleOp(rotor.OP_COMPUTE, 1, "b1_loss", -1)


def test_solve_chain_kats(kat):
    menu = tiny_chain_menu()
    chain = rotor.Chain.skeleton(2)
    for e in kat["solve"]:
        if e["status"] == 0:
            sol = rotor.solve_chain(chain, menu, e["budget"], e["units"])
            assert (sol.opt_time, sol.unit, sol.m_top) == (e["opt_time"], e["unit"], e["m_top"])
            assert [list(x) for x in sol.raw_ops] == e["ops"]
        elif e["status"] == 2:
            with pytest.raises(rotor.InfeasibleBudget) as ei:
                rotor.solve_chain(chain, menu, e["budget"], e["units"])
            assert ei.value.min_feasible_budget == e["min_feasible"]
        else:
            with pytest.raises(rotor.ValidationError):
                rotor.solve_chain(chain, menu, e["budget"], e["units"])


# ---------------------------------------------------------------------------
# Reference random-menu suites (test_chain_dp.cpp:109-201): whole tables
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("suite", ["monotone", "ample", "symmetry", "enumeration", "work_bound",
                                   "relaxed"])
@pytest.mark.parametrize("width", WIDTHS)
@pytest.mark.parametrize("kernel", KERNELS)
def test_random_suites_whole_tables(random_suites, suite, width, kernel):
    S = random_suites[suite]
    for e in S["menus"]:
        menu = Menu.from_json(e["menu"])
        o, k, v, _ = dev_tables(menu, 1, S["M"], width, kernel)
        if "opt" in e:
            assert o.tolist() == e["opt"]
            assert k.tolist() == e["kind"]
            assert v.tolist() == e["value"]
        else:
            assert table_digest(o, k, v) == e["digest"]
        L = menu.L
        top = o[tri_row(L, 0, L - 1)]
        assert np.all(top[:-1] >= top[1:])  # monotone in m (:109-118)
        if suite == "enumeration":  # DP == exhaustive enumeration (:156-174)
            for i, m in enumerate(range(0, 21, 2)):
                ref = e["chain_oracle"][i]
                assert (top[m] >= INF and ref >= INF) or top[m] == ref


def test_ample_memory_identity(random_suites):
    # test_chain_dp.cpp:120-135
    for e in random_suites["ample"]["menus"]:
        menu = Menu.from_json(e["menu"])
        expect = 0
        for b in range(menu.L):
            expect += min(o.time_fwd + o.time_bwd for o in menu.options(b) if o.time_bwd is not None)
        with rotor.DpTable(menu, 1, 4096) as t:
            assert t.opt(0, menu.L - 1, 4096) == expect


def test_class_permutation_symmetry(random_suites):
    # test_chain_dp.cpp:137-154
    for e in random_suites["symmetry"]["menus"]:
        menu = Menu.from_json(e["menu"])
        if menu.L < 2:
            continue
        opts = [menu.options(b) for b in range(menu.L)]
        act = list(menu.act_sizes)
        act[1] = act[0]
        act[2] = act[0]
        opts[1] = opts[0]
        a = Menu.from_options(opts, act)
        sw = list(opts)
        sw[0], sw[1] = sw[1], sw[0]
        b = Menu.from_options(sw, act)
        with rotor.DpTable(a, 1, 20) as ta, rotor.DpTable(b, 1, 20) as tb:
            for m in range(21):
                assert ta.opt(0, a.L - 1, m) == tb.opt(0, b.L - 1, m)


# ---------------------------------------------------------------------------
# Synthetic chains against golden digests and the oracle
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("width", WIDTHS)
@pytest.mark.parametrize("kernel", KERNELS)
def test_synthetic_golden_tables(synthetic, width, kernel):
    for e in synthetic["tables"]:
        menu = synthetic_menu(e["L"], e["B"], e["M"], e["seed"], tie_stress=e["tie_stress"])
        o, k, v, _ = dev_tables(menu, 1, e["M"], width, kernel)
        assert table_digest(o, k, v) == e["digest"], (e["L"], e["M"])
        L = e["L"]
        r = tri_row(L, 0, L - 1)
        assert o[r].tolist() == e["top"]


def test_config1_solves_with_replay(synthetic, orc):
    chain = rotor.Chain.skeleton(24)
    for e in synthetic["solves"]:
        menu = synthetic_menu(e["L"], e["B"], e["M"], e["seed"], byte_scale=e["byte_scale"])
        if e["status"] == 0:
            sol = rotor.solve_chain(chain, menu, e["budget"], e["units"])
            assert (sol.opt_time, sol.unit, sol.m_top) == (e["opt_time"], e["unit"], e["m_top"])
            assert ops_digest(sol.raw_ops) == e["ops_digest"]
            peak, tm = orc.atomic_replay(menu, sol.raw_ops)  # simulated peak must be exact
            assert (peak, tm) == (e["replay_peak"], e["replay_time"])
            assert tm == sol.opt_time and peak <= e["budget"]
        else:
            with pytest.raises(rotor.InfeasibleBudget) as ei:
                rotor.solve_chain(chain, menu, e["budget"], e["units"])
            assert ei.value.min_feasible_budget == e["min_feasible"]


@pytest.mark.parametrize("L,B,M,seed,tie", [
    (5, 3, 40, 11, True), (17, 5, 300, 12, False), (40, 12, 700, 13, True), (64, 8, 1000, 14, False),
    (2, 40, 60, 15, True), (1, 4, 30, 16, False),
])
@pytest.mark.parametrize("width", WIDTHS)
@pytest.mark.parametrize("kernel", KERNELS)
def test_fresh_synthetic_vs_oracle(orc, L, B, M, seed, tie, width, kernel):
    menu = synthetic_menu(L, B, M, seed, tie_stress=tie)
    st, *ref = orc.fill(menu, 1, M)
    assert st == 0
    o, k, v, _ = dev_tables(menu, 1, M, width, kernel)
    assert_same((o, k, v), ref[:3])
    with rotor.DpTable(menu, 1, M, width=width, kernel=kernel) as t:
        assert t.max_candidates_per_cell == ref[3]
        ff = t.first_feasible(0, L - 1)
        top = ref[0][tri_row(L, 0, L - 1)]
        fin = np.nonzero(top < INF)[0]
        assert ff == (int(fin[0]) if len(fin) else -1)
        # device backtrack == oracle backtrack, at several budgets and sub-cells
        for (s, tt) in ((0, L - 1), (L // 2, L - 1), (0, max(0, L // 2 - 1))):
            for m in sorted(set([0, ff, M // 3, M // 2, M, M + 5, ff - 1, -1])):
                bst, bops = orc.build_schedule(menu, 1, M, tuple(ref[:3]), s, tt, m)
                if bst == 0:
                    assert t.backtrack(s, tt, m) == bops
                else:
                    with pytest.raises(rotor.InfeasibleBudget):
                        t.backtrack(s, tt, m)


@pytest.mark.parametrize("kernel", KERNELS)
def test_config3_reduced_twin_vs_oracle(orc, kernel):
    """GPT-2-XL-like chain (L=96, B=32) at M=1024: whole table bit-exact."""
    menu = synthetic_menu(96, 32, 1024, 45)
    st, *ref = orc.fill(menu, 1, 1024)
    o, k, v, w = dev_tables(menu, 1, 1024, "auto", kernel)
    assert w == 32
    assert_same((o, k, v), ref[:3])


@pytest.mark.parametrize("M", [9000, 20000])
def test_wide_budget_twin_vs_oracle(orc, M):
    """Several column groups, halo tiles and R=2 tiles (persistent kernel), both widths."""
    menu = synthetic_menu(24, 6, M, 46, tie_stress=True)
    st, *ref = orc.fill(menu, 1, M)
    for width in WIDTHS:
        assert_same(dev_tables(menu, 1, M, width)[:3], ref[:3])


def test_persistent_matches_diagonal_full_config3():
    """Full config 3: the persistent dataflow fill and the per-diagonal fill
    produce identical tables (sampled rows + digest of the top rows)."""
    L, M = 96, 16384
    menu = synthetic_menu(L, 32, M, 45)
    with rotor.DpTable(menu, 1, M) as a, rotor.DpTable(menu, 1, M, kernel="diagonal") as b:
        for (s, tt) in ((0, L - 1), (1, L - 1), (0, L - 2), (5, 60), (40, 41), (17, 17)):
            assert_same(a.row(s, tt), b.row(s, tt))


def test_config2_full_both_widths(synthetic):
    e = [x for x in synthetic["tables"] if x["L"] == 33][0]
    menu = synthetic_menu(33, 16, 4096, 44)
    a = dev_tables(menu, 1, 4096, "auto")
    b = dev_tables(menu, 1, 4096, "64")
    assert table_digest(*a[:3]) == e["digest"] == table_digest(*b[:3])


def test_config3_full_size_properties(orc):
    """Full GPT-2-XL-like size (96/32/16384): size-independent properties --
    monotone rows, schedules that replay to exactly opt with peak within the
    budget, and agreement of the 32- and 64-bit kernels on sampled rows."""
    L, M = 96, 16384
    menu = synthetic_menu(L, 32, M, 45)
    with rotor.DpTable(menu, 1, M) as t, rotor.DpTable(menu, 1, M, width="64") as t64:
        assert t.width() == 32 and t64.width() == 64
        for (s, tt) in ((0, L - 1), (0, L // 2), (L // 3, L - 1), (10, 20), (95, 95)):
            a, b = t.row(s, tt), t64.row(s, tt)
            assert_same(a, b)
            assert np.all(a[0][:-1] >= a[0][1:])
        ff = t.first_feasible(0, L - 1)
        assert ff > 0
        a0 = int(menu.act_sizes[0])
        for m in (ff, ff + 7, (ff + M) // 2, M):
            ops = t.backtrack(0, L - 1, m)
            peak, tm = orc.atomic_replay(menu, ops)
            assert tm == t.opt(0, L - 1, m)
            assert 0 <= peak <= m + a0
        with pytest.raises(rotor.InfeasibleBudget):
            t.backtrack(0, L - 1, ff - 1)


# ---------------------------------------------------------------------------
# Edge cases
# ---------------------------------------------------------------------------
def _edge_menus():
    out = []
    # option 0 not first, duplicate saved ids, a block with no saved option
    out.append(Menu.from_options([
        [BlockOption(2, 5, 4, 9, 10, 9, 11), BlockOption(0, 3, None, 4, 7, 7, 0),
         BlockOption(2, 4, 6, 8, 9, 9, 10), BlockOption(1, 6, 2, 12, 12, 11, 13)],
        [BlockOption(0, 2, None, 3, 6, 6, 0)],
        [BlockOption(0, 2, None, 3, 6, 6, 0), BlockOption(7, 3, 3, 6, 8, 7, 9)],
    ], [4, 3, 3, 2]))
    # zero-size activations and zero times
    out.append(Menu.from_options([
        [BlockOption(0, 0, None, 0, 0, 0, 0), BlockOption(1, 0, 0, 0, 0, 0, 0)],
        [BlockOption(0, 1, None, 0, 1, 1, 0), BlockOption(1, 0, 1, 1, 1, 1, 1)],
    ], [0, 0, 0]))
    # huge times: the 32-bit proof fails, the 64-bit kernels must take over
    big = 10**15
    out.append(Menu.from_options([
        [BlockOption(0, big, None, 2, 5, 5, 0), BlockOption(1, big, big, 6, 7, 6, 8)],
        [BlockOption(0, big, None, 2, 5, 5, 0), BlockOption(1, big + 1, big, 5, 6, 6, 7),
         BlockOption(2, big, big + 1, 5, 6, 6, 7)],
        [BlockOption(0, 1, None, 2, 5, 5, 0), BlockOption(1, 1, 1, 5, 6, 6, 7)],
    ], [2, 2, 2, 2]))
    # negative times (allowed by the reference types; 64-bit path)
    out.append(Menu.from_options([
        [BlockOption(0, -3, None, 2, 5, 5, 0), BlockOption(1, 4, -2, 6, 7, 6, 8)],
        [BlockOption(0, 5, None, 2, 5, 5, 0), BlockOption(1, -1, 3, 5, 6, 6, 7)],
    ], [2, 2, 2]))
    # thresholds far above any m, and peaks below the input (negative requirements)
    out.append(Menu.from_options([
        [BlockOption(0, 3, None, 2, 1, 1, 0), BlockOption(1, 4, 2, 3, 1, 1, 10**12)],
        [BlockOption(0, 5, None, 2, 1, 1, 0), BlockOption(1, 1, 3, 2, 1, 0, 1)],
    ], [2, 2, 2]))
    return out


@pytest.mark.parametrize("idx", range(5))
@pytest.mark.parametrize("M", [0, 1, 7, 40])
@pytest.mark.parametrize("unit", [1, 3])
def test_edge_menus_vs_oracle(orc, idx, M, unit):
    menu = _edge_menus()[idx]
    st, *ref = orc.fill(menu, unit, M)
    assert st == 0
    for width, kernel in ((w_, k_) for w_ in WIDTHS for k_ in KERNELS):
        if kernel == "tiles" and (width == "64" or idx in (2, 3)):
            continue  # K1t is 32-bit only (idx 2, 3 fail the overflow proof)
        o, k, v, w = dev_tables(menu, unit, M, width, kernel)
        if idx in (2, 3):
            assert w == 64
        assert_same((o, k, v), ref[:3])
        with rotor.DpTable(menu, unit, M, width=width) as t:
            assert t.max_candidates_per_cell == ref[3]
            for m in (-1, 0, M, M + 3):
                bst, bops = orc.build_schedule(menu, unit, M, tuple(ref[:3]), 0, menu.L - 1, m)
                if bst == 0:
                    assert t.backtrack(0, menu.L - 1, m) == bops
                else:
                    with pytest.raises(rotor.InfeasibleBudget):
                        t.backtrack(0, menu.L - 1, m)


def test_rejects_reference_out_of_bounds_shifts():
    m = Menu.from_options([[BlockOption(0, 1, None, 5, 6, 6, 0),
                            BlockOption(1, 1, 1, 2, 6, 6, 6)]], [5, 1])
    with pytest.raises(rotor.ValidationError, match="negative pack shift"):
        rotor.DpTable(m, 1, 10)


def test_accessor_ranges():
    with rotor.DpTable(tiny_chain_menu(), 1, 8) as t:
        with pytest.raises(IndexError):
            t.opt(1, 0, 3)
        with pytest.raises(IndexError):
            t.opt(0, 2, 3)
        assert (t.length(), t.unit(), t.m_max()) == (2, 1, 8)
        assert [t.act_units(i) for i in range(3)] == [4, 4, 2]


def test_cpp_drop_in_program():
    """The reference's DP test cases, compiled against include/remat_b200 and run."""
    import subprocess

    from paper_2307_01236_b200.build import build_cpp_tests

    path = build_cpp_tests()
    r = subprocess.run([path], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failed" in r.stdout


# ---------------------------------------------------------------------------
# Fill + walk in one call (rkr_table_refill_walk; fused into the K1t launch)
# ---------------------------------------------------------------------------
def _walk_or_inf(fn):
    try:
        return fn()
    except rotor.InfeasibleBudget:
        return "infeasible"


@pytest.mark.parametrize("kernel", KERNELS)
@pytest.mark.parametrize("L,B,M,seed", [(16, 6, 300, 3), (33, 16, 4096, 42 + 2), (5, 3, 40, 9)])
def test_refill_walk_matches_oracle(orc, kernel, L, B, M, seed):
    menu = synthetic_menu(L, B, M, seed, tie_stress=True)
    st, o, k, v, _, _ = orc.fill(menu, 1, M)
    assert st == 0
    cells = [(0, L - 1, M), (0, L - 1, M // 3), (0, L - 1, 2), (1, L - 1, M), (L // 2, L - 1, M // 2),
             (0, L // 2, M), (L - 1, L - 1, M), (0, L - 1, M + 5), (0, L - 1, -1)]
    with rotor.DpTable(menu, 1, M, kernel=kernel) as t:
        for s, tt, m in cells:
            bst, ref_ops = orc.build_schedule(menu, 1, M, (o, k, v), s, tt, m)
            want = ref_ops if bst == 0 else "infeasible"
            t.refill_walk(s, tt, m)
            assert _walk_or_inf(t.backtrack_fetch) == want, (s, tt, m)
            assert _walk_or_inf(lambda: t.backtrack(s, tt, m)) == want
        # the table after a fused fill is the oracle's table
        do, dk, dv = t.download()
        assert_same((do, dk, dv), (o, k, v))


@pytest.mark.parametrize("rows", [1, 2])
def test_tiles_without_communication_warp(orc, rows):
    """The barrier-aligned K1t variant (large tables) on small tables, fill and fused walk."""
    for L, B, M, seed in [(12, 6, 200, 7), (40, 8, 1500, 11), (3, 2, 20, 5)]:
        menu = synthetic_menu(L, B, M, seed, tie_stress=True)
        st, o, k, v, _, _ = orc.fill(menu, 1, M)
        with rotor.tuning("comm_off", tile_rows=rows), rotor.DpTable(menu, 1, M, kernel="tiles") as t:
            assert_same(t.download(), (o, k, v))
            t.refill_walk(0, L - 1, M)
            bst, ref_ops = orc.build_schedule(menu, 1, M, (o, k, v), 0, L - 1, M)
            assert bst == 0 and t.backtrack_fetch() == ref_ops


@pytest.mark.parametrize("L, B, M, seed", [(12, 6, 200, 7), (33, 16, 1500, 44), (9, 5, 40, 3),
                                          (40, 8, 3000, 12)])
def test_tiles_as_mixed_width_jobs(orc, L, B, M, seed):
    """Tile jobs whose later tiles are 16-slot (two rows per warp) after
    32-slot ones -- the plan config 3 runs to even out its last wave, forced
    here at half the tiles: whole table and the fused walk against the oracle."""
    menu = synthetic_menu(L, B, M, seed, tie_stress=True)
    st, o, k, v, _, _ = orc.fill(menu, 1, M)
    with rotor.tuning("jobs", "mixed"), rotor.DpTable(menu, 1, M, kernel="tiles") as t:
        assert_same(t.download(), (o, k, v))
        for m in (M, M // 2, M // 5):
            t.refill_walk(0, L - 1, m)
            bst, ref_ops = orc.build_schedule(menu, 1, M, (o, k, v), 0, L - 1, m)
            assert _walk_or_inf(t.backtrack_fetch) == (ref_ops if bst == 0 else "infeasible")
        assert_same(t.download(), (o, k, v))


@pytest.mark.parametrize("rows", [1, 2])
@pytest.mark.parametrize("comm", ["comm_on", "comm_off"])
def test_tiles_as_jobs(orc, comm, rows):
    """K1t as a one-table job queue (tables with more tiles than SMs, forced
    here on small ones), with and without the communication warp, one or two
    rows per warp: the whole table and the fused walk against the oracle."""
    for L, B, M, seed in [(12, 6, 200, 7), (33, 16, 1500, 44), (3, 2, 20, 5), (9, 5, 40, 3)]:
        menu = synthetic_menu(L, B, M, seed, tie_stress=True)
        st, o, k, v, _, _ = orc.fill(menu, 1, M)
        with rotor.tuning("jobs", comm, tile_rows=rows), rotor.DpTable(menu, 1, M, kernel="tiles") as t:
            assert_same(t.download(), (o, k, v))
            for m in (M, M // 2):
                t.refill_walk(0, L - 1, m)
                bst, ref_ops = orc.build_schedule(menu, 1, M, (o, k, v), 0, L - 1, m)
                got = _walk_or_inf(t.backtrack_fetch)
                assert got == (ref_ops if bst == 0 else "infeasible")
            assert_same(t.download(), (o, k, v))


@pytest.mark.parametrize("rows", [1, 2])
@pytest.mark.parametrize("flags", [("stream",), ("stream", "comm_off"), ("stream", "jobs")])
def test_tiles_streamed_programs(orc, flags, rows):
    """K1t with programs, thresholds and option data read from global memory
    (the long-chain variant), co-resident / without the communication warp /
    as tile jobs, one or two rows per warp: whole tables and the fused walk
    against the oracle."""
    # (200 x 32: the walk's menu copy (53 KB) exceeds the streamed kernels'
    # 32 KB program slices and option slices -- it must use the global menu)
    for L, B, M, seed in [(12, 6, 200, 7), (40, 20, 900, 45), (3, 2, 20, 5), (70, 9, 300, 8),
                          (200, 32, 40, 9)]:
        menu = synthetic_menu(L, B, M, seed, tie_stress=True)
        st, o, k, v, _, _ = orc.fill(menu, 1, M)
        with rotor.tuning(*flags, tile_rows=rows), rotor.DpTable(menu, 1, M, kernel="tiles") as t:
            assert_same(t.download(), (o, k, v))
            t.refill_walk(0, L - 1, M)
            bst, ref_ops = orc.build_schedule(menu, 1, M, (o, k, v), 0, L - 1, M)
            assert _walk_or_inf(t.backtrack_fetch) == (ref_ops if bst == 0 else "infeasible")


def _caller_menus(menu: Menu, seed: int):
    """A copy with the pack size of some saved options changed, and one with
    a saved option of every other block dropped (ids then missing)."""
    rng = np.random.default_rng(seed)
    bumped = Menu.from_options([menu.options(b) for b in range(menu.L)], list(menu.act_sizes))
    for o in range(len(bumped.save_mem)):
        if bumped.has_bwd[o] and rng.random() < 0.5:
            bumped.save_mem[o] += int(rng.integers(0, 12))
    blocks = []
    for b in range(menu.L):
        opts = menu.options(b)
        saved = [o for o in opts if o.option_id != 0]
        if b % 2 == 1 and len(saved) > 1:
            opts = [o for o in opts if o.option_id != saved[0].option_id]
        blocks.append(opts)
    dropped = Menu.from_options(blocks, list(menu.act_sizes))
    return bumped, dropped


@pytest.mark.parametrize("L, B, M, seed", [(12, 6, 200, 7), (20, 9, 400, 3), (33, 16, 600, 44)])
def test_build_schedule_rec_uses_the_callers_menu(orc, L, B, M, seed):
    """build_schedule_rec(table, menu, ...) looks options up in the CALLER's
    menu (chain_dp.hpp:200-205, :228), as the oracle does: a menu with other
    pack sizes walks other cells, a menu lacking a decided option raises
    ValidationError with the ops emitted before it (rkr_backtrack_menu)."""
    menu = synthetic_menu(L, B, M, seed, tie_stress=True)
    st, o, k, v, _, _ = orc.fill(menu, 1, M)
    assert st == 0
    bumped, dropped = _caller_menus(menu, seed)
    chain = rotor.Chain.skeleton(L)
    with rotor.DpTable(menu, 1, M) as t:
        for m in (M, 3 * M // 4, M // 2):
            # the table's own menu: identical to the plain walk
            assert t.backtrack(0, L - 1, m, menu=menu) == t.backtrack(0, L - 1, m)
            for caller in (bumped, dropped):
                rst, want = orc.build_schedule(caller, 1, M, (o, k, v), 0, L - 1, m)
                if rst == 0:
                    assert t.backtrack(0, L - 1, m, menu=caller) == want, m
                    continue
                done = []
                exc = rotor.ValidationError if rst == 1 else rotor.InfeasibleBudget
                with pytest.raises(exc):
                    rotor.build_schedule_rec(t, caller, chain, 0, L - 1, m, out=done)
                assert [(x.kind, x.block, x.option) for x in done] == want, m
