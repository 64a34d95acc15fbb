"""Small workload for compute-sanitizer (memcheck / racecheck / synccheck):
every kernel family once, both widths, sharded + batched paths."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2307_01236_b200 import rotor  # noqa: E402
from paper_2307_01236_b200.menu import synthetic_menu, tiny_chain_menu  # noqa: E402

for width in ("auto", "64"):
    for kernel in ("tiles", "queue", "diagonal"):
        if kernel == "tiles" and width == "64":
            continue  # K1t is 32-bit only
        m = synthetic_menu(10, 4, 600, 5, tie_stress=True)
        with rotor.DpTable(m, 1, 600, width=width, kernel=kernel) as t:
            t.download()
            t.backtrack(0, 9, 600)
            t.refill_walk(0, 9, 600)  # fused walk (K1t) / fill + walk
            t.backtrack_fetch()
            t.first_feasible(0, 9)
    with rotor.ShardedTable(synthetic_menu(12, 4, 900, 6), 1, 900, 3, width=width) as sh:
        sh.download()
        sh.backtrack(0, 11, 900)
# K1t split tails (>= 2 option batches: 12 options per block)
with rotor.DpTable(synthetic_menu(14, 12, 600, 7, tie_stress=True), 1, 600, kernel="tiles") as t:
    t.refill_walk(0, 13, 600)
    t.backtrack_fetch()
# streamed K1t as tile jobs with the fused walk on a long chain (the walk's
# menu copy does not fit the program slices: global-menu walk)
with rotor.tuning("jobs"), rotor.DpTable(synthetic_menu(200, 32, 40, 9), 1, 40, kernel="tiles") as t:
    t.refill_walk(0, 199, 40)
    t.backtrack_fetch()
# two rows per warp (16-slot tiles), co-resident and as tile jobs
for fl in ((), ("jobs",)):
    with rotor.tuning(*fl, tile_rows=2), rotor.DpTable(synthetic_menu(21, 6, 500, 4), 1, 500,
                                                       kernel="tiles") as t:
        t.refill_walk(0, 20, 500)
        t.backtrack_fetch()
# K1t without the communication warp (the large-table variant)
with rotor.tuning("comm_off"), rotor.DpTable(synthetic_menu(10, 4, 600, 5), 1, 600, kernel="tiles") as t:
    t.refill_walk(0, 9, 600)
    t.backtrack_fetch()
for kernel in ("persistent", "queue"):  # tile jobs / row-segment queue
    b = rotor.Batch([tiny_chain_menu(), synthetic_menu(8, 3, 300, 7)], [1, 1], [64, 300],
                    kernel=kernel)
    b.table(1).download()
    b.refill()
    b.table(0).download()
    b.close()
rotor.sweep_raw(synthetic_menu(12, 4, 500, 8, byte_scale=64), [3000, 20000, 60000], 500)
rotor.solve_chain(rotor.Chain.skeleton(2), tiny_chain_menu(), 16, 16)
print("sanitize workload done")
# round 2: mixed-width tile jobs, the caller's-menu walk, the min-feasible
# threshold kernel (an infeasible solve and an infeasible sweep budget)
with rotor.tuning("jobs", "mixed"), rotor.DpTable(synthetic_menu(21, 6, 700, 4), 1, 700,
                                                   kernel="tiles") as t:
    t.refill_walk(0, 20, 700)
    t.backtrack_fetch()
    t.backtrack(0, 20, 700, menu=synthetic_menu(21, 6, 700, 4))
try:
    rotor.solve_chain(rotor.Chain.skeleton(2), tiny_chain_menu(), 12, 12)
except rotor.InfeasibleBudget:
    pass
rotor.sweep_raw(synthetic_menu(9, 4, 300, 3, byte_scale=64), [50, 400, 3000, 20000], 300)
# round 2 (late): dominance-pruned open rows and paired tail units of the
# one-table tile-job kernel, on a tie-stress menu
with rotor.tuning("jobs", "mixed"), rotor.DpTable(synthetic_menu(24, 8, 900, 11, tie_stress=True), 1, 900,
                                                   kernel="tiles") as t:
    t.refill_walk(0, 23, 900)
    t.backtrack_fetch()
print("sanitize workload (pruned rows) done")
