"""Small workload for compute-sanitizer (memcheck / racecheck / synccheck):
every kernel family once, both widths, sharded + batched paths."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2307_01236_b200 import rotor  # noqa: E402
from paper_2307_01236_b200.menu import synthetic_menu, tiny_chain_menu  # noqa: E402

for width in ("auto", "64"):
    for kernel in ("persistent", "diagonal"):
        m = synthetic_menu(10, 4, 600, 5, tie_stress=True)
        with rotor.DpTable(m, 1, 600, width=width, kernel=kernel) as t:
            t.download()
            t.backtrack(0, 9, 600)
            t.first_feasible(0, 9)
    with rotor.ShardedTable(synthetic_menu(12, 4, 900, 6), 1, 900, 3, width=width) as sh:
        sh.download()
        sh.backtrack(0, 11, 900)
b = rotor.Batch([tiny_chain_menu(), synthetic_menu(8, 3, 300, 7)], [1, 1], [64, 300])
b.table(1).download()
b.close()
rotor.sweep_raw(synthetic_menu(12, 4, 500, 8, byte_scale=64), [3000, 20000, 60000], 500)
rotor.solve_chain(rotor.Chain.skeleton(2), tiny_chain_menu(), 16, 16)
print("sanitize workload done")
