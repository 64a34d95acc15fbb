"""Long randomised check of the one-table tile-job kernel (pruned open rows,
paired tail units, mixed widths) against the CPU oracle: whole tables and
the fused walk, for as many menus as fit in --seconds.

    python scripts/fuzz_mixed.py --seconds 480
"""
import argparse
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle.pyoracle import Orc  # noqa: E402  (test infrastructure: the checker)
from paper_2307_01236_b200 import rotor  # noqa: E402
from paper_2307_01236_b200.menu import synthetic_menu  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--seconds", type=float, default=300)
ap.add_argument("--seed", type=int, default=2024)
ap.add_argument("--mode", default="mixed", choices=["mixed", "auto", "comm_off"],
                help="mixed: one-table tile jobs with half tiles (pruned open rows); auto: the "
                     "default plan (co-resident for small tables); comm_off: no communication warp")
a = ap.parse_args()
FLAGS = {"mixed": ("jobs", "mixed"), "auto": (), "comm_off": ("comm_off",)}[a.mode]
orc = Orc()
rng = np.random.default_rng(a.seed)
t_end = time.time() + a.seconds
n = cells = 0
while time.time() < t_end:
    L = int(rng.integers(2, 41))
    B = int(rng.integers(1, 33))
    M = int(rng.integers(60, 2500))
    tie = bool(rng.integers(0, 2))
    menu = synthetic_menu(L, B, M, int(rng.integers(0, 1 << 30)), tie_stress=tie)
    st, o, k, v, _, _ = orc.fill(menu, 1, M)
    assert st == 0
    rows = int(rng.integers(0, 3))  # 0 auto, 1, 2
    with rotor.tuning(*FLAGS, tile_rows=rows), rotor.DpTable(menu, 1, M, kernel="tiles") as t:
        go, gk, gv = t.download()
        if not (np.array_equal(go, o) and np.array_equal(gk, k) and np.array_equal(gv, v)):
            raise SystemExit(f"MISMATCH L={L} B={B} M={M} tie={tie} rows={rows}")
        m = int(rng.integers(0, M + 1))
        t.refill_walk(0, L - 1, m)
        try:
            ops = t.backtrack_fetch()
        except rotor.InfeasibleBudget:
            ops = "infeasible"
        bst, ref = orc.build_schedule(menu, 1, M, (o, k, v), 0, L - 1, m)
        if ops != (ref if bst == 0 else "infeasible"):
            raise SystemExit(f"WALK MISMATCH L={L} B={B} M={M} m={m}")
    n += 1
    cells += o.size
print(f"fuzz_mixed ({a.mode}): {n} tables ({cells / 1e6:.1f} M cells) bit-exact against the oracle, walks equal")
