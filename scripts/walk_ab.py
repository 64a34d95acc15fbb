"""Device cost of the schedule walk: stand-alone backtrack launches and the
walk fused into the fill (refill_walk - refill), per config menu."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2307_01236_b200 import rotor  # noqa: E402
from paper_2307_01236_b200.menu import config_menu  # noqa: E402

GEOM = {1: (24, 500), 2: (33, 4096), 3: (96, 16384)}


def per_call(fn, t, n):
    for _ in range(3):
        fn()
    t.sync()
    t0 = time.perf_counter()
    for _ in range(n):
        fn()
    t.sync()
    return 1e6 * (time.perf_counter() - t0) / n


for cfg in (1, 2, 3):
    L, M = GEOM[cfg]
    menu = config_menu(cfg)
    t = rotor.DpTable(menu, 1, M)
    n = 20 if cfg == 3 else 200
    bt = per_call(lambda: t.backtrack_async(0, L - 1, M), t, n)
    rf = per_call(t.refill, t, n)
    rw = per_call(lambda: t.refill_walk(0, L - 1, M), t, n)
    ops = t.backtrack_fetch()
    t.backtrack_async(0, L - 1, M)
    assert t.backtrack_fetch() == ops == t.backtrack(0, L - 1, M)
    print(f"{os.environ.get('TAG', '')} cfg {cfg}: ops {len(ops)} backtrack {bt:7.1f} us  "
          f"refill {rf:8.1f}  refill_walk {rw:8.1f}  fused walk {rw - rf:6.1f} us")
