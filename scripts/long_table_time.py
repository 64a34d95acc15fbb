"""Device time of a long chain's fill as tile jobs with streamed programs
(L=200, B=32, M=16384): refill and refill + fused walk."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2307_01236_b200 import rotor  # noqa: E402
from paper_2307_01236_b200.menu import synthetic_menu  # noqa: E402

L, B, M = 200, 32, 16384
t = rotor.DpTable(synthetic_menu(L, B, M, 77), 1, M)
print("kernel", t.kernel())
for fn, name in ((t.refill, "refill"), (lambda: t.refill_walk(0, L - 1, M), "refill_walk")):
    fn()
    t.sync()
    t0 = time.perf_counter()
    for _ in range(5):
        fn()
    t.sync()
    print(f"{os.environ.get('TAG', '')} {name}: {1e3 * (time.perf_counter() - t0) / 5:.2f} ms")
