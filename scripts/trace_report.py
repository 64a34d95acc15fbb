"""Per-item timing of the persistent fill (diagnostics for kernel tuning).

    python scripts/trace_report.py --config 3
Stamps per item: dequeued, diag k-2 met, bulk done, diag k-1 met, tail done, published.
"""
import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2307_01236_b200 import rotor  # noqa: E402
from paper_2307_01236_b200.menu import config_menu, CONFIGS  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=2)
a = ap.parse_args()
c = CONFIGS[a.config]
menu = config_menu(a.config)
t = rotor.DpTable(menu, 1, c["M"])
t.trace(True)
for _ in range(3):
    t.refill()
t.sync()
st, k, j = t.trace_read()
st = st.astype(np.float64)
s = (st - st[:, 0].min()) / 1e3  # us
span = s[:, 5].max()
d = np.diff(s, axis=1)  # wait2, bulk, wait1, tail, publish
names = ["wait_k-2", "bulk", "wait_k-1", "tail", "publish"]
print(f"config {a.config}: items {len(k)}, fill span {span:.1f} us")
print("  mean us: " + "  ".join(f"{n} {d[:, i].mean():.2f}" for i, n in enumerate(names)))
L = c["L"]
for kk in sorted(set(list(range(0, L, max(1, L // 12))) + [L - 1])):
    m = k == kk
    print(f"  k={kk:4d} n={m.sum():6d} start {s[m, 0].min():8.1f} k-1met {s[m, 3].min():8.1f}.."
          f"{s[m, 3].max():8.1f} end {s[m, 5].max():8.1f} | " +
          " ".join(f"{d[m, i].mean():6.2f}" for i in range(5)))
