"""Per-item timing of the persistent fill (diagnostics for kernel tuning).

    python scripts/trace_report.py --config 3
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
t0 = st[:, 0].min()
s = (st - t0) / 1e3  # us
span = s[:, 3].max()
wait = s[:, 1] - s[:, 0]
comp = s[:, 2] - s[:, 1]
pub = s[:, 3] - s[:, 2]
print(f"config {a.config}: items {len(k)}, fill span {span:.1f} us")
print(f"  per item us: wait {wait.mean():.2f} (p90 {np.percentile(wait, 90):.2f})  "
      f"compute {comp.mean():.2f} (p90 {np.percentile(comp, 90):.2f})  publish {pub.mean():.2f}")
L = c["L"]
for kk in sorted(set(list(range(0, L, max(1, L // 12))) + [L - 1])):
    m = k == kk
    print(f"  k={kk:4d} n={m.sum():6d} start {s[m, 0].min():9.1f} end {s[m, 3].max():9.1f} "
          f"wait {wait[m].mean():7.2f} compute {comp[m].mean():7.2f} publish {pub[m].mean():6.2f}")
# handoff latency: for each (k, j), first start of diag k+1 after last end of diag k
