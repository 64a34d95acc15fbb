"""Per-(diagonal, tile) stamps of the K1t fill: where the waits sit.

    python scripts/trace_tiles.py --config 2
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
t = rotor.DpTable(config_menu(a.config), 1, c["M"])
assert t.kernel() == "tiles", t.kernel()
t.trace(True)
for _ in range(3):
    t.refill()
t.sync()
st, k, j = t.trace_read()
st = st.astype(np.float64)
st = (st - st[:, 0].min()) / 1e3
L, T = k.max() + 1, j.max() + 1
S = st.reshape(L, T, 6)
print(f"config {a.config}: L={L} tiles={T} span {S[:, :, 5].max():.1f} us")
print("per-step mean (us): bulk %.2f wait %.2f tail %.2f publish %.2f" % tuple(
    np.diff(S[:, :, 1:], axis=2).mean(axis=(0, 1))))
for kk in [1, 2, L // 4, L // 2, 3 * L // 4, L - 1]:
    w = S[kk, :, 3] - S[kk, :, 2]
    print(f"k={kk:3d}: step start j=0 {S[kk,0,0]:7.1f} j=T/2 {S[kk,T//2,0]:7.1f} j=T-1 {S[kk,T-1,0]:7.1f} | "
          f"wait by tile quartile: " + " ".join(f"{w[q*T//4:(q+1)*T//4].mean():.2f}" for q in range(4)) +
          f" | tail {np.mean(S[kk,:,4]-S[kk,:,3]):.2f}")
# lag of tile j behind tile 0 at the end
print("end lag vs tile 0 (us), every T/8 tiles:",
      " ".join(f"{S[L-1, q, 5] - S[L-1, 0, 5]:.1f}" for q in range(0, T, max(1, T // 8))))
