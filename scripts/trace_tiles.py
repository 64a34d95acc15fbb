"""Per-(diagonal, tile) stamps of the K1t fill: the cross-SM timeline and,
within each step, who holds the READY barrier -- the communication warp
(waiting for the lower tiles' diagonal k-1) or the compute warps (their bulk).

    python scripts/trace_tiles.py --config 3

Stamps (rkr_tiles.cu): [0] globaltimer at the step start; SM cycles: [1]
step start, [2] warp 0's bulk done, [3] the communication warp's acquisition
of diagonal k-1, [4] READY passed, [5] warp 0's tail done.  Cycle stamps of
one step come from one SM, so their differences are exact.
"""
import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2307_01236_b200 import rotor  # noqa: E402
from paper_2307_01236_b200.menu import config_menu, CONFIGS  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=3)
ap.add_argument("--sm-mhz", type=float, default=1965.0)
ap.add_argument("--tile-rows", type=int, default=0)
a = ap.parse_args()
c = CONFIGS[a.config]
with rotor.tuning(tile_rows=a.tile_rows):
    t = rotor.DpTable(config_menu(a.config), 1, c["M"])
assert t.kernel() == "tiles", t.kernel()
t.trace(True)
for _ in range(3):
    t.refill()
t.sync()
st, k, j = t.trace_read()
L, T = k.max() + 1, j.max() + 1
S = st.astype(np.float64).reshape(L, T, 6)
us = 1.0 / a.sm_mhz  # cycles -> us
g0 = (S[..., 0] - S[..., 0].min()) / 1e3
c0, bulk, comm, ready, tail = S[..., 1], S[..., 2], S[..., 3], S[..., 4], S[..., 5]
step = (tail - c0) * us
print(f"config {a.config}: L={L} tiles={T} span {(g0 + step).max():.1f} us (globaltimer + cycles)")
w_ready = (ready - bulk) * us           # warp 0 waits at READY after its bulk
comm_late = (comm - bulk) * us          # comm acquired after warp 0's bulk
after_comm = (ready - comm) * us        # READY passed after the comm warp arrived
print(f"mean per step (us): step {step.mean():.2f}  warp0 bulk {((bulk - c0) * us).mean():.2f}  "
      f"READY wait (warp 0) {w_ready.mean():.2f}  tail {((tail - ready) * us).mean():.2f}")
print(f"READY held by the comm warp (acquired after warp 0's bulk) in {(comm_late > 0).mean() * 100:.0f} % "
      f"of steps; READY passes {after_comm.mean():.2f} us after the comm warp arrives on average")
for kk in sorted({1, L // 8, L // 4, L // 2, 3 * L // 4, L - 2}):
    print(f"k={kk:3d}: step {step[kk].mean():6.2f}  bulk0 {((bulk - c0) * us)[kk].mean():5.2f}  "
          f"ready_wait {w_ready[kk].mean():5.2f}  comm_after_bulk0 {comm_late[kk].mean():6.2f}  "
          f"ready_after_comm {after_comm[kk].mean():5.2f}  tail {((tail - ready) * us)[kk].mean():5.2f}  "
          f"start j=0 {g0[kk, 0]:7.1f} j=T-1 {g0[kk, T - 1]:7.1f}")
