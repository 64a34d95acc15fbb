"""Who holds the READY barrier of the K1t fill: the communication warp
(waiting for the lower tiles' diagonal k-1) or the compute warps (their
bulk)?  Per (diagonal, tile) stamps: t0 step start (warp 0), t1 warp 0's bulk
done, c the comm warp's acquisition of k-1, t2 READY passed (warp 0), t3
tail done.

    python scripts/trace_ready.py --config 3
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
base = st[:, 0].min()
L, T = k.max() + 1, j.max() + 1
S = ((st - base) / 1e3).reshape(L, T, 6)
t0, comm, t1, t2, t3 = S[..., 0], S[..., 1], S[..., 2], S[..., 3], S[..., 4]
step = t3 - t0
ready_wait = t2 - t1                     # warp 0: bulk done -> READY passed
after_comm = t2 - comm                   # READY passed after the comm warp arrived
comm_late = comm - t1                    # comm acquired after warp 0's bulk
print(f"config {a.config}: L={L} tiles={T} span {S[..., 4].max():.1f} us")
print(f"mean per step (us): step {step.mean():.2f}  warp0 bulk {(t1 - t0).mean():.2f}  "
      f"READY wait (warp 0) {ready_wait.mean():.2f}  tail {(t3 - t2).mean():.2f}")
print(f"READY passed after the comm warp's acquisition by {after_comm.mean():.2f} us on average; "
      f"comm warp later than warp 0's bulk in {(comm_late > 0.05).mean() * 100:.0f} % of steps "
      f"(by {np.clip(comm_late, 0, None).mean():.2f} us on average)")
for kk in [1, L // 8, L // 4, L // 2, 3 * L // 4, L - 2]:
    print(f"k={kk:3d}: step {step[kk].mean():6.2f}  bulk0 {(t1 - t0)[kk].mean():6.2f}  "
          f"ready_wait {ready_wait[kk].mean():5.2f}  comm_after_bulk0 {comm_late[kk].mean():6.2f}  "
          f"ready_after_comm {after_comm[kk].mean():5.2f}  tail {(t3 - t2)[kk].mean():5.2f}")
