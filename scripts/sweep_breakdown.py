"""Where the end-to-end time of one config-4 rkr_sweep call goes (per chain)."""
import ctypes
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

sys.argv = sys.argv[:1]
import bench  # noqa: E402
from paper_2307_01236_b200 import rotor  # noqa: E402
from paper_2307_01236_b200.sweep import SWEEP_UNITS  # noqa: E402

menus, rows = bench.sweep_instances()
lib = rotor.lib()
ex = rotor._exec(0, "auto")
for ci in sorted(set(r[1] for r in rows)):
    rs = [r for r in rows if r[1] == ci and r[4] >= 0]
    bs = [r[2] for r in rs]
    n = len(bs)
    m = menus[ci]
    t0 = time.perf_counter()
    b = rotor.Batch([m] * n, [r[3] for r in rs], [r[4] for r in rs])
    b.sync() if hasattr(b, "sync") else torch.cuda.synchronize()
    t1 = time.perf_counter()
    b.refill()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    b.close()
    t3 = time.perf_counter()
    cap = max(1024, 8 * n * m.L)
    args = (ctypes.byref(m.struct()), (ctypes.c_int64 * n)(*bs), n, SWEEP_UNITS, ctypes.byref(ex),
            (ctypes.c_int32 * n)(), (ctypes.c_int64 * n)(), (ctypes.c_int64 * n)(),
            (ctypes.c_int32 * n)(), (ctypes.c_int64 * n)(), (rotor.RkrOp * cap)(), cap,
            (ctypes.c_int64 * (n + 1))())
    ms = m.struct()
    for _ in range(2):
        t4 = time.perf_counter()
        assert lib.rkr_sweep(ctypes.byref(ms), *args[1:]) == 0
        t5 = time.perf_counter()
    print(f"chain {ci} L={m.L} n={n}: batch create+fill {1e3*(t1-t0):.1f} ms, refill {1e3*(t2-t1):.1f} ms, "
          f"destroy {1e3*(t3-t2):.1f} ms, rkr_sweep {1e3*(t5-t4):.1f} ms")
