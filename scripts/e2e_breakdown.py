"""Where the end-to-end time of one config-2 solve goes (host vs device)."""
import ctypes
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2307_01236_b200 import rotor  # noqa: E402
from paper_2307_01236_b200.menu import config_menu  # noqa: E402

menu = config_menu(2)
L, M = 33, 4096
budget = M + int(menu.act_sizes[0])
lib = rotor.lib()
chain = rotor.Chain.skeleton(L)
N = 50


def timeit(label, fn):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(N):
        fn()
    torch.cuda.synchronize()
    print(f"{label:45s} {1e6 * (time.perf_counter() - t0) / N:9.1f} us")


timeit("python rotor.solve_chain", lambda: rotor.solve_chain(chain, menu, budget, budget))
ms = menu.struct()
ex = rotor._exec(0, "auto")
cap = 4096
buf = (rotor.RkrOp * cap)()
n, ot, un, mf = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
mt = ctypes.c_int32()


def raw():
    st = lib.rkr_solve_chain(ctypes.byref(ms), budget, budget, ctypes.byref(ex), buf, cap,
                             ctypes.byref(n), ctypes.byref(ot), ctypes.byref(un), ctypes.byref(mt),
                             ctypes.byref(mf))
    assert st == 0


timeit("raw rkr_solve_chain (preallocated buffers)", raw)
timeit("menu.struct()", lambda: menu.struct())
timeit("RkrOp buffer 4*L*L", lambda: (rotor.RkrOp * (4 * L * L))())
h = ctypes.c_void_p()


def create_destroy():
    st = lib.rkr_table_create(ctypes.byref(ms), 1, M, ctypes.byref(ex), ctypes.byref(h))
    assert st == 0
    lib.rkr_table_sync(h)
    lib.rkr_table_destroy(h)


timeit("rkr_table_create + sync + destroy", create_destroy)
t = rotor.DpTable(menu, 1, M)


def refill_only():
    t.refill()
    t.sync()


timeit("refill + sync (device fill only)", refill_only)
timeit("backtrack (async + fetch)", lambda: t.backtrack(0, L - 1, M))
