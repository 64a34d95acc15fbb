"""ctypes bindings for the test-only checkers (C restatement and reference shim)."""
from __future__ import annotations

import ctypes
import os
import subprocess
from typing import List, Tuple

import numpy as np

from paper_2307_01236_b200.menu import Menu, RkrMenu

HERE = os.path.dirname(os.path.abspath(__file__))
ORC_PATH = os.path.join(HERE, "liborc.so")
REF_PATH = os.path.join(HERE, "_ref", "libremat_ref.so")

i32, i64, p = ctypes.c_int32, ctypes.c_int64, ctypes.c_void_p
P = ctypes.POINTER


def build() -> None:
    """make -f oracle/Makefile (the reference shim only where /root/reference exists)."""
    subprocess.run(["make", "-s", "-f", os.path.join(HERE, "Makefile")], check=True)


def _tri_rows(L: int) -> int:
    return L * (L + 1) // 2


class _Base:
    prefix = ""

    def __init__(self, path: str):
        self.lib = ctypes.CDLL(path)
        f = lambda n: getattr(self.lib, self.prefix + n)  # noqa: E731
        f("last_error").restype = ctypes.c_char_p
        f("quantize").argtypes = [i64, i32, P(i64), P(i64)]
        f("table_fill").argtypes = [P(RkrMenu), i64, i32, p, p, p, P(i64), P(i64)]
        f("build_schedule").restype = i32
        f("solve_chain").argtypes = [P(RkrMenu), i64, i32, P(i32), i64, P(i64), P(i64), P(i64),
                                     P(i32), P(i64)]
        self.f = f

    def err(self) -> str:
        return self.f("last_error")().decode()

    def quantize(self, budget: int, units: int) -> Tuple[int, int, int]:
        u, b = i64(), i64()
        st = self.f("quantize")(budget, units, ctypes.byref(u), ctypes.byref(b))
        return st, u.value, b.value

    def fill(self, menu: Menu, unit: int, M: int):
        """Returns (status, opt[rows, M+1] int64, kind int8, value int32, max_cands, worst_allow)."""
        rows = _tri_rows(menu.L)
        o = np.empty((rows, M + 1), np.int64)
        k = np.empty((rows, M + 1), np.int8)
        v = np.empty((rows, M + 1), np.int32)
        mc, wa = i64(), i64()
        ms = menu.struct()
        st = self.f("table_fill")(ctypes.byref(ms), unit, M, o.ctypes.data, k.ctypes.data,
                                  v.ctypes.data, ctypes.byref(mc), ctypes.byref(wa))
        return st, o, k, v, mc.value, wa.value

    def solve_chain(self, menu: Menu, budget: int, units: int):
        """Returns (status, ops, opt_time, unit, m_top, min_feasible)."""
        cap = max(4096, 8 * menu.L * menu.L)
        ops = np.zeros(3 * cap, np.int32)
        n, ot, un, mf = i64(), i64(), i64(), i64()
        mt = i32()
        ms = menu.struct()
        st = self.f("solve_chain")(ctypes.byref(ms), budget, units,
                                   ops.ctypes.data_as(P(i32)), cap, ctypes.byref(n),
                                   ctypes.byref(ot), ctypes.byref(un), ctypes.byref(mt),
                                   ctypes.byref(mf))
        trip = [tuple(int(x) for x in ops[3 * i:3 * i + 3]) for i in range(min(n.value, cap))]
        return st, trip, ot.value, un.value, mt.value, mf.value


class Orc(_Base):
    """The C restatement (oracle/rotor_oracle.c)."""

    prefix = "orc_"

    def __init__(self, path: str = ORC_PATH):
        super().__init__(path)
        self.lib.orc_build_schedule.argtypes = [P(RkrMenu), i64, i32, p, p, p, i32, i32, i32,
                                                P(i32), i64, P(i64)]
        self.lib.orc_atomic_replay.argtypes = [P(RkrMenu), P(i32), i64, P(i64)]
        self.lib.orc_atomic_replay.restype = i64

    def build_schedule(self, menu: Menu, unit: int, M: int, tables, s: int, t: int, m: int):
        o, k, v = tables
        cap = max(4096, 8 * menu.L * menu.L)
        ops = np.zeros(3 * cap, np.int32)
        n = i64()
        ms = menu.struct()
        st = self.lib.orc_build_schedule(ctypes.byref(ms), unit, M, o.ctypes.data, k.ctypes.data,
                                         v.ctypes.data, s, t, m, ops.ctypes.data_as(P(i32)), cap,
                                         ctypes.byref(n))
        trip = [tuple(int(x) for x in ops[3 * i:3 * i + 3]) for i in range(min(n.value, cap))]
        return st, trip

    def atomic_replay(self, menu: Menu, ops: List[Tuple[int, int, int]]) -> Tuple[int, int]:
        arr = np.array(ops, dtype=np.int32).reshape(-1)
        tm = i64()
        ms = menu.struct()
        peak = self.lib.orc_atomic_replay(ctypes.byref(ms), arr.ctypes.data_as(P(i32)), len(ops),
                                          ctypes.byref(tm))
        return peak, tm.value


class Ref(_Base):
    """The unmodified reference behind oracle/ref_driver.cpp."""

    prefix = "ref_"

    def __init__(self, path: str = REF_PATH):
        super().__init__(path)
        L = self.lib
        L.ref_build_schedule.argtypes = [P(RkrMenu), i64, i32, i32, i32, i32, P(i32), i64, P(i64)]
        L.ref_table_bench.argtypes = [P(RkrMenu), i64, i32, i32, P(i64)]
        L.ref_table_bench.restype = ctypes.c_double
        L.ref_solve_bench.argtypes = [P(RkrMenu), i64, i32, i32, P(i64), P(i64), P(i32), P(i32)]
        L.ref_solve_bench.restype = ctypes.c_double
        L.ref_fill_and_walk.argtypes = [P(RkrMenu), i64, i32, p, p, p, P(i64), i32, P(i32), P(i32),
                                        P(i32), i64, P(i64)]
        L.ref_fill_and_walk.restype = i32
        L.ref_rng_new.argtypes = [ctypes.c_uint32]
        L.ref_rng_new.restype = p
        L.ref_rng_free.argtypes = [p]
        L.ref_random_menu.argtypes = [p, i32, i32, i32, i32] + [p] * 10
        L.ref_random_menu.restype = i32
        L.ref_chain_oracle.argtypes = [P(RkrMenu), i64]
        L.ref_chain_oracle.restype = i64
        L.ref_chain_oracle_dijkstra.argtypes = [P(RkrMenu), i64, i32]
        L.ref_chain_oracle_dijkstra.restype = i64
        L.ref_atomic_replay.argtypes = [P(RkrMenu), P(i32), i64, P(i64)]
        L.ref_atomic_replay.restype = i64

    def build_schedule(self, menu: Menu, unit: int, M: int, s: int, t: int, m: int):
        cap = max(4096, 8 * menu.L * menu.L)
        ops = np.zeros(3 * cap, np.int32)
        n = i64()
        ms = menu.struct()
        st = self.lib.ref_build_schedule(ctypes.byref(ms), unit, M, s, t, m,
                                         ops.ctypes.data_as(P(i32)), cap, ctypes.byref(n))
        trip = [tuple(int(x) for x in ops[3 * i:3 * i + 3]) for i in range(max(0, min(n.value, cap)))]
        return st, trip

    def table_bench(self, menu: Menu, unit: int, M: int, threads: int = 1) -> Tuple[float, int]:
        top = i64()
        ms = menu.struct()
        secs = self.lib.ref_table_bench(ctypes.byref(ms), unit, M, threads, ctypes.byref(top))
        return secs, top.value

    def solve_bench(self, menu: Menu, budget: int, units: int, threads: int = 1):
        """remat::solve_chain (fill + top cell + build_schedule_rec) on `threads`
        concurrent host threads; returns (seconds of the slowest, status,
        opt_time, n_ops, m_top) of thread 0."""
        ot, no, mt, st = i64(), i64(), i32(), i32()
        ms = menu.struct()
        secs = self.lib.ref_solve_bench(ctypes.byref(ms), budget, units, threads, ctypes.byref(ot),
                                        ctypes.byref(no), ctypes.byref(mt), ctypes.byref(st))
        return secs, st.value, ot.value, no.value, mt.value

    def fill_and_walk(self, menu: Menu, unit: int, M: int, cells, want_table: bool = True):
        """One reference DpTable and build_schedule_rec from every (s, t, m) in
        `cells`.  Returns (status, (opt, kind, value) or None, max_cands,
        [(walk status, ops)])."""
        rows = _tri_rows(menu.L)
        if want_table:
            o = np.empty((rows, M + 1), np.int64)
            k = np.empty((rows, M + 1), np.int8)
            v = np.empty((rows, M + 1), np.int32)
            tp = (o.ctypes.data, k.ctypes.data, v.ctypes.data)
        else:
            o = k = v = None
            tp = (None, None, None)
        n = len(cells)
        stm = np.array(cells, np.int32).reshape(-1)
        wst = np.zeros(max(n, 1), np.int32)
        cap = max(4096, 8 * menu.L * menu.L) * max(n, 1)
        ops = np.zeros(3 * cap, np.int32)
        off = np.zeros(n + 1, np.int64)
        mc = i64()
        ms = menu.struct()
        st = self.lib.ref_fill_and_walk(ctypes.byref(ms), unit, M, *tp, ctypes.byref(mc), n,
                                        stm.ctypes.data_as(P(i32)), wst.ctypes.data_as(P(i32)),
                                        ops.ctypes.data_as(P(i32)), cap,
                                        off.ctypes.data_as(P(i64)))
        walks = []
        for i in range(n):
            a, b = int(off[i]), int(off[i + 1])
            walks.append((int(wst[i]), [tuple(int(x) for x in ops[3 * q:3 * q + 3]) for q in range(a, b)]))
        return st, ((o, k, v) if want_table else None), mc.value, walks

    def random_menus(self, seed: int, count: int, max_blocks: int, max_options: int) -> List[Menu]:
        """Successive testing::random_menu(rng, max_blocks, max_options) draws from
        std::mt19937(seed), as the reference's property tests do."""
        rng = self.lib.ref_rng_new(seed)
        out = []
        try:
            for _ in range(count):
                cb, co = max_blocks, max_blocks * (max_options + 1)
                offs = np.zeros(cb + 1, np.int32)
                ids = np.zeros(co, np.int32)
                a64 = [np.zeros(co, np.int64) for _ in range(6)]
                hb = np.zeros(co, np.uint8)
                act = np.zeros(cb + 1, np.int64)
                L = self.lib.ref_random_menu(rng, max_blocks, max_options, cb, co, offs.ctypes.data,
                                             ids.ctypes.data, a64[0].ctypes.data, a64[1].ctypes.data,
                                             hb.ctypes.data, a64[2].ctypes.data, a64[3].ctypes.data,
                                             a64[4].ctypes.data, a64[5].ctypes.data, act.ctypes.data)
                assert L > 0
                n = int(offs[L])
                out.append(Menu(offs[:L + 1].copy(), ids[:n].copy(), a64[0][:n].copy(),
                                a64[1][:n].copy(), hb[:n].copy(), a64[2][:n].copy(),
                                a64[3][:n].copy(), a64[4][:n].copy(), a64[5][:n].copy(),
                                act[:L + 1].copy()))
        finally:
            self.lib.ref_rng_free(rng)
        return out

    def chain_oracle(self, menu: Menu, budget_units: int) -> int:
        ms = menu.struct()
        return self.lib.ref_chain_oracle(ctypes.byref(ms), budget_units)

    def chain_oracle_dijkstra(self, menu: Menu, budget_units: int, fwd_cap: int) -> int:
        ms = menu.struct()
        return self.lib.ref_chain_oracle_dijkstra(ctypes.byref(ms), budget_units, fwd_cap)

    def atomic_replay(self, menu: Menu, ops) -> Tuple[int, int]:
        arr = np.array(ops, dtype=np.int32).reshape(-1)
        tm = i64()
        ms = menu.struct()
        peak = self.lib.ref_atomic_replay(ctypes.byref(ms), arr.ctypes.data_as(P(i32)), len(ops),
                                          ctypes.byref(tm))
        return peak, tm.value


HAVE_ORC = os.path.exists(ORC_PATH)
HAVE_REF = os.path.exists(REF_PATH)
