"""Python host mirror of the reference solver API, over librkr's C ABI.

Names, argument meaning and error behaviour follow namespace ``remat`` in
/root/reference/proj/include/remat/chain_dp.hpp:

    quantize / to_units            chain_dp.hpp:25-41
    DpArg                          chain_dp.hpp:44-47
    DpTable(menu, unit, m_max)     chain_dp.hpp:54-196   (filled on the GPU)
    build_schedule_rec(...)        chain_dp.hpp:211-246  (walked on the GPU)
    ChainSolution / solve_chain    chain_dp.hpp:248-296
    ValidationError / InfeasibleBudget   errors.hpp:14-16, :51-55

The C++ drop-in with the identical signatures is include/remat_b200/chain_dp.hpp;
this module is the same surface for Python callers, tests and bench.py.
All DP work runs in librkr.so on an sm_100 device.  There is no CPU
fallback: if the library or the device is missing, calls raise.
"""
from __future__ import annotations

import contextlib
import contextvars
import ctypes
import os
from dataclasses import dataclass, field
from typing import List, Optional, Sequence, Tuple

import numpy as np

from .menu import Menu, RkrMenu

K_INF_TIME = (2**63 - 1) // 4  # remat::kInfTime, chain_dp.hpp:23

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("RKR_LIB") or os.path.join(_HERE, "librkr.so")  # RKR_LIB: A/B tuning

RKR_OK, RKR_ERR_INVALID, RKR_ERR_INFEASIBLE, RKR_ERR_CUDA, RKR_ERR_OOM, RKR_ERR_CAPACITY, \
    RKR_ERR_ARGUMENT = range(7)


class ValidationError(RuntimeError):
    """remat::ValidationError (errors.hpp:14-16)."""


class InfeasibleBudget(RuntimeError):
    """remat::InfeasibleBudget (errors.hpp:51-55)."""

    def __init__(self, what: str, min_feasible_budget: int = -1):
        super().__init__(what)
        self.min_feasible_budget = min_feasible_budget


class DeviceError(RuntimeError):
    """CUDA failure, missing device or missing librkr.so (no CPU fallback)."""


class RkrOp(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int32), ("block", ctypes.c_int32), ("option", ctypes.c_int32)]


class RkrExec(ctypes.Structure):
    _fields_ = [("device", ctypes.c_int32), ("stream", ctypes.c_void_p), ("width", ctypes.c_int32),
                ("kernel", ctypes.c_int32), ("tune", ctypes.c_int32), ("tile_rows", ctypes.c_int32),
                ("reserved", ctypes.c_int32 * 2)]


_lib = None


def lib() -> ctypes.CDLL:
    """Load librkr.so (in-tree build).  Raises DeviceError if it is absent."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise DeviceError(f"librkr.so not built at {LIB_PATH}: run __graft_entry__.build()")
    L = ctypes.CDLL(LIB_PATH)
    i32, i64, p = ctypes.c_int32, ctypes.c_int64, ctypes.c_void_p
    P = ctypes.POINTER
    L.rkr_last_error.restype = ctypes.c_char_p
    L.rkr_abi_version.restype = i32
    L.rkr_device_ok.argtypes = [i32]
    L.rkr_device_ok.restype = i32
    L.rkr_quantize.argtypes = [i64, i32, P(i64), P(i64)]
    L.rkr_to_units.argtypes = [i64, i64]
    L.rkr_to_units.restype = i64
    L.rkr_table_create.argtypes = [P(RkrMenu), i64, i32, P(RkrExec), P(p)]
    L.rkr_table_destroy.argtypes = [p]
    L.rkr_table_destroy.restype = None
    for name, rt in (("rkr_table_length", i32), ("rkr_table_unit", i64), ("rkr_table_m_max", i32),
                     ("rkr_table_width", i32), ("rkr_table_kernel", i32)):
        getattr(L, name).argtypes = [p]
        getattr(L, name).restype = rt
    L.rkr_table_act_units.argtypes = [p, i32]
    L.rkr_table_act_units.restype = i64
    L.rkr_table_work_bound.argtypes = [p, P(i64), P(i64)]
    L.rkr_table_opt.argtypes = [p, i32, i32, i32, P(i64)]
    L.rkr_table_arg.argtypes = [p, i32, i32, i32, P(i32), P(i32)]
    L.rkr_table_row.argtypes = [p, i32, i32, p, p, p]
    L.rkr_table_download.argtypes = [p, p, p, p]
    L.rkr_backtrack.argtypes = [p, i32, i32, i32, P(RkrOp), i64, P(i64)]
    L.rkr_backtrack_menu.argtypes = [p, P(RkrMenu), i32, i32, i32, P(RkrOp), i64, P(i64)]
    L.rkr_first_feasible.argtypes = [p, i32, i32, P(i32)]
    L.rkr_solve_chain.argtypes = [P(RkrMenu), i64, i32, P(RkrExec), P(RkrOp), i64, P(i64), P(i64),
                                  P(i64), P(i32), P(i64)]
    L.rkr_table_sync.argtypes = [p]
    L.rkr_table_refill.argtypes = [p]
    L.rkr_table_refill_walk.argtypes = [p, i32, i32, i32]
    L.rkr_table_stream.argtypes = [p]
    L.rkr_table_stream.restype = p
    L.rkr_table_h2d_bytes.argtypes = [p]
    L.rkr_table_h2d_bytes.restype = i64
    L.rkr_table_device_bytes.argtypes = [p]
    L.rkr_table_device_bytes.restype = i64
    L.rkr_debug_trace.argtypes = [p, i32]
    L.rkr_debug_trace_items.argtypes = [p]
    L.rkr_debug_trace_items.restype = i64
    L.rkr_debug_trace_read.argtypes = [p, p, p, p]
    L.rkr_batch_create.argtypes = [P(P(RkrMenu)), P(i64), P(i32), i32, P(RkrExec), P(p)]
    L.rkr_batch_size.argtypes = [p]
    L.rkr_batch_size.restype = i32
    L.rkr_batch_table.argtypes = [p, i32]
    L.rkr_batch_table.restype = p
    L.rkr_batch_refill.argtypes = [p]
    L.rkr_batch_stream.argtypes = [p]
    L.rkr_batch_stream.restype = p
    L.rkr_batch_sync.argtypes = [p]
    L.rkr_batch_destroy.argtypes = [p]
    L.rkr_batch_destroy.restype = None
    L.rkr_sweep.argtypes = [P(RkrMenu), P(i64), i32, i32, P(RkrExec), P(i32), P(i64), P(i64), P(i32),
                            P(i64), P(RkrOp), i64, P(i64)]
    L.rkr_sweep_chains.argtypes = [P(P(RkrMenu)), P(i32), i32, P(i64), i32, P(RkrExec), P(i32),
                                   P(i64), P(i64), P(i32), P(i64), P(RkrOp), i64, P(i64)]
    L.rkr_sharded_create.argtypes = [P(RkrMenu), i64, i32, i32, P(i32), P(RkrExec), P(p)]
    L.rkr_sharded_count.argtypes = [p]
    L.rkr_sharded_count.restype = i32
    L.rkr_sharded_range.argtypes = [p, i32, P(i32), P(i32)]
    L.rkr_sharded_shard.argtypes = [p, i32]
    L.rkr_sharded_shard.restype = p
    L.rkr_sharded_refill.argtypes = [p]
    L.rkr_sharded_sync.argtypes = [p]
    L.rkr_sharded_opt.argtypes = [p, i32, i32, i32, P(i64)]
    L.rkr_sharded_row.argtypes = [p, i32, i32, p, p, p]
    L.rkr_sharded_backtrack.argtypes = [p, i32, i32, i32, P(RkrOp), i64, P(i64)]
    L.rkr_sharded_destroy.argtypes = [p]
    L.rkr_sharded_destroy.restype = None
    L.rkr_shard_create.argtypes = [P(RkrMenu), i64, i32, i32, i32, P(RkrExec), P(p)]
    L.rkr_shard_range.argtypes = [p, P(i32), P(i32)]
    L.rkr_shard_export.argtypes = [p, p, P(i64)]
    L.rkr_shard_link.argtypes = [p, p, P(i64)]
    L.rkr_shard_mirror.argtypes = [p, i32, p, P(i64)]
    L.rkr_shard_attach_mirror.argtypes = [p, p, P(i64)]
    L.rkr_shard_zero.argtypes = [p]
    L.rkr_shard_launch.argtypes = [p]
    L.rkr_shard_backtrack.argtypes = [p, i32, P(p), P(i64), i32, i32, i32, P(RkrOp), i64, P(i64)]
    L.rkr_replay.argtypes = [P(RkrMenu), P(RkrOp), i64, P(i64), P(i64), P(i64)]
    L.rkr_backtrack_async.argtypes = [p, i32, i32, i32]
    L.rkr_backtrack_fetch.argtypes = [p, P(RkrOp), i64, P(i64)]
    _lib = L
    return L


def _check(st: int, min_feasible: int = -1) -> None:
    if st == RKR_OK:
        return
    msg = lib().rkr_last_error().decode()
    if st == RKR_ERR_INVALID:
        raise ValidationError(msg)
    if st == RKR_ERR_INFEASIBLE:
        raise InfeasibleBudget(msg, min_feasible)
    if st == RKR_ERR_ARGUMENT:
        raise IndexError(msg)
    raise DeviceError(f"librkr status {st}: {msg}")


KERNELS = {"persistent": 0, "diagonal": 1, "queue": 2, "tiles": 3}

# rkr_exec.tune bits (include/rkr.h rkr_tune)
TUNE = {"no_tiles": 1 << 0, "jobs": 1 << 1, "comm_off": 1 << 2, "comm_on": 1 << 3,
        "split_off": 1 << 4, "split_on": 1 << 5, "stream": 1 << 6, "batch_queue": 1 << 7,
        "profile": 1 << 8, "wide_search": 1 << 9, "uniform": 1 << 10,
        "mixed": 1 << 11, "no_prune": 1 << 12}
_tuning: contextvars.ContextVar = contextvars.ContextVar("rkr_tuning", default=(0, 0))


@contextlib.contextmanager
def tuning(*flags: str, tile_rows: int = 0):
    """Kernel-variant overrides for every table created inside the block
    (rkr_exec.tune / tile_rows; A/B measurements and variant-pinning tests).
    Results are identical under every setting."""
    bits = 0
    for f in flags:
        bits |= TUNE[f]
    tok = _tuning.set((bits, tile_rows))
    try:
        yield
    finally:
        _tuning.reset(tok)


def _exec(device: int, width: str, stream: Optional[int] = None,
          kernel: str = "persistent") -> RkrExec:
    e = RkrExec()
    e.device = device
    e.stream = stream
    e.width = 64 if width == "64" else 0
    e.kernel = KERNELS[kernel]
    e.tune, e.tile_rows = _tuning.get()
    return e


@dataclass
class Quantization:
    unit: int = 1
    budget_units: int = 0


def quantize(budget_bytes: int, units: int) -> Quantization:
    u, b = ctypes.c_int64(), ctypes.c_int64()
    _check(lib().rkr_quantize(budget_bytes, units, ctypes.byref(u), ctypes.byref(b)))
    return Quantization(u.value, b.value)


def to_units(nbytes: int, unit: int) -> int:
    return lib().rkr_to_units(nbytes, unit)


@dataclass(frozen=True)
class DpArg:
    """remat::DpArg: kind None=0 / Option=1 / Cut=2, value = option id or cut index."""

    kind: int = 0
    value: int = -1

    NONE, OPTION, CUT = 0, 1, 2


# ScheduleOp kinds (types.hpp:346-362)
OP_COMPUTE, OP_FORGET, OP_BLOCK_FWD, OP_BLOCK_BWD = 0, 1, 2, 3


@dataclass(frozen=True)
class ScheduleOp:
    kind: int
    block: int
    target: str = ""
    option: int = -1


@dataclass
class Chain:
    """The id-bearing part of remat::Chain that build_schedule_rec reads:
    per block, the input dnode id and the loss cnode id."""

    input_ids: List[str]
    loss_ids: List[str]

    @staticmethod
    def skeleton(L: int) -> "Chain":
        return Chain([f"b{i}_in" for i in range(L)], [f"b{i}_loss" for i in range(L)])

    def length(self) -> int:
        return len(self.input_ids)


class DpTable:
    """remat::DpTable (chain_dp.hpp:54-196); cells live in device memory."""

    def __init__(self, menu: Menu, unit: int, m_max: int, device: int = 0, width: str = "auto",
                 stream: Optional[int] = None, kernel: str = "persistent"):
        self._lib = lib()
        self._h = ctypes.c_void_p()
        self._owned = True
        self._menu_struct = menu.struct()
        ex = _exec(device, width, stream, kernel)
        _check(self._lib.rkr_table_create(ctypes.byref(self._menu_struct), unit, m_max,
                                          ctypes.byref(ex), ctypes.byref(self._h)))
        self.menu = menu
        self._host: Optional[Tuple[np.ndarray, np.ndarray, np.ndarray]] = None

    @classmethod
    def _borrow(cls, handle, menu: Menu, owner) -> "DpTable":
        t = cls.__new__(cls)
        t._lib = lib()
        t._h = ctypes.c_void_p(handle)
        t._owned = False
        t._owner = owner  # keeps the batch alive
        t.menu = menu
        t._host = None
        return t

    def close(self) -> None:
        if self._h and self._owned:
            self._lib.rkr_table_destroy(self._h)
        self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    # accessors (chain_dp.hpp:103-116)
    def length(self) -> int:
        return self._lib.rkr_table_length(self._h)

    def unit(self) -> int:
        return self._lib.rkr_table_unit(self._h)

    def m_max(self) -> int:
        return self._lib.rkr_table_m_max(self._h)

    def act_units(self, i: int) -> int:
        return self._lib.rkr_table_act_units(self._h, i)

    def width(self) -> int:
        return self._lib.rkr_table_width(self._h)

    def kernel(self) -> str:
        """The fill kernel this table runs: "tiles", "queue" or "diagonal"."""
        k = self._lib.rkr_table_kernel(self._h)
        return {v: n for n, v in KERNELS.items()}[k]

    def sync(self) -> None:
        _check(self._lib.rkr_table_sync(self._h))

    # device-resident re-solve hooks (bench.py)
    def refill(self) -> None:
        """Enqueue the whole fill again from the device-resident menu (async)."""
        _check(self._lib.rkr_table_refill(self._h))

    def stream(self) -> int:
        return self._lib.rkr_table_stream(self._h) or 0

    def h2d_bytes(self) -> int:
        return self._lib.rkr_table_h2d_bytes(self._h)

    def device_bytes(self) -> int:
        return self._lib.rkr_table_device_bytes(self._h)

    def trace(self, enable: bool = True) -> None:
        """Record per-item timestamps on the next fills (persistent kernel)."""
        _check(self._lib.rkr_debug_trace(self._h, 1 if enable else 0))

    def trace_read(self):
        n = self._lib.rkr_debug_trace_items(self._h)
        st = np.zeros((n, 6), np.uint64)
        k = np.zeros(n, np.int32)
        j = np.zeros(n, np.int32)
        _check(self._lib.rkr_debug_trace_read(self._h, st.ctypes.data, k.ctypes.data, j.ctypes.data))
        return st, k, j

    def backtrack_async(self, s: int, t: int, m: int) -> None:
        _check(self._lib.rkr_backtrack_async(self._h, s, t, m))

    def refill_walk(self, s: int, t: int, m: int) -> None:
        """Refill and walk from (s, t, m) on the device (async; the walk is
        fused into the fill launch with the budget-tile kernel).  Collect the
        ops with backtrack_fetch()."""
        _check(self._lib.rkr_table_refill_walk(self._h, s, t, m))

    def backtrack_fetch(self, cap: int = 1 << 16) -> List[Tuple[int, int, int]]:
        buf = (RkrOp * cap)()
        n = ctypes.c_int64()
        _check(self._lib.rkr_backtrack_fetch(self._h, buf, cap, ctypes.byref(n)))
        return [(buf[i].kind, buf[i].block, buf[i].option) for i in range(n.value)]

    @property
    def max_candidates_per_cell(self) -> int:
        return self._work_bound()[0]

    @property
    def worst_cell_allowance(self) -> int:
        return self._work_bound()[1]

    def _work_bound(self) -> Tuple[int, int]:
        a, b = ctypes.c_int64(), ctypes.c_int64()
        _check(self._lib.rkr_table_work_bound(self._h, ctypes.byref(a), ctypes.byref(b)))
        return a.value, b.value

    def opt(self, s: int, t: int, m: int) -> int:
        if self._host is not None:
            return self._host_opt(s, t, m)
        v = ctypes.c_int64()
        _check(self._lib.rkr_table_opt(self._h, s, t, m, ctypes.byref(v)))
        return v.value

    def arg(self, s: int, t: int, m: int) -> DpArg:
        k, v = ctypes.c_int32(), ctypes.c_int32()
        _check(self._lib.rkr_table_arg(self._h, s, t, m, ctypes.byref(k), ctypes.byref(v)))
        return DpArg(k.value, v.value)

    def row(self, s: int, t: int) -> Tuple[np.ndarray, np.ndarray, np.ndarray]:
        W = self.m_max() + 1
        o = np.empty(W, np.int64)
        k = np.empty(W, np.int8)
        v = np.empty(W, np.int32)
        _check(self._lib.rkr_table_row(self._h, s, t, o.ctypes.data, k.ctypes.data, v.ctypes.data))
        return o, k, v

    def download(self) -> Tuple[np.ndarray, np.ndarray, np.ndarray]:
        """Whole table, rows in s-major triangular order, reference types."""
        L, W = self.length(), self.m_max() + 1
        rows = L * (L + 1) // 2
        o = np.empty((rows, W), np.int64)
        k = np.empty((rows, W), np.int8)
        v = np.empty((rows, W), np.int32)
        _check(self._lib.rkr_table_download(self._h, o.ctypes.data, k.ctypes.data, v.ctypes.data))
        self._host = (o, k, v)
        return o, k, v

    def _host_opt(self, s, t, m):
        if m < 0:
            return K_INF_TIME
        m = min(m, self.m_max())
        L = self.length()
        return int(self._host[0][s * L - s * (s - 1) // 2 + (t - s), m])

    def backtrack(self, s: int, t: int, m: int, menu: Optional[Menu] = None,
                  partial: Optional[list] = None) -> List[Tuple[int, int, int]]:
        """Raw device backtrack: (kind, block, option) triples.  menu: the
        caller's menu for the option lookups and pack shifts (as
        build_schedule_rec does, chain_dp.hpp:200-205, :228); default the
        table's own.  On an error, `partial` receives the ops emitted before it."""
        ms = menu.struct() if menu is not None else None
        cap = 4096
        while True:
            buf = (RkrOp * cap)()
            n = ctypes.c_int64()
            if ms is None:
                st = self._lib.rkr_backtrack(self._h, s, t, m, buf, cap, ctypes.byref(n))
            else:
                st = self._lib.rkr_backtrack_menu(self._h, ctypes.byref(ms), s, t, m, buf, cap,
                                                  ctypes.byref(n))
            if st == RKR_ERR_CAPACITY:
                cap = n.value
                continue
            ops = [(buf[i].kind, buf[i].block, buf[i].option) for i in range(min(n.value, cap))]
            if st != 0 and partial is not None:
                partial.extend(ops)
            _check(st)
            return ops

    def first_feasible(self, s: int, t: int) -> int:
        m = ctypes.c_int32()
        _check(self._lib.rkr_first_feasible(self._h, s, t, ctypes.byref(m)))
        return m.value


def _named(ops, chain: Chain) -> List[ScheduleOp]:
    out = []
    for k, b, o in ops:
        if k == OP_COMPUTE:
            out.append(ScheduleOp(k, b, chain.loss_ids[b], -1))
        elif k == OP_FORGET:
            out.append(ScheduleOp(k, b, chain.input_ids[b], -1))
        else:
            out.append(ScheduleOp(k, b, "", o))
    return out


def build_schedule_rec(table: DpTable, menu: Menu, chain: Chain, s: int, t: int, m: int,
                       out: Optional[list] = None) -> List[ScheduleOp]:
    """remat::build_schedule_rec (chain_dp.hpp:211-246), walked on the device
    with the caller's menu for the option lookups (ValidationError when it
    lacks a decided option; `out` then holds the ops emitted before)."""
    done: list = []
    try:
        ops = _named(table.backtrack(s, t, m, menu=menu, partial=done), chain)
    except Exception:
        if out is not None:
            out.extend(_named(done, chain))
        raise
    if out is not None:
        out.extend(ops)
    return ops


@dataclass
class ChainSolution:
    schedule: List[ScheduleOp] = field(default_factory=list)
    opt_time: int = 0
    unit: int = 1
    m_top: int = 0
    raw_ops: List[Tuple[int, int, int]] = field(default_factory=list)


def solve_chain(chain: Chain, menu: Menu, budget_bytes: int, units: int, device: int = 0,
                width: str = "auto") -> ChainSolution:
    """remat::solve_chain (chain_dp.hpp:255-296) in one C-ABI call."""
    L = lib()
    ms = menu.struct()
    ex = _exec(device, width)
    cap = max(4096, 4 * menu.L * menu.L)
    while True:
        buf = (RkrOp * cap)()
        n, ot, un, mf = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
        mt = ctypes.c_int32()
        st = L.rkr_solve_chain(ctypes.byref(ms), budget_bytes, units, ctypes.byref(ex), buf, cap,
                               ctypes.byref(n), ctypes.byref(ot), ctypes.byref(un), ctypes.byref(mt),
                               ctypes.byref(mf))
        if st == RKR_ERR_CAPACITY:
            cap = n.value
            continue
        _check(st, mf.value)
        raw = [(buf[i].kind, buf[i].block, buf[i].option) for i in range(n.value)]
        return ChainSolution(_named(raw, chain), ot.value, un.value, mt.value, raw)


class Batch:
    """Many independent DP tables filled by ONE persistent launch (rkr_batch_*)."""

    def __init__(self, menus: Sequence[Menu], units: Sequence[int], m_maxs: Sequence[int],
                 device: int = 0, width: str = "auto", stream: Optional[int] = None,
                 kernel: str = "persistent"):
        """kernel: "persistent" (budget-tile jobs when every table qualifies,
        else the row-segment queue) or "queue"."""
        self._lib = lib()
        n = len(menus)
        self._structs = [m.struct() for m in menus]
        arr = (ctypes.POINTER(RkrMenu) * n)(*[ctypes.pointer(x) for x in self._structs])
        u = (ctypes.c_int64 * n)(*units)
        mm = (ctypes.c_int32 * n)(*m_maxs)
        ex = _exec(device, width, stream, kernel)
        self._h = ctypes.c_void_p()
        _check(self._lib.rkr_batch_create(arr, u, mm, n, ctypes.byref(ex), ctypes.byref(self._h)))
        self.menus = list(menus)

    def __len__(self) -> int:
        return self._lib.rkr_batch_size(self._h)

    def table(self, i: int) -> DpTable:
        h = self._lib.rkr_batch_table(self._h, i)
        if not h:
            raise IndexError(i)
        return DpTable._borrow(h, self.menus[i], self)

    def refill(self) -> None:
        _check(self._lib.rkr_batch_refill(self._h))

    def stream(self) -> int:
        return self._lib.rkr_batch_stream(self._h) or 0

    def sync(self) -> None:
        _check(self._lib.rkr_batch_sync(self._h))

    def close(self) -> None:
        if self._h:
            self._lib.rkr_batch_destroy(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()


@dataclass
class SweepRow:
    budget: int
    feasible: bool
    opt_time: int = 0
    unit: int = 1
    m_top: int = 0
    min_feasible: int = -1
    ops: List[Tuple[int, int, int]] = field(default_factory=list)
    peak: int = -1        # replayed peak bytes (sweep() fills it)


def sweep_raw(menu: Menu, budgets: Sequence[int], units: int, device: int = 0,
              width: str = "auto") -> List[SweepRow]:
    """rkr_sweep: solve_chain for every budget (given order) in batched device calls."""
    L = lib()
    n = len(budgets)
    ms = menu.struct()
    ex = _exec(device, width)
    b = (ctypes.c_int64 * n)(*budgets)
    st = (ctypes.c_int32 * n)()
    ot = (ctypes.c_int64 * n)()
    un = (ctypes.c_int64 * n)()
    mt = (ctypes.c_int32 * n)()
    mf = (ctypes.c_int64 * n)()
    offs = (ctypes.c_int64 * (n + 1))()
    cap = max(1024, 8 * n * menu.L)
    while True:
        ops = (RkrOp * cap)()
        rc = L.rkr_sweep(ctypes.byref(ms), b, n, units, ctypes.byref(ex), st, ot, un, mt, mf, ops,
                         cap, offs)
        if rc == RKR_ERR_CAPACITY and offs[n] > cap:
            cap = offs[n]
            continue
        _check(rc)
        break
    rows = []
    for i in range(n):
        r = SweepRow(int(budgets[i]), st[i] == RKR_OK, ot[i], un[i], mt[i], mf[i])
        r.ops = [(ops[o].kind, ops[o].block, ops[o].option) for o in range(offs[i], offs[i + 1])]
        rows.append(r)
    return rows


def sweep_chains_raw(menus: Sequence[Menu], budgets: Sequence[Sequence[int]], units: int,
                     device: int = 0, width: str = "auto") -> List[List[SweepRow]]:
    """rkr_sweep_chains: sweep_raw for several chains in one batched device
    call (one fill launch); rows per chain, budgets in the given order."""
    L = lib()
    nc = len(menus)
    counts = [len(b) for b in budgets]
    flat = [int(x) for b in budgets for x in b]
    n = len(flat)
    structs = [m.struct() for m in menus]
    mp = (ctypes.POINTER(RkrMenu) * nc)(*[ctypes.pointer(x) for x in structs])
    nb = (ctypes.c_int32 * nc)(*counts)
    ex = _exec(device, width)
    b = (ctypes.c_int64 * n)(*flat)
    st = (ctypes.c_int32 * n)()
    ot = (ctypes.c_int64 * n)()
    un = (ctypes.c_int64 * n)()
    mt = (ctypes.c_int32 * n)()
    mf = (ctypes.c_int64 * n)()
    offs = (ctypes.c_int64 * (n + 1))()
    cap = max(1024, sum(8 * c * m.L for c, m in zip(counts, menus)))
    while True:
        ops = (RkrOp * cap)()
        rc = L.rkr_sweep_chains(mp, nb, nc, b, units, ctypes.byref(ex), st, ot, un, mt, mf, ops,
                                cap, offs)
        if rc == RKR_ERR_CAPACITY and offs[n] > cap:
            cap = offs[n]
            continue
        _check(rc)
        break
    out, i = [], 0
    for c in counts:
        rows = []
        for _ in range(c):
            r = SweepRow(flat[i], st[i] == RKR_OK, ot[i], un[i], mt[i], mf[i])
            r.ops = [(ops[o].kind, ops[o].block, ops[o].option) for o in range(offs[i], offs[i + 1])]
            rows.append(r)
            i += 1
        out.append(rows)
    return out


def sweep(menu: Menu, budgets: Sequence[int], units: int, device: int = 0,
          width: str = "auto", validate: bool = True) -> List[SweepRow]:
    """The reference's cmd_sweep loop (tools/remat.cpp:217-263) on the device:
    budgets sorted and de-duplicated, every solve batched, then the makespan
    monotonicity check of remat.cpp:256-263 (optimality implies it never rises
    with budget).  Every feasible schedule is replayed in the chain-level
    block-atomic model (rkr_replay) to report its peak.

    validate=True adds a self-check the reference does not make: the replayed
    makespan must equal the DP optimum and the peak must fit the budget.  (The
    reference's own gate, schedule_with_menu's simulate call at pipeline.hpp:
    200-203, replays the CD graphs of real blocks and only raises
    BudgetExceeded; synthetic menus have no CD graphs.)"""
    bs = sorted(set(int(x) for x in budgets))
    rows = sweep_raw(menu, bs, units, device, width)
    prev = K_INF_TIME
    for r in rows:
        if not r.feasible:
            continue
        r.peak, makespan = replay(menu, r.ops)
        if validate and makespan != r.opt_time:
            raise RuntimeError(f"replayed makespan {makespan} != DP optimum {r.opt_time}")
        if validate and r.peak > r.budget:
            raise RuntimeError(f"BudgetExceeded: peak {r.peak} > budget {r.budget}")
        if r.opt_time > prev:
            raise RuntimeError("sweep makespan increased with budget")
        prev = r.opt_time
    return rows


class ShardedTable:
    """One DP table split along the budget axis into shards (rkr_sharded_*):
    config 5.  Shards may live on one GPU or on several (peer memory)."""

    def __init__(self, menu: Menu, unit: int, m_max: int, n_shards: int,
                 devices: Optional[Sequence[int]] = None, width: str = "auto",
                 kernel: str = "persistent"):
        """kernel: "persistent" (budget-tile jobs when every shard qualifies,
        else the row-segment queue) or "queue"."""
        self._lib = lib()
        self._ms = menu.struct()
        ex = _exec(devices[0] if devices else 0, width, None, kernel)
        dv = (ctypes.c_int32 * n_shards)(*devices) if devices else None
        self._h = ctypes.c_void_p()
        _check(self._lib.rkr_sharded_create(ctypes.byref(self._ms), unit, m_max, n_shards, dv,
                                            ctypes.byref(ex), ctypes.byref(self._h)))
        self.menu = menu
        self.L = menu.L
        self.M = m_max

    def ranges(self) -> List[Tuple[int, int]]:
        out = []
        for i in range(self._lib.rkr_sharded_count(self._h)):
            lo, hi = ctypes.c_int32(), ctypes.c_int32()
            _check(self._lib.rkr_sharded_range(self._h, i, ctypes.byref(lo), ctypes.byref(hi)))
            out.append((lo.value, hi.value))
        return out

    def shard(self, i: int) -> DpTable:
        return DpTable._borrow(self._lib.rkr_sharded_shard(self._h, i), self.menu, self)

    def refill(self) -> None:
        _check(self._lib.rkr_sharded_refill(self._h))

    def sync(self) -> None:
        _check(self._lib.rkr_sharded_sync(self._h))

    def opt(self, s: int, t: int, m: int) -> int:
        v = ctypes.c_int64()
        _check(self._lib.rkr_sharded_opt(self._h, s, t, m, ctypes.byref(v)))
        return v.value

    def row(self, s: int, t: int):
        W = self.M + 1
        o = np.empty(W, np.int64)
        k = np.empty(W, np.int8)
        v = np.empty(W, np.int32)
        _check(self._lib.rkr_sharded_row(self._h, s, t, o.ctypes.data, k.ctypes.data,
                                         v.ctypes.data))
        return o, k, v

    def download(self):
        """Whole table (global slots), rows in s-major triangular order: every
        shard's local columns, side by side."""
        parts = [self.shard(i).download() for i in range(len(self.ranges()))]
        return tuple(np.ascontiguousarray(np.concatenate([p[i] for p in parts], axis=1))
                     for i in range(3))

    def backtrack(self, s: int, t: int, m: int) -> List[Tuple[int, int, int]]:
        cap = 4096
        while True:
            buf = (RkrOp * cap)()
            n = ctypes.c_int64()
            st = self._lib.rkr_sharded_backtrack(self._h, s, t, m, buf, cap, ctypes.byref(n))
            if st == RKR_ERR_CAPACITY:
                cap = n.value
                continue
            _check(st)
            return [(buf[i].kind, buf[i].block, buf[i].option) for i in range(n.value)]

    def close(self) -> None:
        if self._h:
            self._lib.rkr_sharded_destroy(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()


class ProcessShard:
    """Shard `rank` of a budget-sharded table built by one process per GPU
    (rkr_shard_*); neighbours exchange CUDA IPC handles through any host
    channel (bench.py and the tests use torch.distributed)."""

    def __init__(self, menu: Menu, unit: int, m_max: int, n_shards: int, rank: int,
                 device: int = 0, width: str = "auto"):
        self._lib = lib()
        self._ms = menu.struct()
        ex = _exec(device, width)
        self._h = ctypes.c_void_p()
        _check(self._lib.rkr_shard_create(ctypes.byref(self._ms), unit, m_max, n_shards, rank,
                                          ctypes.byref(ex), ctypes.byref(self._h)))
        self.menu, self.n, self.rank, self.M = menu, n_shards, rank, m_max
        self.table = DpTable._borrow(self._h.value, menu, self)

    def range(self) -> Tuple[int, int]:
        lo, hi = ctypes.c_int32(), ctypes.c_int32()
        _check(self._lib.rkr_shard_range(self._h, ctypes.byref(lo), ctypes.byref(hi)))
        return lo.value, hi.value

    def export(self) -> Tuple[bytes, List[int]]:
        hnd = ctypes.create_string_buffer(64)
        info = (ctypes.c_int64 * 8)()
        _check(self._lib.rkr_shard_export(self._h, hnd, info))
        return hnd.raw, list(info)

    def mirror(self) -> Tuple[bytes, List[int]]:
        """Shard 0: allocate and export the walk mirror (rkr_shard_mirror)."""
        hnd = ctypes.create_string_buffer(64)
        info = (ctypes.c_int64 * 8)()
        _check(self._lib.rkr_shard_mirror(self._h, self.M, hnd, info))
        return hnd.raw, list(info)

    def attach_mirror(self, handle: bytes, info: Sequence[int]) -> None:
        hnd = ctypes.create_string_buffer(handle, 64)
        inf = (ctypes.c_int64 * 8)(*info)
        _check(self._lib.rkr_shard_attach_mirror(self._h, hnd, inf))

    def link(self, next_handle: bytes, next_info: Sequence[int]) -> None:
        hnd = ctypes.create_string_buffer(next_handle, 64)
        info = (ctypes.c_int64 * 8)(*next_info)
        _check(self._lib.rkr_shard_link(self._h, hnd, info))

    def zero(self) -> None:
        _check(self._lib.rkr_shard_zero(self._h))

    def launch(self) -> None:
        _check(self._lib.rkr_shard_launch(self._h))

    def sync(self) -> None:
        self.table.sync()

    def backtrack(self, handles: Sequence[bytes], infos: Sequence[Sequence[int]], s: int, t: int,
                  m: int) -> List[Tuple[int, int, int]]:
        n = len(handles)
        bufs = [ctypes.create_string_buffer(h, 64) for h in handles]
        hp = (ctypes.c_void_p * n)(*[ctypes.cast(b, ctypes.c_void_p) for b in bufs])
        flat = (ctypes.c_int64 * (8 * n))(*[x for inf in infos for x in inf])
        cap = 4096
        while True:
            buf = (RkrOp * cap)()
            nn = ctypes.c_int64()
            st = self._lib.rkr_shard_backtrack(self._h, n, hp, flat, s, t, m, buf, cap,
                                               ctypes.byref(nn))
            if st == RKR_ERR_CAPACITY:
                cap = nn.value
                continue
            _check(st)
            return [(buf[i].kind, buf[i].block, buf[i].option) for i in range(nn.value)]

    def close(self) -> None:
        if self._h:
            self._lib.rkr_table_destroy(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def link_process_shards(shard: "ProcessShard", all_gather,
                        mirror: bool = True) -> Tuple[List[bytes], List[List[int]]]:
    """Exchange IPC handles with every rank (all_gather: obj -> list of objs)
    and link this shard to the next one; with `mirror`, shard 0's walk mirror
    is shared too, so the cross-shard walk reads local memory only.  Returns
    all handles and infos."""
    mine = shard.export()
    everyone = all_gather(mine)
    if shard.rank + 1 < shard.n:
        shard.link(*everyone[shard.rank + 1])
    if mirror and shard.n > 1:
        m0 = all_gather(shard.mirror() if shard.rank == 0 else None)[0]
        if shard.rank != 0:
            shard.attach_mirror(*m0)
    return [e[0] for e in everyone], [e[1] for e in everyone]


def replay(menu: Menu, ops: Sequence[Tuple[int, int, int]]) -> Tuple[int, int]:
    """Schedule validation gate (rkr_replay): (peak bytes, makespan) of a
    schedule in the DP's block-atomic memory model; raises ValidationError
    on a malformed schedule."""
    n = len(ops)
    arr = (RkrOp * max(n, 1))(*[RkrOp(*o) for o in ops])
    ms = menu.struct()
    pk, tm, bad = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
    _check(lib().rkr_replay(ctypes.byref(ms), arr, n, ctypes.byref(pk), ctypes.byref(tm),
                            ctypes.byref(bad)))
    return pk.value, tm.value
