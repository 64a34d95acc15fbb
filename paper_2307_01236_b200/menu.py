"""Option menus in the flat layout of ``include/rkr.h`` (``rkr_menu``).

A ``Menu`` is the Python image of ``remat::OptionMenu``
(/root/reference/proj/include/remat/chain_dp.hpp:16-21): per block, a list of
``BlockOption`` records (types.hpp:330-344) in menu order, plus the activation
sizes a_0..a_L.  It is stored CSR-style as numpy arrays so the same buffers can
be handed to librkr (product), and to the test-only checkers under oracle/.

Also here: the deterministic synthetic generator of SURVEY.md section 8(d)
(splitmix64, explicit draw order) that bench.py and the tests use, and the
reference's worked two-block example (test_helpers.hpp:64-82).
"""
from __future__ import annotations

import ctypes
import json
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

_MASK = (1 << 64) - 1


class RkrMenu(ctypes.Structure):
    """ctypes mirror of ``rkr_menu`` (include/rkr.h)."""

    _fields_ = [
        ("n_blocks", ctypes.c_int32),
        ("option_offsets", ctypes.POINTER(ctypes.c_int32)),
        ("option_id", ctypes.POINTER(ctypes.c_int32)),
        ("time_fwd", ctypes.POINTER(ctypes.c_int64)),
        ("time_bwd", ctypes.POINTER(ctypes.c_int64)),
        ("has_bwd", ctypes.POINTER(ctypes.c_uint8)),
        ("save_mem", ctypes.POINTER(ctypes.c_int64)),
        ("peak_fwd", ctypes.POINTER(ctypes.c_int64)),
        ("peak_fwd_pre", ctypes.POINTER(ctypes.c_int64)),
        ("peak_bwd", ctypes.POINTER(ctypes.c_int64)),
        ("act_sizes", ctypes.POINTER(ctypes.c_int64)),
    ]


@dataclass
class BlockOption:
    """remat::BlockOption (types.hpp:330-344), DP-relevant fields only."""

    option_id: int
    time_fwd: int
    time_bwd: Optional[int]
    save_mem: int
    peak_fwd: int
    peak_fwd_pre: int
    peak_bwd: int = 0


_FIELDS64 = ("time_fwd", "time_bwd", "save_mem", "peak_fwd", "peak_fwd_pre", "peak_bwd")


@dataclass
class Menu:
    option_offsets: np.ndarray  # int32 [L+1]
    option_id: np.ndarray  # int32 [n]
    time_fwd: np.ndarray  # int64 [n]
    time_bwd: np.ndarray  # int64 [n]
    has_bwd: np.ndarray  # uint8 [n]
    save_mem: np.ndarray
    peak_fwd: np.ndarray
    peak_fwd_pre: np.ndarray
    peak_bwd: np.ndarray
    act_sizes: np.ndarray  # int64 [L+1]
    _keep: list = field(default_factory=list, repr=False, compare=False)

    # ---- construction -----------------------------------------------------
    @staticmethod
    def from_options(options: Sequence[Sequence[BlockOption]], act_sizes: Sequence[int]) -> "Menu":
        offs = [0]
        rows = []
        for blk in options:
            rows.extend(blk)
            offs.append(len(rows))
        n = len(rows)

        def col(name, dt):
            return np.array([getattr(o, name) or 0 for o in rows], dtype=dt).reshape(n)

        return Menu(
            option_offsets=np.array(offs, dtype=np.int32),
            option_id=col("option_id", np.int32),
            time_fwd=col("time_fwd", np.int64),
            time_bwd=np.array([o.time_bwd if o.time_bwd is not None else 0 for o in rows], dtype=np.int64),
            has_bwd=np.array([1 if o.time_bwd is not None else 0 for o in rows], dtype=np.uint8),
            save_mem=col("save_mem", np.int64),
            peak_fwd=col("peak_fwd", np.int64),
            peak_fwd_pre=col("peak_fwd_pre", np.int64),
            peak_bwd=col("peak_bwd", np.int64),
            act_sizes=np.array(act_sizes, dtype=np.int64),
        )

    @property
    def L(self) -> int:
        return int(len(self.option_offsets) - 1)

    def length(self) -> int:
        return self.L

    def options(self, block: int) -> List[BlockOption]:
        out = []
        for o in range(int(self.option_offsets[block]), int(self.option_offsets[block + 1])):
            out.append(
                BlockOption(
                    int(self.option_id[o]),
                    int(self.time_fwd[o]),
                    int(self.time_bwd[o]) if self.has_bwd[o] else None,
                    int(self.save_mem[o]),
                    int(self.peak_fwd[o]),
                    int(self.peak_fwd_pre[o]),
                    int(self.peak_bwd[o]),
                )
            )
        return out

    def n_saved(self) -> np.ndarray:
        blk = np.repeat(np.arange(self.L), np.diff(self.option_offsets))
        return np.bincount(blk[self.option_id != 0], minlength=self.L)

    def struct(self) -> RkrMenu:
        """A ctypes ``rkr_menu`` pointing at this menu's (contiguous) arrays."""
        arrs = {
            "option_offsets": np.ascontiguousarray(self.option_offsets, dtype=np.int32),
            "option_id": np.ascontiguousarray(self.option_id, dtype=np.int32),
            "has_bwd": np.ascontiguousarray(self.has_bwd, dtype=np.uint8),
            "act_sizes": np.ascontiguousarray(self.act_sizes, dtype=np.int64),
        }
        for f in _FIELDS64:
            arrs[f] = np.ascontiguousarray(getattr(self, f), dtype=np.int64)
        self._keep = list(arrs.values())
        ptr = lambda a, t: a.ctypes.data_as(ctypes.POINTER(t))  # noqa: E731
        return RkrMenu(
            self.L,
            ptr(arrs["option_offsets"], ctypes.c_int32),
            ptr(arrs["option_id"], ctypes.c_int32),
            ptr(arrs["time_fwd"], ctypes.c_int64),
            ptr(arrs["time_bwd"], ctypes.c_int64),
            ptr(arrs["has_bwd"], ctypes.c_uint8),
            ptr(arrs["save_mem"], ctypes.c_int64),
            ptr(arrs["peak_fwd"], ctypes.c_int64),
            ptr(arrs["peak_fwd_pre"], ctypes.c_int64),
            ptr(arrs["peak_bwd"], ctypes.c_int64),
            ptr(arrs["act_sizes"], ctypes.c_int64),
        )

    # ---- fixtures -----------------------------------------------------------
    def to_json(self) -> dict:
        d = {k: getattr(self, k).tolist() for k in
             ("option_offsets", "option_id", "time_fwd", "time_bwd", "has_bwd", "save_mem",
              "peak_fwd", "peak_fwd_pre", "peak_bwd", "act_sizes")}
        return d

    @staticmethod
    def from_json(d: dict) -> "Menu":
        return Menu(
            option_offsets=np.array(d["option_offsets"], dtype=np.int32),
            option_id=np.array(d["option_id"], dtype=np.int32),
            time_fwd=np.array(d["time_fwd"], dtype=np.int64),
            time_bwd=np.array(d["time_bwd"], dtype=np.int64),
            has_bwd=np.array(d["has_bwd"], dtype=np.uint8),
            save_mem=np.array(d["save_mem"], dtype=np.int64),
            peak_fwd=np.array(d["peak_fwd"], dtype=np.int64),
            peak_fwd_pre=np.array(d["peak_fwd_pre"], dtype=np.int64),
            peak_bwd=np.array(d["peak_bwd"], dtype=np.int64),
            act_sizes=np.array(d["act_sizes"], dtype=np.int64),
        )

    def dumps(self) -> str:
        return json.dumps(self.to_json())


# ---------------------------------------------------------------------------
# The reference's worked example: tiny_chain_menu (test_helpers.hpp:64-82)
# ---------------------------------------------------------------------------
def tiny_chain_menu() -> Menu:
    def opt(i, ef, eb, save, pf, pre, pb):
        return BlockOption(i, ef, eb if i != 0 else None, save, pf, pre, pb)

    return Menu.from_options(
        [
            [opt(0, 10, 0, 4, 8, 8, 0), opt(1, 10, 12, 10, 10, 10, 14)],
            [opt(0, 8, 0, 4, 6, 6, 0), opt(1, 8, 9, 8, 8, 8, 10)],
        ],
        [4, 4, 2],
    )


# ---------------------------------------------------------------------------
# Synthetic chains
# ---------------------------------------------------------------------------
class SplitMix64:
    def __init__(self, seed: int):
        self.state = seed & _MASK

    def next(self) -> int:
        self.state = (self.state + 0x9E3779B97F4A7C15) & _MASK
        z = self.state
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _MASK
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _MASK
        return z ^ (z >> 31)

    def u(self, lo: int, hi: int) -> int:
        return lo + self.next() % (hi - lo + 1)


def synthetic_menu(L: int, B: int, M: int, seed: int, tie_stress: bool = False,
                   byte_scale: int = 1) -> Menu:
    """Deterministic chain of L blocks with B saved options each, sized so the
    first feasible budget is a few percent of M and M itself is ample.

    Draw order (fixed, documented in DESIGN.md): a_0..a_L; then per block:
    option 0 (time_fwd, peak extra), then options 1..B (time_fwd extra,
    time_bwd, save extra, peak extra, peak_fwd_pre, peak_bwd extra).
    ``tie_stress`` draws times in [1, 9] (frequent argmin ties).
    ``byte_scale`` > 1 turns unit sizes into byte sizes: x -> x*byte_scale + u(0, byte_scale-1)
    (so quantization by solve_chain is non-trivial).
    """
    r = SplitMix64(seed)
    a = max(1, M // (2 * L))
    act = [r.u(a // 2 + 1, 3 * a // 2 + 1) for _ in range(L + 1)]
    blocks = []
    for i in range(L):
        a_in, a_out = act[i], act[i + 1]
        if tie_stress:
            tf0 = r.u(1, 5)
        else:
            tf0 = r.u(50, 500)
        pf0 = a_in + a_out + r.u(0, a)
        opts = [BlockOption(0, tf0, None, a_in, pf0, pf0, 0)]
        for o in range(1, B + 1):
            if tie_stress:
                tf = tf0 + r.u(0, 4)
                tb = r.u(1, 9)
            else:
                tf = tf0 + r.u(0, 100)
                tb = r.u(100, 1000)
            save = a_in + a_out + r.u(0, 3 * a)
            pf = max(save, pf0) + r.u(0, a)
            pre = r.u(max(save, pf - a_out), pf)
            pb = save + a_out + r.u(0, a)
            opts.append(BlockOption(o, tf, tb, save, pf, pre, pb))
        blocks.append(opts)
    menu = Menu.from_options(blocks, act)
    if byte_scale > 1:
        for f in ("save_mem", "peak_fwd", "peak_fwd_pre", "peak_bwd"):
            v = getattr(menu, f)
            setattr(menu, f, v * byte_scale + np.array(
                [r.u(0, byte_scale - 1) for _ in range(len(v))], dtype=np.int64))
        menu.act_sizes = menu.act_sizes * byte_scale + np.array(
            [r.u(0, byte_scale - 1) for _ in range(L + 1)], dtype=np.int64)
    return menu


# BASELINE.json configs.  seed = 42 + config index.
CONFIGS = {
    1: dict(name="gpt2-small-like", L=24, B=8, M=500),
    2: dict(name="resnet101-like", L=33, B=16, M=4096),
    3: dict(name="gpt2-xl-like", L=96, B=32, M=16384),
    5: dict(name="synthetic-1024", L=1024, B=64, M=65536),
}


def config_menu(idx: int, tie_stress: bool = False) -> Menu:
    c = CONFIGS[idx]
    return synthetic_menu(c["L"], c["B"], c["M"], seed=42 + idx, tie_stress=tie_stress)
