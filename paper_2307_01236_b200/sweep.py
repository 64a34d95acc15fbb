"""Host-side sweep helpers: budget grids, the no-recompute ceiling, the
BASELINE config-4 workload and the instance partition across GPUs.

Nothing here computes DP cells; the solves go through rotor.sweep / rkr_sweep.
"""
from __future__ import annotations

import heapq
from dataclasses import dataclass
from typing import List, Sequence, Tuple

from .menu import Menu, synthetic_menu


def even_spacing(lo: int, hi: int, n: int) -> List[int]:
    """Evenly spaced inclusive integer range, duplicates dropped; a single
    point (or an empty range) takes the upper endpoint.  Same arithmetic as
    remat::even_spacing (/root/reference/proj/include/remat/ilp_model.hpp:462-469)."""
    if n <= 1 or lo >= hi:
        return [hi]
    out: List[int] = []
    for i in range(n):
        v = lo + (hi - lo) * i // (n - 1)
        if not out or out[-1] != v:
            out.append(v)
    return out


def one_pass_peak(menu: Menu) -> int:
    """Peak bytes of the one-pass, no-recomputation schedule that runs every
    block with its fastest saved option -- the chain-level counterpart of
    remat::chain_max_peak (pipeline.hpp:251-274), evaluated in the
    block-atomic memory model the DP itself uses (a block's forward holds its
    input, output and pack; its backward releases the pack, the output and
    the incoming gradient and creates the input gradient)."""
    L = menu.L
    a = [int(x) for x in menu.act_sizes]
    pick = []
    for b in range(L):
        best = None
        for o in menu.options(b):
            if o.time_bwd is None:
                continue
            if best is None or o.time_fwd + o.time_bwd < best.time_fwd + best.time_bwd:
                best = o
        if best is None:
            raise ValueError(f"block {b} has no saved option")
        pick.append(best)
    cur = a[0]
    peak = cur
    for b, o in enumerate(pick):  # forwards, outputs kept, packs kept
        peak = max(peak, cur + o.peak_fwd - a[b])
        cur += a[b + 1] + (o.save_mem - a[b] - a[b + 1])
        peak = max(peak, cur)
    cur += a[L]  # loss gradient
    peak = max(peak, cur)
    for b in range(L - 1, -1, -1):
        o = pick[b]
        peak = max(peak, cur - (o.save_mem + a[b + 1]) + o.peak_bwd)
        cur -= (o.save_mem - a[b] - a[b + 1]) + 2 * a[b + 1]
        cur += a[b]
        peak = max(peak, cur)
    return peak


# BASELINE config 4: 256 budgets x 4 synthetic model chains.
SWEEP_CHAINS: Tuple[Tuple[str, int, int], ...] = (
    ("gpt2-small-like", 24, 8),
    ("resnet101-like", 33, 16),
    ("gpt2-medium-like", 48, 16),
    ("gpt2-xl-like", 96, 32),
)
SWEEP_UNITS = 500


@dataclass
class SweepInstance:
    chain: int       # index into the workload's menus
    budget: int      # bytes


def sweep_workload(n_budgets: int = 256, byte_scale: int = 1024):
    """Menus (bytes, so quantization is exercised) and the instance list:
    for each chain, budgets evenly spaced from 1/32 of its no-recompute peak
    up to the peak itself (min-feasible .. chain_max_peak).  The
    min-feasible budgets of these chains sit at 4-9 % of the peak (chain 0:
    below 1/32 the top slot is negative), so the low end of every sweep but
    chain 0's is infeasible and the batched min-feasible search runs too."""
    menus: List[Menu] = []
    inst: List[SweepInstance] = []
    for ci, (_, L, B) in enumerate(SWEEP_CHAINS):
        m = synthetic_menu(L, B, SWEEP_UNITS, seed=400 + ci, byte_scale=byte_scale)
        menus.append(m)
        hi = one_pass_peak(m)
        for b in even_spacing(hi // 32, hi, n_budgets):
            inst.append(SweepInstance(ci, b))
    return menus, inst


def instance_cost(menu: Menu, m_slots: int) -> int:
    """DP work estimate L^2 (M+1) (L + B) used to balance instances."""
    L = menu.L
    B = int(menu.n_saved().max()) if L else 0
    return L * L * (m_slots + 1) * (L + B)


def partition_lpt(costs: Sequence[int], n_ranks: int) -> List[List[int]]:
    """Longest-processing-time-first greedy assignment of independent
    instances to ranks; deterministic (ties by index)."""
    order = sorted(range(len(costs)), key=lambda i: (-costs[i], i))
    heap = [(0, r) for r in range(n_ranks)]
    heapq.heapify(heap)
    parts: List[List[int]] = [[] for _ in range(n_ranks)]
    for i in order:
        load, r = heapq.heappop(heap)
        parts[r].append(i)
        heapq.heappush(heap, (load + costs[i], r))
    return [sorted(p) for p in parts]
