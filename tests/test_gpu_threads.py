"""Concurrent host threads (SURVEY §8b threading contract: distinct handles
usable from distinct threads).  Each thread creates, fills, reads back and
walks its own tables -- single tables on every kernel, solve_chain, a batch --
while the others do the same; every result is compared with the CPU oracle,
computed beforehand on the main thread.  ctypes releases the GIL around every
librkr call, so the C ABI really runs concurrently (thread-local staging
buffers and error strings, one shared per-device stream)."""
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest

from paper_2307_01236_b200 import rotor
from paper_2307_01236_b200.menu import synthetic_menu

pytestmark = pytest.mark.gpu

KERNELS = ["persistent", "tiles", "queue", "diagonal"]


def _cases(orc):
    cases = []
    for i in range(8):
        L, B, M = 6 + 3 * i, 2 + i % 5, 150 + 60 * i
        menu = synthetic_menu(L, B, M, 100 + i, tie_stress=bool(i & 1))
        st, *ref = orc.fill(menu, 1, M)
        assert st == 0
        top = ref[0][L - 1]
        fin = np.nonzero(top < rotor.K_INF_TIME)[0]
        walk = None
        if len(fin):
            mm = int(fin[0])
            _, ops = orc.build_schedule(menu, 1, M, tuple(ref[:3]), 0, L - 1, mm)
            walk = (mm, ops)
        budget = int(M // 2 + menu.act_sizes[0])
        sol = orc.solve_chain(menu, budget, budget)
        cases.append((menu, M, ref[:3], walk, budget, sol))
    return cases


def _work(arg):
    idx, cases = arg
    bad = []
    for rep in range(3):
        for ci, (menu, M, ref, walk, budget, sol) in enumerate(cases):
            kernel = KERNELS[(idx + ci + rep) % len(KERNELS)]
            with rotor.DpTable(menu, 1, M, kernel=kernel) as t:
                got = t.download()
                if not all(np.array_equal(x, y) for x, y in zip(got, ref)):
                    bad.append(("table", idx, ci, kernel))
                if walk is not None:
                    mm, ops = walk
                    t.refill_walk(0, menu.L - 1, mm)
                    if t.backtrack_fetch() != ops or t.backtrack(0, menu.L - 1, mm) != ops:
                        bad.append(("walk", idx, ci, kernel))
            st, ops, opt_time, unit, m_top, _ = sol
            chain = rotor.Chain.skeleton(menu.L)
            if st == 0:
                s = rotor.solve_chain(chain, menu, budget, budget)
                if (s.opt_time, s.unit, s.m_top) != (opt_time, unit, m_top) or s.raw_ops != ops:
                    bad.append(("solve", idx, ci))
        with rotor.Batch([c[0] for c in cases], [1] * len(cases), [c[1] for c in cases]) as b:
            for ci, c in enumerate(cases):
                if not all(np.array_equal(x, y) for x, y in zip(b.table(ci).download(), c[2])):
                    bad.append(("batch", idx, ci))
    return bad


def test_threads_share_the_library(orc):
    cases = _cases(orc)
    with ThreadPoolExecutor(max_workers=4) as ex:
        bad = [b for res in ex.map(_work, [(i, cases) for i in range(4)]) for b in res]
    assert bad == []
