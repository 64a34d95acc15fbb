"""Reference-generated goldens for the full-size BASELINE configurations.

Run in the build container (where /root/reference exists), after
`make -f oracle/Makefile`:

    python tests/golden/gen_golden_large.py cfg3 cfg4 cfg5twin l1024

Every number comes from the UNMODIFIED reference (oracle/_ref: remat::DpTable,
build_schedule_rec, solve_chain compiled from /root/reference/proj/include)
and testing::atomic_replay (tests/test_helpers.hpp:249-322).  Outputs
(committed, small): large_<part>.json with

  cfg3      config 3 (L=96, B=32, M=16384, seed 45 -- bench.py's chain): the
            sha256 of the whole reference table (opt int64 | kind int8 | value
            int32, s-major triangular rows), one short digest per diagonal,
            the top row, and schedules (ops digest, replayed peak/time) from
            several cells
  cfg4      config 4 (sweep.sweep_workload: 4 chains x 256 budgets, units=500):
            every instance's solve_chain result
  cfg5twin  config-5 twin (L=256, B=64, M=4096, seed 47 -- bench.py's N=1
            sharded chain): as cfg3
  l1024     config-5 chain length (L=1024, B=64) at M=64: as cfg3
  l1024m256 the same chain length at M=256 (seed 49): as cfg3
"""
from __future__ import annotations

import concurrent.futures as cf
import hashlib
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle.pyoracle import Ref  # noqa: E402
from paper_2307_01236_b200.menu import synthetic_menu  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def table_digest(o, k, v) -> str:
    h = hashlib.sha256()
    h.update(np.ascontiguousarray(o, dtype="<i8").tobytes())
    h.update(np.ascontiguousarray(k, dtype="i1").tobytes())
    h.update(np.ascontiguousarray(v, dtype="<i4").tobytes())
    return h.hexdigest()


def tri_row(L, s, t):
    return s * L - s * (s - 1) // 2 + (t - s)


def diag_digests(o, k, v, L):
    """16-hex sha256 prefix per anti-diagonal k (rows (s, s+k), s ascending)."""
    out = []
    for d in range(L):
        idx = np.array([tri_row(L, s, s + d) for s in range(L - d)], np.int64)
        out.append(table_digest(o[idx], k[idx], v[idx])[:16])
    return out


def ops_digest(ops) -> str:
    return hashlib.sha256(np.array(ops, dtype="<i4").reshape(-1).tobytes()).hexdigest()


def table_part(ref, L, B, M, seed):
    menu = synthetic_menu(L, B, M, seed)
    cells = [(0, L - 1, M >> q) for q in range(0, 7)] + [
        (1, L - 1, M), (L // 2, L - 1, M // 2), (0, L // 2, M), (L - 1, L - 1, M)]
    t0 = time.time()
    st, (o, k, v), mc, walks = ref.fill_and_walk(menu, 1, M, cells)
    secs = time.time() - t0
    assert st == 0
    top = o[tri_row(L, 0, L - 1)]
    fin = np.nonzero(top < (2**63 - 1) // 4)[0]
    ff = int(fin[0]) if len(fin) else -1
    wl = []
    for (s, t, m), (ws, ops) in zip(cells, walks):
        e = {"s": s, "t": t, "m": m, "status": ws}
        if ws == 0:
            peak, tm = ref.atomic_replay(menu, ops) if s == 0 and t == L - 1 else (None, None)
            e.update(n_ops=len(ops), ops_digest=ops_digest(ops), replay_peak=peak, replay_time=tm,
                     opt=int(o[tri_row(L, s, t), m]))
        wl.append(e)
    r = tri_row(L, 0, L - 1)
    return {"L": L, "B": B, "M": M, "seed": seed, "digest": table_digest(o, k, v),
            "diag_digests": diag_digests(o, k, v, L), "max_cands": mc, "first_feasible": ff,
            "top": o[r].tolist(), "top_kind": k[r].tolist(), "top_value": v[r].tolist(),
            "walks": wl, "ref_seconds": round(secs, 1)}


def cfg4_part(ref):
    from paper_2307_01236_b200.sweep import SWEEP_UNITS, sweep_workload

    menus, inst = sweep_workload()

    def one(i):
        x = inst[i]
        st, ops, ot, un, mt, mf = ref.solve_chain(menus[x.chain], x.budget, SWEEP_UNITS)
        e = {"chain": x.chain, "budget": x.budget, "status": st, "min_feasible": mf}
        if st == 0:
            peak, tm = ref.atomic_replay(menus[x.chain], ops)
            e.update(opt_time=ot, unit=un, m_top=mt, n_ops=len(ops), ops_digest=ops_digest(ops),
                     replay_peak=peak, replay_time=tm)
        return e

    with cf.ThreadPoolExecutor(int(os.environ.get("GEN_THREADS", "6"))) as ex:
        res = list(ex.map(one, range(len(inst))))
    return {"units": SWEEP_UNITS, "instances": res}


PARTS = {
    "cfg3": lambda ref: table_part(ref, 96, 32, 16384, 45),
    "cfg4": cfg4_part,
    "cfg5twin": lambda ref: table_part(ref, 256, 64, 4096, 47),
    "l1024": lambda ref: table_part(ref, 1024, 64, 64, 48),
    # config-5 chain length at M = 256 (~55 G candidates, ~10 min of reference CPU)
    "l1024m256": lambda ref: table_part(ref, 1024, 64, 256, 49),
}


def main(parts):
    ref = Ref()
    for p in parts:
        t0 = time.time()
        d = PARTS[p](ref)
        with open(os.path.join(OUT, f"large_{p}.json"), "w") as f:
            json.dump(d, f)
        print(f"{p}: written in {time.time() - t0:.0f} s", flush=True)


if __name__ == "__main__":
    main(sys.argv[1:] or list(PARTS))
