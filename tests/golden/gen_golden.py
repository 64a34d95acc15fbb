"""Generate the golden fixtures from the UNMODIFIED reference (oracle/_ref).

Run in the build container (where /root/reference exists):

    make -f oracle/Makefile && python tests/golden/gen_golden.py

Outputs (committed):
  kat.json            the reference's known-answer cases (test_chain_dp.cpp:9-107,
                      :203-221) as produced by the reference itself
  random_menus.json   testing::random_menu draws for the property/oracle tests
                      (seeds 5, 9, 13, 37, 41, 53 with the reference's sizes),
                      plus, per menu, the reference's full opt/arg tables (small M),
                      chain_oracle / chain_oracle_dijkstra values
  synthetic.json      SURVEY 8(d) synthetic chains: sha256 of the reference's
                      whole tables, top rows, and solve_chain results over budgets
"""
from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle.pyoracle import Ref  # noqa: E402
from paper_2307_01236_b200.menu import Menu, synthetic_menu, tiny_chain_menu  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def table_digest(o, k, v) -> str:
    h = hashlib.sha256()
    h.update(np.ascontiguousarray(o, dtype="<i8").tobytes())
    h.update(np.ascontiguousarray(k, dtype="i1").tobytes())
    h.update(np.ascontiguousarray(v, dtype="<i4").tobytes())
    return h.hexdigest()


def ops_digest(ops) -> str:
    return hashlib.sha256(np.array(ops, dtype="<i4").reshape(-1).tobytes()).hexdigest()


def main():
    ref = Ref()
    tiny = tiny_chain_menu()

    # ---- KATs ---------------------------------------------------------------
    kat = {"quantize": [], "tiny": {}, "single": {}, "solve": []}
    for b, u in ((1000, 10), (7, 1), (0, 5), (999, 1000), (12345, 500)):
        st, unit, bu = ref.quantize(b, u)
        kat["quantize"].append([b, u, st, unit, bu])
    st, unit, bu = ref.quantize(10, 0)
    kat["quantize"].append([10, 0, st, 0, 0])
    st, o, k, v, mc, wa = ref.fill(tiny, 1, 64)
    kat["tiny"] = {"M": 64, "opt": o.tolist(), "kind": k.tolist(), "value": v.tolist(),
                   "max_cands": mc, "worst_allow": wa}
    for M, m in ((12, 12), (10, 10), (9, 9)):
        st, ops = ref.build_schedule(tiny, 1, M, 0, 1, m)
        kat["tiny"][f"schedule_M{M}"] = {"status": st, "ops": ops}
    for budget, units in ((16, 16), (14, 14), (12, 12), (3, 3), (300, 7), (64, 64)):
        st, ops, ot, un, mt, mf = ref.solve_chain(tiny, budget, units)
        kat["solve"].append({"budget": budget, "units": units, "status": st, "ops": ops,
                             "opt_time": ot if st == 0 else None, "unit": un if st == 0 else None,
                             "m_top": mt if st == 0 else None, "min_feasible": mf})
    with open(os.path.join(OUT, "kat.json"), "w") as f:
        json.dump(kat, f)

    # ---- random menus (test_chain_dp.cpp:109-201) ----------------------------
    suites = {
        "monotone": dict(seed=5, count=60, blocks=4, opts=3, M=24),
        "ample": dict(seed=9, count=40, blocks=4, opts=3, M=4096),
        "symmetry": dict(seed=13, count=20, blocks=3, opts=2, M=20),
        "enumeration": dict(seed=37, count=60, blocks=4, opts=3, M=20),
        "work_bound": dict(seed=41, count=20, blocks=4, opts=3, M=20),
        "relaxed": dict(seed=53, count=15, blocks=3, opts=2, M=16),
    }
    rnd = {}
    for name, cfg in suites.items():
        menus = ref.random_menus(cfg["seed"], cfg["count"], cfg["blocks"], cfg["opts"])
        entries = []
        for mm in menus:
            st, o, k, v, mc, wa = ref.fill(mm, 1, cfg["M"])
            e = {"menu": mm.to_json(), "max_cands": mc, "worst_allow": wa}
            if cfg["M"] <= 64:
                e.update(opt=o.tolist(), kind=k.tolist(), value=v.tolist())
            else:
                e.update(digest=table_digest(o, k, v), top=o[mm.L - 1].tolist()[-1:])
            L = mm.L
            if name == "enumeration":
                e["chain_oracle"] = [ref.chain_oracle(mm, m + int(mm.act_sizes[0]))
                                     for m in range(0, 21, 2)]
            if name == "relaxed":
                e["dijkstra"] = [ref.chain_oracle_dijkstra(mm, m + int(mm.act_sizes[0]), L + 3)
                                 for m in range(0, 17, 4)]
            entries.append(e)
        rnd[name] = dict(cfg, menus=entries)
    with open(os.path.join(OUT, "random_menus.json"), "w") as f:
        json.dump(rnd, f)

    # ---- synthetic chains ---------------------------------------
    syn = {"tables": [], "solves": []}
    for (L, B, M, seed, tie) in ((8, 4, 64, 1, False), (12, 6, 128, 2, True), (24, 8, 500, 43, False),
                                 (33, 16, 4096, 44, False), (16, 8, 256, 7, True)):
        mm = synthetic_menu(L, B, M, seed, tie_stress=tie)
        st, o, k, v, mc, wa = ref.fill(mm, 1, M)
        syn["tables"].append({"L": L, "B": B, "M": M, "seed": seed, "tie_stress": tie,
                              "digest": table_digest(o, k, v), "max_cands": mc,
                              "top": o[L - 1].tolist(), "top_kind": k[L - 1].tolist(),
                              "top_value": v[L - 1].tolist()})
    # config 1: real bytes through solve_chain with units=500
    mm = synthetic_menu(24, 8, 500, 41, byte_scale=1024)
    st, ops, ot, un, mt, mf = ref.solve_chain(mm, 512000, 500)
    lo = mf if st == 2 else 0
    budgets = sorted(set([1000, 20000, 40000, 60000, 80000, 120000, 200000, 512000, 2000000]))
    for b in budgets:
        st, ops, ot, un, mt, mf = ref.solve_chain(mm, b, 500)
        peak, tm = ref.atomic_replay(mm, ops) if st == 0 else (-1, -1)
        syn["solves"].append({"L": 24, "B": 8, "M": 500, "seed": 41, "byte_scale": 1024,
                              "budget": b, "units": 500, "status": st,
                              "opt_time": ot if st == 0 else None, "unit": un if st == 0 else None,
                              "m_top": mt if st == 0 else None, "min_feasible": mf,
                              "n_ops": len(ops), "ops_digest": ops_digest(ops) if st == 0 else None,
                              "replay_peak": peak, "replay_time": tm})
    with open(os.path.join(OUT, "synthetic.json"), "w") as f:
        json.dump(syn, f)
    print("golden fixtures written to", OUT)


if __name__ == "__main__":
    main()
