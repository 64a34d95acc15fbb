"""Host logic of the multi-GPU paths, on CPU: budget grids, the one-pass
ceiling, LPT instance partitioning, and a world_size-2 gloo run of the
instance-sharded sweep protocol (each rank solves its share with the CPU
oracle; the gathered results equal a single-rank run)."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2307_01236_b200.menu import synthetic_menu
from paper_2307_01236_b200.sweep import (
    even_spacing,
    instance_cost,
    one_pass_peak,
    partition_lpt,
    sweep_workload,
)


def test_even_spacing_matches_reference_rule():
    # remat::even_spacing: inclusive, integer (hi-lo)*i/(n-1), duplicates dropped
    assert even_spacing(0, 10, 6) == [0, 2, 4, 6, 8, 10]
    assert even_spacing(5, 5, 4) == [5]
    assert even_spacing(7, 3, 4) == [3]
    assert even_spacing(0, 3, 7) == [0, 1, 2, 3]
    assert even_spacing(1, 9, 1) == [9]


def test_one_pass_peak_equals_replay_of_the_one_pass_schedule(orc):
    for seed in range(8):
        m = synthetic_menu(6 + seed, 3, 200, 900 + seed, byte_scale=1 + seed % 3)
        pick = []
        for b in range(m.L):
            best = min((o for o in m.options(b) if o.time_bwd is not None),
                       key=lambda o: o.time_fwd + o.time_bwd)
            pick.append(best.option_id)
        ops = [(2, b, pick[b]) for b in range(m.L)] + [(0, m.L - 1, -1)]
        ops += [(3, b, pick[b]) for b in range(m.L - 1, -1, -1)]
        peak, _ = orc.atomic_replay(m, ops)
        assert peak == one_pass_peak(m)


def test_partition_lpt_is_a_balanced_partition():
    rng = np.random.default_rng(3)
    costs = [int(x) for x in rng.integers(1, 1000, 200)]
    for n in (1, 2, 3, 8):
        parts = partition_lpt(costs, n)
        flat = sorted(i for p in parts for i in p)
        assert flat == list(range(len(costs)))
        loads = [sum(costs[i] for i in p) for p in parts]
        assert max(loads) - min(loads) <= max(costs)


def test_sweep_workload_shape():
    menus, inst = sweep_workload(n_budgets=256)
    assert [m.L for m in menus] == [24, 33, 48, 96]
    assert 900 <= len(inst) <= 1024
    assert all(instance_cost(menus[x.chain], 500) > 0 for x in inst)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle.pyoracle import Orc

    orc = Orc()
    menus = [synthetic_menu(6, 3, 120, 70 + i, byte_scale=16) for i in range(3)]
    inst = [(ci, b) for ci in range(3) for b in even_spacing(300, 2600, 9)]
    costs = [instance_cost(menus[ci], 120) for ci, _ in inst]
    mine = partition_lpt(costs, world)[rank]
    res = {}
    for i in mine:
        ci, b = inst[i]
        st, ops, ot, un, mt, mf = orc.solve_chain(menus[ci], b, 120)
        res[i] = (st, ot if st == 0 else mf)
    gathered = [None] * world
    dist.all_gather_object(gathered, res)
    if rank == 0:
        merged = {}
        for g in gathered:
            assert not (set(g) & set(merged))  # disjoint shares
            merged.update(g)
        out.put(merged)
    dist.barrier()
    dist.destroy_process_group()


def test_instance_sharding_gloo_world2(orc):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    merged = q.get(timeout=120)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    # single-rank reference of the same protocol
    menus = [synthetic_menu(6, 3, 120, 70 + i, byte_scale=16) for i in range(3)]
    inst = [(ci, b) for ci in range(3) for b in even_spacing(300, 2600, 9)]
    assert sorted(merged) == list(range(len(inst)))
    for i, (ci, b) in enumerate(inst):
        st, ops, ot, un, mt, mf = orc.solve_chain(menus[ci], b, 120)
        assert merged[i] == (st, ot if st == 0 else mf)
