"""bench.py -- rk-Rotor chain DP throughput (DP cell-updates/s) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference] [--config 2]

One step = one full rk-Rotor solve of one chain: every cell (s <= t, m) of
the DP table filled on the GPU (the wavefront kernels) plus the device
backtrack of the top cell into a schedule (BASELINE.json metric: "DP
cell-updates/sec and solve wall-time").  Workload at N=1: BASELINE.json
configs[1] (ResNet-101-like chain, L=33, B=16, M=4096), synthetic menus from
the deterministic generator of SURVEY.md 8(d).  Under torchrun each rank
solves its own independent chain of the same shape (budget sweeps / model
instances shard with no communication: "scaling": "weak"); the only
collectives are the timing barrier and the max-over-ranks reduction.

The JSON line carries: value (device-timed, inputs resident), e2e (the same
metric through the public C-ABI call with host menu arrays, H2D + fill +
backtrack + D2H of the schedule inside the timed region), roofline of the
dominant kernel (fill_diag) against the measured HBM copy bandwidth, the
reference CPU solver timed on this host (cpu_baseline), clocks.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_2307_01236_b200.menu import CONFIGS, synthetic_menu  # noqa: E402

FALLBACK_HBM_GBS = 6650.0


def cells_of(L, M):
    return L * (L + 1) // 2 * (M + 1)


def alg_bytes(L, M):
    """bytes(s,t,m) = 16(t-s) + 24, summed exactly."""
    return sum((L - k) * (16 * k + 24) for k in range(L)) * (M + 1)


def candidates_of(L, B, M):
    return sum((L - k) * (B + k) for k in range(L)) * (M + 1)


def rank_menu(cfg_idx, rank):
    c = CONFIGS[cfg_idx]
    return synthetic_menu(c["L"], c["B"], c["M"], seed=42 + cfg_idx + 1000 * rank)


def measured_peak():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md)"


def ncu_traffic(cfg_idx, kernel):
    """dram__bytes_read.sum + dram__bytes_write.sum of one fill launch of
    `kernel` (profiles/ncu_traffic.json, from an ncu capture of this bench)."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return d.get(f"config{cfg_idx}", {}).get(kernel, {}).get("dram_bytes_per_fill")
    except Exception:
        return None


FILL_KERNELS = {
    "tiles": "fill_tiles (K1t budget tiles: one co-resident CTA per 32-slot tile; tables with more "
             "tiles than SMs run the same tiles as jobs, fill_tiles_batch)",
    "queue": "fill_persistent (K1p: one persistent launch, dataflow work queue)",
    "diagonal": "fill_diag (K1: one launch per anti-diagonal)",
}


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.rows = []
        self._stop = threading.Event()
        self._t = None

    def _one(self):
        try:
            out = subprocess.run(["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}",
                                  "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                 timeout=5).stdout.strip()
            if out:
                self.rows.append([x.strip() for x in out.split(",")])
        except Exception:
            pass

    def _loop(self):
        while not self._stop.is_set():
            self._one()
            self._stop.wait(0.05)

    def __enter__(self):
        self._t = threading.Thread(target=self._loop, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)
        if not self.rows:
            self._one()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4)
                          if len(r) > 2 + i and r[2 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.rows)}


def dist_setup():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def reference_arm(args, world, rank):
    """The reference's own CPU implementation (oracle/_ref: remat::DpTable from
    the unmodified headers) on this host's cores; rank 0 only."""
    if rank != 0:
        return
    from oracle.pyoracle import HAVE_REF, Orc, Ref

    c = CONFIGS[args.config]
    L, B, M = c["L"], c["B"], c["M"]
    menu = rank_menu(args.config, 0)
    if args.config == 5:  # bounded sample: the full table needs 550 GB / ~107 h on CPU
        L, B, M = 256, 64, 64
        menu = synthetic_menu(L, B, M, seed=47)
    threads = os.cpu_count() or 1
    if HAVE_REF:
        ref, kind = Ref(), "reference"
    else:  # the C restatement, same algorithm
        ref, kind = None, "port"
    cells = cells_of(L, M)

    def step():
        if ref is not None:
            secs, top = ref.table_bench(menu, 1, M, threads)
        else:
            import concurrent.futures as cf
            t0 = time.perf_counter()
            with cf.ThreadPoolExecutor(threads) as ex:
                list(ex.map(lambda _: Orc().fill(menu, 1, M), range(threads)))
            secs = time.perf_counter() - t0
        return secs

    for _ in range(args.warmup):
        step()
    times = [step() for _ in range(args.steps)]
    total = sum(times)
    value = threads * cells * args.steps / total
    line = {
        "impl": "reference",
        "metric": "DP cell-updates/sec (rk-Rotor chain DP, full table fill)",
        "value": value, "unit": "cells/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * total / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "int64",
        "data": "synthetic (SURVEY.md 8(d) splitmix64 generator)",
        "config": {"workload": f"config{args.config}: {c['name']} chain, L={L}, B={B}, M={M}; "
                               f"reference remat::DpTable fill, {threads} concurrent solves/step",
                   "L": L, "B": B, "M": M},
        "cpu_baseline": {"value": value, "unit": "cells/s", "cores": threads, "kind": kind,
                         "sample": f"each step = {threads} concurrent full config-{args.config} "
                                   f"table fills (one per host thread; the reference solver "
                                   f"itself is single-threaded, pipeline.hpp:58)"},
        "e2e": {"value": value, "unit": "cells/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def cpu_baseline_sample(cfg_idx, menu, L, M):
    """Reference CPU solver on this host, 1 thread (as it ships), bounded sample."""
    from oracle.pyoracle import HAVE_REF, Orc, Ref

    reps = 3
    if HAVE_REF:
        ref = Ref()
        secs = [ref.table_bench(menu, 1, M, 1)[0] for _ in range(reps)]
        kind = "reference"
    else:
        orc = Orc()
        secs = []
        for _ in range(reps):
            t0 = time.perf_counter()
            orc.fill(menu, 1, M)
            secs.append(time.perf_counter() - t0)
        kind = "port"
    s = statistics.median(secs)
    return {"value": cells_of(L, M) / s, "unit": "cells/s", "cores": 1, "kind": kind,
            "sample": f"full config-{cfg_idx} table fill (L={L}, M={M}), median of {reps}, "
                      f"1 thread (the reference solver is single-threaded)",
            "seconds_per_solve": s}


def b200_arm(args, world, rank, local):
    import torch

    from paper_2307_01236_b200 import rotor

    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    if not rotor.lib().rkr_device_ok(local):
        raise SystemExit("bench: no sm_100 device")
    c = CONFIGS[args.config]
    L, B, M = c["L"], c["B"], c["M"]
    menu = rank_menu(args.config, rank)
    stream = torch.cuda.Stream(device=local)
    table = rotor.DpTable(menu, 1, M, device=local, stream=stream.cuda_stream)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=f"cuda:{local}")

    def barrier():
        if world > 1:
            torch.distributed.barrier()

    def max_over_ranks(x):
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=f"cuda:{local}")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        return float(t.item())

    # ---- device-resident solves -----------------------------------------------
    # one step = the whole device solve: fill + schedule walk from the top
    # cell (one launch with the budget-tile kernel, whose last CTA walks)
    def one_step(ev=None):
        if ev is not None:
            ev[0].record(stream)
        table.refill_walk(0, L - 1, M)
        if ev is not None:
            ev[1].record(stream)

    sampler = ClockSampler(local)
    with sampler:
        for _ in range(args.warmup):
            with torch.cuda.stream(stream):
                flush.zero_()
            one_step()
        ops_ref = table.backtrack_fetch()
        evs = [[torch.cuda.Event(enable_timing=True) for _ in range(2)] for _ in range(args.steps)]
        barrier()
        torch.cuda.synchronize()
        for i in range(args.steps):
            with torch.cuda.stream(stream):
                flush.zero_()  # L2 flush between timed steps (outside the events)
            one_step(evs[i])
        torch.cuda.synchronize()
        barrier()
        ops = table.backtrack_fetch()
        # the dominant kernel alone (fill without the walk), same L2 flushes,
        # events on the stream it is launched on: the roofline's duration
        kevs = [[torch.cuda.Event(enable_timing=True) for _ in range(2)] for _ in range(args.steps)]
        for i in range(args.steps):
            with torch.cuda.stream(stream):
                flush.zero_()
            kevs[i][0].record(stream)
            table.refill()
            kevs[i][1].record(stream)
        torch.cuda.synchronize()
    fill_ms = [e[0].elapsed_time(e[1]) for e in kevs]
    step_ms = [e[0].elapsed_time(e[1]) for e in evs]
    assert ops == ops_ref
    top = table.opt(0, L - 1, M)
    tot_s = max_over_ranks(sum(step_ms) / 1e3)
    fill_mean_s = statistics.mean(fill_ms) / 1e3

    # ---- end to end through the public API (host menu arrays) -------------------
    h2d = table.h2d_bytes()
    e2e_times = []
    n_ops = 0
    # one C-ABI call per step: rkr_solve_chain(host menu arrays) with
    # budget = M + a_0 bytes and units = budget (unit 1, m_top = M, i.e.
    # exactly this table); output buffers preallocated on the host, as a C
    # caller would
    import ctypes

    lib = rotor.lib()
    budget = M + int(menu.act_sizes[0])
    ms = menu.struct()
    ex = rotor._exec(local, "auto")
    cap = 1 << 16
    obuf = (rotor.RkrOp * cap)()
    n_, ot_, un_, mf_ = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
    mt_ = ctypes.c_int32()
    for i in range(args.warmup + args.steps):
        with torch.cuda.stream(stream):
            flush.zero_()
        torch.cuda.synchronize()
        barrier()
        t0 = time.perf_counter()
        st = lib.rkr_solve_chain(ctypes.byref(ms), budget, budget, ctypes.byref(ex), obuf, cap,
                                 ctypes.byref(n_), ctypes.byref(ot_), ctypes.byref(un_),
                                 ctypes.byref(mt_), ctypes.byref(mf_))
        dt = time.perf_counter() - t0
        assert st == 0, lib.rkr_last_error()
        if i >= args.warmup:
            e2e_times.append(dt)
    n_ops = n_.value
    sched = [(obuf[q].kind, obuf[q].block, obuf[q].option) for q in range(n_ops)]
    assert ot_.value == top and sched == ops
    e2e_s = max_over_ranks(sum(e2e_times))
    d2h = 8 + 2 + 32 + 12 * n_ops

    cells = cells_of(L, M)
    if rank != 0:
        return
    peak, peak_src = measured_peak()
    ab = alg_bytes(L, M)
    achieved = ab / fill_mean_s / 1e9
    kern = table.kernel()
    traffic = ncu_traffic(args.config, kern)
    line = {
        "metric": "DP cell-updates/sec (rk-Rotor chain DP, full table fill + backtrack)",
        "value": world * cells * args.steps / tot_s,
        "unit": "cells/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": 1e3 * tot_s / args.steps,
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "int64" if table.width() == 64 else "int64 (stored as u32, overflow-proven)",
        "data": "synthetic (SURVEY.md 8(d) splitmix64 generator; one independent chain per rank)",
        "config": {
            "workload": f"config{args.config}: {c['name']} chain, L={L} blocks, B={B} options/block, "
                        f"M={M} budget slots; full DP fill + device backtrack per step",
            "L": L, "B": B, "M": M, "cells_per_solve": cells,
            "candidates_per_solve": candidates_of(L, B, M),
            "l2": "flushed between timed steps (256 MiB write, outside the events)",
            "parallelism": f"instances x{world} (no data-path collective)",
            "solve_ms": 1e3 * tot_s / args.steps,
            "top_opt": top,
        },
        "e2e": {"value": world * cells * args.steps / e2e_s, "unit": "cells/s",
                "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                "ms_per_step": 1e3 * e2e_s / args.steps,
                "path": "rkr_solve_chain(host menu arrays): quantize, H2D, fill, top cell, "
                        "device backtrack, D2H of the schedule"},
        # per step: the fill (one launch, or L for the per-diagonal kernel) and
        # the walk (fused into the budget-tile fill, its own launch otherwise)
        "gpu_launches": args.steps * ((L if kern == "diagonal" else 1) + (0 if kern == "tiles" else 1)),
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic,
                     "kernel": FILL_KERNELS[kern],
                     "alg_bytes_per_fill": ab, "fill_ms": 1e3 * fill_mean_s,
                     "peak_source": peak_src},
        "clocks": sampler.summary(),
    }
    if world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline_sample(args.config, menu, L, M)
    print(json.dumps(line), flush=True)
    table.close()


# ---------------------------------------------------------------------------
# config 4: budget sweep (256 budgets x 4 chains), instances sharded by LPT
# ---------------------------------------------------------------------------
def sweep_instances():
    """All config-4 instances with their quantization (host arithmetic only)."""
    from paper_2307_01236_b200 import rotor
    from paper_2307_01236_b200.sweep import SWEEP_UNITS, sweep_workload

    menus, inst = sweep_workload()
    rows = []
    for i, x in enumerate(inst):
        q = rotor.quantize(x.budget, SWEEP_UNITS)
        a0 = rotor.to_units(int(menus[x.chain].act_sizes[0]), q.unit)
        rows.append((i, x.chain, x.budget, q.unit, q.budget_units - a0))
    return menus, rows


def sweep_cells(menus, rows):
    return sum(menus[ci].L * (menus[ci].L + 1) // 2 * (mt + 1) for _, ci, _, _, mt in rows if mt >= 0)


def sweep_alg_bytes(menus, rows):
    return sum(alg_bytes(menus[ci].L, mt) for _, ci, _, _, mt in rows if mt >= 0)


def b200_arm_sweep(args, world, rank, local):
    import torch

    from paper_2307_01236_b200 import rotor
    from paper_2307_01236_b200.sweep import SWEEP_CHAINS, SWEEP_UNITS, instance_cost, partition_lpt

    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    menus, rows_all = sweep_instances()
    costs = [instance_cost(menus[ci], max(mt, 0)) for _, ci, _, _, mt in rows_all]
    mine = set(partition_lpt(costs, world)[rank])
    rows = [r for r in rows_all if r[0] in mine]
    res = [r for r in rows if r[4] >= 0]
    stream = torch.cuda.Stream(device=local)
    batch = rotor.Batch([menus[ci] for _, ci, _, _, _ in res], [u for *_, u, _ in res],
                        [mt for *_, mt in res], device=local, stream=stream.cuda_stream)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=f"cuda:{local}")

    def barrier():
        if world > 1:
            torch.distributed.barrier()

    def max_over_ranks(x):
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=f"cuda:{local}")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        return float(t.item())

    sampler = ClockSampler(local)
    with sampler:
        for _ in range(args.warmup):
            batch.refill()
        evs = [[torch.cuda.Event(enable_timing=True) for _ in range(2)] for _ in range(args.steps)]
        barrier()
        torch.cuda.synchronize()
        for i in range(args.steps):
            with torch.cuda.stream(stream):
                flush.zero_()
            evs[i][0].record(stream)
            batch.refill()
            evs[i][1].record(stream)
        torch.cuda.synchronize()
        barrier()
    fill_ms = [e[0].elapsed_time(e[1]) for e in evs]
    tot_s = max_over_ranks(sum(fill_ms) / 1e3)
    # bytes each end-to-end step uploads: every table's menu blob (the unit
    # precompute + descriptor) -- the same tables rkr_sweep builds
    h2d = sum(batch.table(i).h2d_bytes() for i in range(len(batch)))
    kern = batch.table(0).kernel()
    batch.close()

    # end to end: one rkr_sweep C-ABI call per chain from host menus (fill,
    # top cells, schedules, min-feasible search; schedules copied back into
    # caller buffers), buffers preallocated as a C caller would
    import ctypes

    lib = rotor.lib()
    by_chain = {}
    for _, ci, b, _, _ in rows:
        by_chain.setdefault(ci, []).append(b)
    # one rkr_sweep_chains call: every chain's budgets in one batch (the
    # reference runs cmd_sweep once per chain; the results are identical)
    chains = sorted(by_chain)
    structs = [menus[ci].struct() for ci in chains]
    mp = (ctypes.POINTER(rotor.RkrMenu) * len(chains))(*[ctypes.pointer(x) for x in structs])
    counts = (ctypes.c_int32 * len(chains))(*[len(by_chain[ci]) for ci in chains])
    flat = [b for ci in chains for b in by_chain[ci]]
    n = len(flat)
    cap = max(1024, sum(8 * len(by_chain[ci]) * menus[ci].L for ci in chains))
    b_ = (ctypes.c_int64 * n)(*flat)
    st_, ot_, un_ = (ctypes.c_int32 * n)(), (ctypes.c_int64 * n)(), (ctypes.c_int64 * n)()
    mt_, mf_ = (ctypes.c_int32 * n)(), (ctypes.c_int64 * n)()
    ops_, offs = (rotor.RkrOp * cap)(), (ctypes.c_int64 * (n + 1))()
    ex = rotor._exec(local, "auto")
    e2e = []
    for it in range(args.warmup + args.steps):
        torch.cuda.synchronize()
        barrier()
        t0 = time.perf_counter()
        rc = lib.rkr_sweep_chains(mp, counts, len(chains), b_, SWEEP_UNITS, ctypes.byref(ex), st_,
                                  ot_, un_, mt_, mf_, ops_, cap, offs)
        assert rc == 0, lib.rkr_last_error()
        dt = time.perf_counter() - t0
        if it >= args.warmup:
            e2e.append(dt)
    n_ops = offs[n]
    n_feas = sum(1 for i in range(n) if st_[i] == 0)
    e2e_s = max_over_ranks(sum(e2e))
    cells_rank = sweep_cells(menus, rows)
    cells_total = sweep_cells(menus, rows_all)
    if rank != 0:
        return
    peak, peak_src = measured_peak()
    ab = sweep_alg_bytes(menus, rows)
    achieved = ab / (statistics.mean(fill_ms) / 1e3) / 1e9
    line = {
        "metric": "DP cell-updates/sec (rk-Rotor chain DP, budget sweep)",
        "value": cells_total * args.steps / tot_s,
        "unit": "cells/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * tot_s / args.steps, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "int64 (stored as u32, overflow-proven)",
        "data": "synthetic (SURVEY.md 8(d) generator, byte-sized menus, units=500)",
        "config": {
            "workload": "config4: budget sweep, 4 chains x 256 budgets "
                        + "/".join(f"{L}x{B}" for _, L, B in SWEEP_CHAINS)
                        + ", every instance's full DP table in one persistent launch per GPU",
            "instances": len(rows_all), "cells_per_step": cells_total,
            "l2": "flushed between timed steps (256 MiB write, outside the events)",
            "parallelism": f"instances LPT-sharded over {world} GPU(s), no data-path collective",
        },
        "e2e": {"value": cells_total * args.steps / e2e_s, "unit": "cells/s",
                "ms_per_step": 1e3 * e2e_s / args.steps,
                "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": 12 * n_ops,
                "path": "one rkr_sweep_chains C-ABI call (all chains' budgets in one batch) "
                        "from host menus: fill + tops + schedules + min-feasible search, "
                        "schedules copied back",
                "feasible_budgets_rank0": n_feas},
        "gpu_launches": args.steps,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": ncu_traffic(4, kern),
                     "kernel": ("fill_tiles_batch (K1t jobs: persistent CTAs take (table, budget tile) "
                                "jobs, every table in one launch)" if kern == "tiles" else
                                "fill_persistent (K1p, every table in one launch)"),
                     "alg_bytes_per_fill": ab, "fill_ms": statistics.mean(fill_ms),
                     "peak_source": peak_src},
        "clocks": sampler.summary(),
    }
    if world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline_sweep(menus, rows_all)
    print(json.dumps(line), flush=True)


def cpu_baseline_sweep(menus, rows_all, per_chain=3):
    """Reference solve_chain on a bounded sample of the sweep (per_chain budgets
    of each chain, spread over the range), 1 thread; rate in cells/s."""
    from oracle.pyoracle import HAVE_REF, Orc, Ref

    from paper_2307_01236_b200.sweep import SWEEP_UNITS

    ref = Ref() if HAVE_REF else Orc()
    sample = []
    for ci in range(len(menus)):
        rs = [r for r in rows_all if r[1] == ci and r[4] >= 0]
        for k in range(per_chain):
            sample.append(rs[(k + 1) * len(rs) // (per_chain + 1)])
    t0 = time.perf_counter()
    for _, ci, b, _, _ in sample:
        ref.solve_chain(menus[ci], b, SWEEP_UNITS)
    secs = time.perf_counter() - t0
    return {"value": sweep_cells(menus, sample) / secs, "unit": "cells/s", "cores": 1,
            "kind": "reference" if HAVE_REF else "port",
            "sample": f"{len(sample)} sweep instances ({per_chain} budgets per chain), "
                      f"reference solve_chain, 1 thread, {secs:.1f} s"}


def reference_arm_sweep(args, world, rank):
    if rank != 0:
        return
    import concurrent.futures as cf

    from oracle.pyoracle import HAVE_REF, Orc, Ref

    from paper_2307_01236_b200.sweep import SWEEP_UNITS

    menus, rows_all = sweep_instances()
    threads = os.cpu_count() or 1
    ref = Ref() if HAVE_REF else Orc()
    # bounded sample per step: 2 instances per host thread, spread over the sweep
    k = 2 * threads
    sample = [rows_all[(i * len(rows_all)) // k] for i in range(k)]
    sample = [r for r in sample if r[4] >= 0]

    def step():
        t0 = time.perf_counter()
        with cf.ThreadPoolExecutor(threads) as ex:
            list(ex.map(lambda r: ref.solve_chain(menus[r[1]], r[2], SWEEP_UNITS), sample))
        return time.perf_counter() - t0

    for _ in range(args.warmup):
        step()
    times = [step() for _ in range(args.steps)]
    value = sweep_cells(menus, sample) * args.steps / sum(times)
    print(json.dumps({
        "impl": "reference", "metric": "DP cell-updates/sec (rk-Rotor chain DP, budget sweep)",
        "value": value, "unit": "cells/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * sum(times) / args.steps,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "int64",
        "data": "synthetic (SURVEY.md 8(d) generator, byte-sized menus, units=500)",
        "config": {"workload": f"config4 sample: {len(sample)} sweep instances per step on "
                               f"{threads} host threads (reference solve_chain)"},
        "cpu_baseline": {"value": value, "unit": "cells/s", "cores": threads,
                         "kind": "reference" if HAVE_REF else "port",
                         "sample": f"{len(sample)} instances per step spread over the sweep"},
        "e2e": {"value": value, "unit": "cells/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }), flush=True)


# ---------------------------------------------------------------------------
# config 5: one huge chain, budget axis sharded across ranks (one shard per GPU)
# ---------------------------------------------------------------------------
def b200_arm_sharded(args, world, rank, local):
    import torch
    import torch.distributed as dist

    from paper_2307_01236_b200 import rotor

    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    c = CONFIGS[5]
    L, B, M = c["L"], c["B"], c["M"]
    twin = world == 1  # the full table (206 GB) needs >= 2 GPUs
    if twin:
        L, B, M = 256, 64, 4096
    menu = synthetic_menu(L, B, M, seed=47)
    sh = rotor.ProcessShard(menu, 1, M, world, rank, device=local)

    def gather(obj):
        if world == 1:
            return [obj]
        out = [None] * world
        dist.all_gather_object(out, obj)
        return out

    def barrier():
        if world > 1:
            dist.barrier()

    handles, infos = rotor.link_process_shards(sh, gather)
    stream = torch.cuda.ExternalStream(sh.table.stream(), device=f"cuda:{local}")
    lo, hi = sh.range()

    def fill(ev=None):
        sh.zero()
        barrier()
        if ev:
            ev[0].record(stream)
        sh.launch()
        if ev:
            ev[1].record(stream)
        sh.sync()
        barrier()

    sampler = ClockSampler(local)
    with sampler:
        for _ in range(args.warmup):
            fill()
        evs = [[torch.cuda.Event(enable_timing=True) for _ in range(2)] for _ in range(args.steps)]
        for i in range(args.steps):
            fill(evs[i])
    ms = [e[0].elapsed_time(e[1]) for e in evs]
    mine = sum(ms) / 1e3
    if world > 1:
        t = torch.tensor([mine], dtype=torch.float64, device=f"cuda:{local}")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        mine = float(t.item())
    ops = sh.backtrack(handles, infos, 0, L - 1, M) if rank == 0 else []
    shard_kern = sh.table.kernel()
    barrier()
    if rank == 0:
        peak, peak_src = measured_peak()
        cells = cells_of(L, M)
        ab = alg_bytes(L, M)
        fill_s = mine / args.steps
        line = {
            "metric": "DP cell-updates/sec (rk-Rotor chain DP, budget-sharded single chain)",
            "value": cells * args.steps / mine, "unit": "cells/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * fill_s,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "int64 (stored as u32, overflow-proven)",
            "data": "synthetic (SURVEY.md 8(d) generator)",
            "config": {"workload": (f"config5{'-twin' if twin else ''}: L={L}, B={B}, M={M}, budget "
                                    f"axis in {world} shard(s), halo pushed in-kernel over peer memory"),
                       "L": L, "B": B, "M": M, "shard0_range": [lo, hi], "schedule_ops": len(ops)},
            "gpu_launches": args.steps * world,
            "roofline": {"bound": "hbm", "achieved": ab / fill_s / 1e9 / world, "peak": peak,
                         "unit": "GB/s", "frac": ab / fill_s / 1e9 / world / peak, "traffic": None,
                         "kernel": (FILL_KERNELS[shard_kern] if shard_kern != "tiles" else
                                    "fill_tiles (K1t budget tiles, streamed programs for long chains)")
                                   + ", one launch per shard per step; halo pushed in-kernel",
                         "alg_bytes_per_fill": ab, "peak_source": peak_src + ", per GPU"},
            "clocks": sampler.summary(),
        }
        print(json.dumps(line), flush=True)
    sh.close()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", type=int, default=2, choices=[1, 2, 3, 4, 5])
    ap.add_argument("--no-cpu-baseline", action="store_true", help="skip the CPU leg (tuning runs)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3) if args.impl == "b200" else args.warmup
    world, rank, local = dist_setup()
    if args.config == 5 and args.impl == "b200":
        b200_arm_sharded(args, world, rank, local)
        return
    if args.config == 4:
        if args.impl == "reference":
            reference_arm_sweep(args, world, rank)
        else:
            b200_arm_sweep(args, world, rank, local)
    elif args.impl == "reference":
        reference_arm(args, world, rank)
    else:
        b200_arm(args, world, rank, local)


if __name__ == "__main__":
    main()
