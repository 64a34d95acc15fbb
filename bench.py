"""bench.py -- rk-Rotor chain DP throughput (DP cell-updates/s) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference] [--config 3]

One step = one full rk-Rotor solve of one chain (remat::solve_chain's work,
chain_dp.hpp:255-296): every cell (s <= t, m) of the DP table filled on the
GPU plus the device backtrack of the top cell into a schedule.  BASELINE.json's
metric ("DP cell-updates/sec and solve wall-time") names no configuration, so
the N=1 workload is the largest single-GPU one, configs[2]: the GPT-2-XL-like
chain, L=96 blocks, B=32 options/block, M=16384 budget slots (synthetic menus
from the deterministic generator of SURVEY.md 8(d), seed 45).  --config 1|2
are the smaller chains, --config 4 the budget sweep, --config 5 the
budget-sharded 1024-block chain.

Under torchrun (N > 1) config 3 runs budget-sharded: the budget axis is cut
into N contiguous shards, one per GPU, the halo travels inside the fill kernel
over NVLink peer memory (CUDA IPC), and rank 0 walks the schedule across the
shards ("scaling": "strong"); the line carries a cross-shard check against an
unsharded solve.  Configs 1-2 at N > 1 run one independent chain per rank
("scaling": "weak").

The JSON line carries: value (device-timed, inputs resident in HBM), e2e (the
same metric through the public C-ABI call rkr_solve_chain with host menu
arrays: H2D + fill + backtrack + D2H of the schedule inside the timed region),
the roofline of the dominant kernel (the fill) against the MEASURED L2 read
bandwidth (tools/l2probe.cu, run live) and the SM issue rate, with DRAM/L2
traffic and issue utilisation measured live by an ncu pass over one fill,
the reference CPU solver timed on this host (cpu_baseline), and clocks.

`--impl reference` times the reference's own solver (oracle/_ref: the
unmodified remat::solve_chain compiled from /root/reference's headers) on this
host's cores for the same metric and configuration.
"""
from __future__ import annotations

import argparse
import ctypes
import hashlib
import json
import os
import shutil
import statistics
import subprocess
import sys
import tempfile
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_2307_01236_b200.menu import CONFIGS, synthetic_menu  # noqa: E402

FALLBACK_HBM_GBS = 6650.0
METRIC = "DP cell-updates/sec (rk-Rotor solve_chain: full DP table fill + schedule backtrack)"
METRIC_SWEEP = "DP cell-updates/sec (rk-Rotor chain DP, budget sweep)"
METRIC_SHARDED = "DP cell-updates/sec (rk-Rotor chain DP, budget-sharded single chain)"
# reference arm: each host thread solves the config-3 chain quantized to
# M / REF_SAMPLE[cfg] budget slots (solve_chain's own `units` knob), so a
# step stays a few seconds; the 1-thread cpu_baseline of the b200 arm solves
# the full-size chain
REF_SAMPLE = {1: 1, 2: 1, 3: 8}


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


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return d, "measured (MEASURED_PEAKS.json)"
    except Exception:
        return {"hbm_gbs": FALLBACK_HBM_GBS, "sm_max_mhz": 1965.0}, "fallback (B200_PROFILING.md)"


def table_digest(o, k, v) -> str:
    import numpy as np

    h = hashlib.sha256()
    h.update(np.ascontiguousarray(o, dtype="<i8").tobytes())
    h.update(np.ascontiguousarray(k, dtype="i1").tobytes())
    h.update(np.ascontiguousarray(v, dtype="<i4").tobytes())
    return h.hexdigest()


def golden(cfg_idx):
    """The reference's digest of this configuration's table, if committed
    (tests/golden/large_cfg*.json, generated from oracle/_ref)."""
    p = os.path.join(ROOT, "tests", "golden", f"large_cfg{cfg_idx}.json")
    try:
        with open(p) as f:
            return json.load(f)
    except Exception:
        return None


FILL_KERNELS = {
    "tiles": "fill_tiles / fill_tiles_jobs1 (K1t budget tiles: one 32-slot tile per CTA, co-resident, "
             "or as a queue of tile jobs when the tiles outnumber the SMs, dominance-pruned open rows; "
             "the fused walk in the same launch)",
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
    """RANK / LOCAL_RANK / WORLD_SIZE from torchrun.  With fewer visible GPUs
    than ranks (a functional check of the N > 1 paths on one GPU), ranks share
    devices round-robin and the process group runs on gloo (NCCL refuses two
    ranks on one device); timing such a run says nothing about scaling."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch

        n = max(1, torch.cuda.device_count())
        if n < world:
            global PG_BACKEND
            PG_BACKEND = "gloo"
            local %= n
    return world, rank, local


PG_BACKEND = "nccl"


def init_pg(local):
    import torch
    import torch.distributed as dist

    if PG_BACKEND == "nccl":
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        dist.init_process_group("gloo")


def reduce_device(local):
    """Where max_over_ranks' tensor lives: the GPU for NCCL, the host for gloo."""
    return f"cuda:{local}" if PG_BACKEND == "nccl" else "cpu"


# ---------------------------------------------------------------------------
# roofline evidence: live L2 micro-benchmark + a live ncu pass over one fill
# ---------------------------------------------------------------------------
def l2_peak(device):
    """Best-of-10 L2 read bandwidth (GB/s) of an L2-resident 48 MiB buffer read
    with the fill's load flavour (ld.global.cg), 16 B and 4 B per lane
    (tools/l2probe.cu)."""
    path = os.path.join(ROOT, "tools", "libl2probe.so")
    try:
        lib = ctypes.CDLL(path)
        lib.l2probe_run.argtypes = [ctypes.c_int, ctypes.c_int64, ctypes.c_int, ctypes.c_int,
                                    ctypes.POINTER(ctypes.c_double)]
        out = {}
        for vec, key in ((1, "vec16_gbs"), (0, "vec4_gbs")):
            g = ctypes.c_double()
            rc = lib.l2probe_run(device, 48 << 20, 8, vec, ctypes.byref(g))
            out[key] = g.value if rc == 0 else None
        return out
    except Exception as e:  # pragma: no cover - the probe is built by build()
        return {"error": str(e)}


NCU_METRICS = ("gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum,"
               "smsp__issue_active.avg.pct_of_peak_sustained_active,sm__inst_executed.sum,"
               "sm__cycles_active.avg,sm__cycles_elapsed.avg,"
               "lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sectors_srcunit_tex_op_write.sum")


def ncu_probe_child(cfg_idx):
    """Child of ncu_pass: build the config's table and run 3 more fills (no
    walk); ncu captures the third fill launch."""
    from paper_2307_01236_b200 import rotor

    c = CONFIGS[cfg_idx]
    menu = rank_menu(cfg_idx, 0)
    with rotor.DpTable(menu, 1, c["M"]) as t:
        for _ in range(3):
            t.refill()
        t.sync()


def ncu_pass(cfg_idx, timeout=240):
    """DRAM and L2 bytes, issue-slot utilisation and warp instructions of ONE
    fill launch, measured by ncu on this box (cold caches, serialised; the
    counters, not the time, are what the roofline uses)."""
    ncu = shutil.which("ncu") or ("/usr/local/cuda/bin/ncu" if os.path.exists("/usr/local/cuda/bin/ncu")
                                  else None)
    if ncu is None:
        return {"error": "ncu not found"}
    log = tempfile.NamedTemporaryFile(suffix=".csv", delete=False).name
    cmd = [ncu, "--metrics", NCU_METRICS, "--clock-control", "none", "-k", "regex:fill_",
           "-s", "3", "-c", "1", "--csv", "--log-file", log, sys.executable,
           os.path.abspath(__file__), "--ncu-probe", "--config", str(cfg_idx)]
    from paper_2307_01236_b200 import rotor

    bits, rows = rotor._tuning.get()  # the same kernel variant as the timed run
    flags = [k for k, v in rotor.TUNE.items() if bits & v]
    if flags:
        cmd += ["--tune", ",".join(flags)]
    if rows:
        cmd += ["--tile-rows", str(rows)]
    try:
        r = subprocess.run(cmd, capture_output=True, text=True, timeout=timeout)
        import csv

        with open(log) as f:
            rows = [x for x in csv.reader(f) if len(x) > 10]
        if not rows:
            return {"error": "ncu produced no rows", "rc": r.returncode,
                    "stderr": (r.stderr or "")[-300:]}
        h = rows[0]
        out = {"kernel": None}
        for x in rows[1:]:
            d = dict(zip(h, x))
            out["kernel"] = d.get("Kernel Name", "")[:120]
            v = d.get("Metric Value", "").replace(",", "")
            try:
                out[d["Metric Name"]] = float(v)
            except ValueError:
                pass
        return out
    except Exception as e:
        return {"error": str(e)[:200]}
    finally:
        try:
            os.unlink(log)
        except OSError:
            pass


def roofline(fill_s, alg, nc, l2, peaks, peak_src, kern_desc, sm_mhz):
    """The fill's roofline: the binding of (L2 read bandwidth, SM issue rate),
    from ncu counters of one launch divided by the CUDA-event duration of the
    same launch; SURVEY 8(d)'s algorithmic-HBM fraction kept beside it."""
    hbm = float(peaks.get("hbm_gbs", FALLBACK_HBM_GBS))
    alg_ach = alg / fill_s / 1e9
    out = {"kernel": kern_desc, "fill_ms": fill_s * 1e3,
           "alg_hbm": {"achieved": alg_ach, "peak": hbm, "unit": "GB/s", "frac": alg_ach / hbm,
                       "alg_bytes_per_fill": alg, "peak_source": peak_src + " hbm_gbs",
                       "note": "SURVEY 8(d) algorithmic bytes (reference 8-byte cells) / event time"}}
    ok = nc and "lts__t_bytes.sum" in nc
    l2pk = (l2 or {}).get("vec16_gbs")
    if ok:
        traffic = nc.get("dram__bytes_read.sum", 0) + nc.get("dram__bytes_write.sum", 0)
        l2b = nc["lts__t_bytes.sum"]
        l2_ach = l2b / fill_s / 1e9
        inst = nc.get("sm__inst_executed.sum")
        sms = 148
        clk = (sm_mhz or float(peaks.get("sm_max_mhz", 1965.0))) * 1e6
        iss_ach = inst / fill_s / 1e9 if inst else None
        iss_pk = sms * 4 * clk / 1e9
        out["l2"] = {"achieved": l2_ach, "peak": l2pk, "unit": "GB/s",
                     "frac": (l2_ach / l2pk) if l2pk else None, "bytes_per_fill": l2b,
                     "peak_source": "live L2 read micro-benchmark (tools/l2probe.cu, 16 B/lane ld.cg)",
                     "peak_4B_lane": (l2 or {}).get("vec4_gbs")}
        out["issue"] = {"achieved": iss_ach, "peak": iss_pk, "unit": "G warp-inst/s",
                        "frac": iss_ach / iss_pk if iss_ach else None,
                        "issue_slots_busy_pct_active": nc.get(
                            "smsp__issue_active.avg.pct_of_peak_sustained_active"),
                        "warp_inst_per_fill": inst,
                        "sm_active_frac": (nc.get("sm__cycles_active.avg", 0) /
                                           nc["sm__cycles_elapsed.avg"]) if nc.get(
                            "sm__cycles_elapsed.avg") else None,
                        "peak_source": "148 SMs x 4 schedulers x SM clock under load"}
        cand = [("l2", out["l2"]), ("issue", out["issue"])]
        bound, b = max(cand, key=lambda kv: kv[1]["frac"] or 0.0)
        out.update({"bound": bound, "achieved": b["achieved"], "peak": b["peak"], "unit": b["unit"],
                    "frac": b["frac"], "traffic": traffic,
                    "traffic_source": "ncu (live pass over one fill launch of this run's config)",
                    "ncu_duration_ms": nc.get("gpu__time_duration.sum", 0) / 1e6})
    else:
        out.update({"bound": "hbm", "achieved": alg_ach, "peak": hbm, "unit": "GB/s",
                    "frac": alg_ach / hbm, "traffic": None, "peak_source": peak_src,
                    "ncu_error": (nc or {}).get("error", "ncu skipped"), "l2_probe": l2})
    return out


# ---------------------------------------------------------------------------
# reference arm (configs 1-3): remat::solve_chain on all host threads
# ---------------------------------------------------------------------------
def ref_sample(cfg_idx, menu, M):
    """(budget, units, m_top) of the reference arm's bounded sample: the same
    chain quantized to M / REF_SAMPLE budget slots through solve_chain's own
    `units` setting (identical candidate structure per cell)."""
    a0 = int(menu.act_sizes[0])
    budget = M + a0
    s = REF_SAMPLE.get(cfg_idx, 1)
    units = budget // s
    unit = -(-budget // units)
    m_top = budget // unit - (-(-a0 // unit))
    return budget, units, m_top


def reference_arm(args, world, rank):
    """The reference's own CPU solver (oracle/_ref: remat::solve_chain from the
    unmodified headers -- DpTable fill + build_schedule_rec, the same work as
    the device step) on this host's cores; rank 0 only."""
    if rank != 0:
        return
    from oracle.pyoracle import HAVE_REF, Orc, Ref

    c = CONFIGS[args.config]
    L, B, M = c["L"], c["B"], c["M"]
    menu = rank_menu(args.config, 0)
    threads = os.cpu_count() or 1
    budget, units, m_top = ref_sample(args.config, menu, M)
    cells = cells_of(L, m_top)
    if HAVE_REF:
        ref, kind = Ref(), "reference"

        def step():
            secs, st, *_ = ref.solve_bench(menu, budget, units, threads)
            assert st == 0
            return secs
    else:  # the C restatement, same algorithm, one solve per thread
        import concurrent.futures as cf
        kind = "port"
        orc = Orc()

        def step():
            t0 = time.perf_counter()
            with cf.ThreadPoolExecutor(threads) as ex:
                list(ex.map(lambda _: orc.solve_chain(menu, budget, units), range(threads)))
            return time.perf_counter() - t0

    for _ in range(args.warmup):
        step()
    times = [step() for _ in range(args.steps)]
    total = sum(times)
    value = threads * cells * args.steps / total
    sample = (f"each step = {threads} concurrent remat::solve_chain calls (one per host thread; the "
              f"reference solver is single-threaded, pipeline.hpp:58) on the config-{args.config} chain"
              + (f" quantized to m_top={m_top} budget slots (units={units}, 1/{REF_SAMPLE[args.config]} "
                 f"of M={M}; same candidates per cell)" if m_top != M else f" at full size (M={M})"))
    line = {
        "impl": "reference", "metric": METRIC,
        "value": value, "unit": "cells/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * total / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "int64",
        "data": "synthetic (SURVEY.md 8(d) splitmix64 generator)",
        "config": {"workload": workload_name(args.config), "L": L, "B": B, "M": M,
                   "sample_m_top": m_top},
        "cpu_baseline": {"value": value, "unit": "cells/s", "cores": threads, "kind": kind,
                         "sample": sample},
        "e2e": {"value": value, "unit": "cells/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def workload_name(cfg_idx):
    c = CONFIGS[cfg_idx]
    return (f"config{cfg_idx}: {c['name']} chain, L={c['L']} blocks, B={c['B']} options/block, "
            f"M={c['M']} budget slots; one full solve_chain (DP fill + schedule backtrack) per step")


def cpu_baseline_full(cfg_idx, menu, L, M):
    """The reference solve_chain at full size on 1 host thread (as it ships)."""
    from oracle.pyoracle import HAVE_REF, Orc, Ref

    a0 = int(menu.act_sizes[0])
    budget = M + a0
    if HAVE_REF:
        secs, st, ot, _, mt = Ref().solve_bench(menu, budget, budget, 1)
        kind = "reference"
    else:
        t0 = time.perf_counter()
        st, _, ot, _, mt, _ = Orc().solve_chain(menu, budget, budget)
        secs = time.perf_counter() - t0
        kind = "port"
    return {"value": cells_of(L, M) / secs, "unit": "cells/s", "cores": 1, "kind": kind,
            "sample": f"one full config-{cfg_idx} remat::solve_chain (L={L}, M={M}: fill + "
                      f"build_schedule_rec), 1 thread (the reference solver is single-threaded)",
            "seconds_per_solve": secs, "opt_time": ot}


# ---------------------------------------------------------------------------
# b200 arm, configs 1-3 at N=1 (and 1-2 as independent replicas at N>1)
# ---------------------------------------------------------------------------
def b200_arm(args, world, rank, local):
    import torch

    from paper_2307_01236_b200 import rotor

    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist
        init_pg(local)
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
        t = torch.tensor([x], dtype=torch.float64, device=reduce_device(local))
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
        # the same solve with every option scanned (RKR_TUNE_NO_PRUNE; the
        # mixed-width tile jobs of config 3 skip options dominated in open
        # rows, an exact reduction): reported beside the headline, not in it
        unpruned = None
        if world == 1 and args.config == 3:
            with rotor.tuning("no_prune"):
                t2 = rotor.DpTable(menu, 1, M, device=local, stream=stream.cuda_stream)
            for _ in range(args.warmup):
                t2.refill_walk(0, L - 1, M)
            uevs = [[torch.cuda.Event(enable_timing=True) for _ in range(2)] for _ in range(args.steps)]
            for i in range(args.steps):
                with torch.cuda.stream(stream):
                    flush.zero_()
                uevs[i][0].record(stream)
                t2.refill_walk(0, L - 1, M)
                uevs[i][1].record(stream)
            torch.cuda.synchronize()
            u_ops = t2.backtrack_fetch()
            u_top = t2.opt(0, L - 1, M)
            t2.close()
            u_ms = statistics.mean(e[0].elapsed_time(e[1]) for e in uevs)
            unpruned = {"solve_ms": u_ms, "schedule_equal": u_ops == ops_ref, "top_equal": None,
                        "_top": u_top,
                        "note": "same solve with every option scanned (RKR_TUNE_NO_PRUNE); the headline "
                                "skips options dominated in open rows (exact: identical tables, tested)"}
    fill_ms = [e[0].elapsed_time(e[1]) for e in kevs]
    step_ms = [e[0].elapsed_time(e[1]) for e in evs]
    assert ops == ops_ref
    top = table.opt(0, L - 1, M)
    if unpruned is not None:
        unpruned["top_equal"] = unpruned.pop("_top") == top
        assert unpruned["schedule_equal"] and unpruned["top_equal"]
    tot_s = max_over_ranks(sum(step_ms) / 1e3)
    fill_mean_s = statistics.mean(fill_ms) / 1e3

    # ---- end to end through the public API (host menu arrays) -------------------
    # one C-ABI call per step: rkr_solve_chain(host menu arrays) with budget =
    # M + a_0 bytes and units = budget (unit 1, m_top = M, i.e. exactly this
    # table); output buffers preallocated on the host, as a C caller would
    lib = rotor.lib()
    h2d = table.h2d_bytes()
    budget = M + int(menu.act_sizes[0])
    ms = menu.struct()
    ex = rotor._exec(local, "auto")
    cap = 1 << 16
    obuf = (rotor.RkrOp * cap)()
    n_, ot_, un_, mf_ = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
    mt_ = ctypes.c_int32()
    e2e_times = []
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
        table.close()
        return
    clocks = sampler.summary()
    kern = table.kernel()
    parity = None
    g = golden(args.config)
    if g is not None and world == 1:
        # the timed table IS the reference's table (every cell, sha256)
        o, k, v = table.download()
        parity = {"table_sha256_equals_reference": table_digest(o, k, v) == g["digest"],
                  "source": f"tests/golden/large_cfg{args.config}.json (oracle/_ref, unmodified "
                            f"reference solver)"}
        del o, k, v
        table._host = None
    table.close()
    del flush
    torch.cuda.empty_cache()
    peaks, peak_src = measured_peaks()
    l2 = l2_peak(local) if world == 1 else None
    nc = ncu_pass(args.config) if (world == 1 and not args.no_ncu) else {"error": "ncu skipped"}
    line = {
        "metric": METRIC,
        "value": world * cells * args.steps / tot_s,
        "unit": "cells/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": 1e3 * tot_s / args.steps,
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "int64 (stored as u32, overflow-proven)",
        "data": "synthetic (SURVEY.md 8(d) splitmix64 generator"
                + ("; one independent chain per rank)" if world > 1 else ")"),
        "config": {
            "workload": workload_name(args.config),
            "L": L, "B": B, "M": M, "cells_per_solve": cells,
            "candidates_per_solve": candidates_of(L, B, M),
            "l2": "flushed between timed steps (256 MiB write, outside the events)",
            "parallelism": f"instances x{world} (no data-path collective)" if world > 1 else "1 GPU",
            "solve_ms": 1e3 * tot_s / args.steps,
            "top_opt": top,
            "note": "the per-menu cell programs (prep_programs) are built when the table is "
                    "created and reused by every refill of the same menu; e2e rebuilds them",
        },
        "e2e": {"value": world * cells * args.steps / e2e_s, "unit": "cells/s",
                "h2d_bytes_per_step": h2d * world, "d2h_bytes_per_step": d2h * world,
                "ms_per_step": 1e3 * e2e_s / args.steps,
                "path": "rkr_solve_chain(host menu arrays): quantize, H2D, fill, top cell, "
                        "device backtrack, D2H of the schedule"},
        # per step: the fill (one launch, or L for the per-diagonal kernel) and
        # the walk (fused into the budget-tile fill, its own launch otherwise)
        "gpu_launches": args.steps * ((L if kern == "diagonal" else 1) + (0 if kern == "tiles" else 1)),
        "roofline": roofline(fill_mean_s, alg_bytes(L, M), nc, l2, peaks, peak_src,
                             FILL_KERNELS[kern], clocks.get("sm_mhz")),
        "clocks": clocks,
    }
    if parity is not None:
        line["parity"] = parity
    if unpruned is not None:
        line["unpruned"] = unpruned
    if world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline_full(args.config, menu, L, M)
        line["cpu_baseline"]["opt_time_equals_device"] = line["cpu_baseline"].pop("opt_time") == top
    print(json.dumps(line), flush=True)


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
        init_pg(local)
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
        t = torch.tensor([x], dtype=torch.float64, device=reduce_device(local))
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

    # end to end: one rkr_sweep_chains C-ABI call (every chain's budgets in
    # one batch; the reference runs cmd_sweep once per chain, results are
    # identical): fill, top cells, schedules, min-feasible search; schedules
    # copied back into caller buffers preallocated as a C caller would
    lib = rotor.lib()
    by_chain = {}
    for _, ci, b, _, _ in rows:
        by_chain.setdefault(ci, []).append(b)
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
    cells_total = sweep_cells(menus, rows_all)
    # parity of this rank's results against the reference's (large_cfg4.json)
    g = golden(4)
    par = None
    if g is not None:
        want = {(e["chain"], e["budget"]): e for e in g["instances"]}
        bad, i = 0, 0
        for ci in chains:
            for b in by_chain[ci]:
                e = want.get((ci, b))
                if e is None or (e["status"] == 0) != (st_[i] == 0) or (
                        e["status"] == 0 and e["opt_time"] != ot_[i]) or (
                        e["status"] == 2 and e["min_feasible"] != mf_[i]):
                    bad += 1
                i += 1
        par = {"instances_checked": n, "mismatches": bad,
               "source": "tests/golden/large_cfg4.json (oracle/_ref solve_chain per instance)"}
    if rank != 0:
        return
    peaks, peak_src = measured_peaks()
    ab = sweep_alg_bytes(menus, rows)
    achieved = ab / (statistics.mean(fill_ms) / 1e3) / 1e9
    hbm = float(peaks.get("hbm_gbs", FALLBACK_HBM_GBS))
    line = {
        "metric": METRIC_SWEEP,
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
                "feasible_budgets_rank0": n_feas, "infeasible_budgets_rank0": n - n_feas},
        "gpu_launches": args.steps,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s",
                     "frac": achieved / hbm, "traffic": None,
                     "kernel": ("fill_tiles_batch (K1t jobs: persistent CTAs take (table, budget tile) "
                                "jobs, every table in one launch)" if kern == "tiles" else
                                "fill_persistent (K1p, every table in one launch)"),
                     "alg_bytes_per_fill": ab, "fill_ms": statistics.mean(fill_ms),
                     "peak_source": peak_src + " hbm_gbs (algorithmic bytes, SURVEY 8(d))"},
        "clocks": sampler.summary(),
    }
    if par is not None:
        line["parity_rank0"] = par
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
        "impl": "reference", "metric": METRIC_SWEEP,
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
# budget-axis sharding across ranks (one shard per GPU): config 3 at N > 1,
# config 5 (its 256/64/4096 twin at N = 1)
# ---------------------------------------------------------------------------
def b200_arm_sharded(args, world, rank, local):
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_2307_01236_b200 import rotor

    torch.cuda.set_device(local)
    if world > 1:
        init_pg(local)
    cfg = args.config
    c = CONFIGS[cfg]
    L, B, M = c["L"], c["B"], c["M"]
    twin = cfg == 5 and world == 1  # the full config-5 table (206 GB) needs >= 2 GPUs
    if twin:
        L, B, M = 256, 64, 4096
    seed = 47 if cfg == 5 else 42 + cfg
    menu = synthetic_menu(L, B, M, seed=seed)

    def gather(obj):
        if world == 1:
            return [obj]
        out = [None] * world
        dist.all_gather_object(out, obj)
        return out

    def barrier():
        if world > 1:
            dist.barrier()

    def max_over_ranks(x):
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=reduce_device(local))
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    sh = rotor.ProcessShard(menu, 1, M, world, rank, device=local)
    handles, infos = rotor.link_process_shards(sh, gather)
    stream = torch.cuda.ExternalStream(sh.table.stream(), device=f"cuda:{local}")
    lo, hi = sh.range()

    def fill(ev=None, wev=None):
        sh.zero()
        barrier()
        if ev:
            ev[0].record(stream)
        sh.launch()
        if ev:
            ev[1].record(stream)
        sh.sync()
        barrier()
        ops = None
        if rank == 0:  # the cross-shard walk from the top cell (peer reads)
            if wev:
                wev[0].record(stream)
            ops = sh.backtrack(handles, infos, 0, L - 1, M)
            if wev:
                wev[1].record(stream)
        return ops

    sampler = ClockSampler(local)
    with sampler:
        for _ in range(args.warmup):
            fill()
        evs = [[torch.cuda.Event(enable_timing=True) for _ in range(2)] for _ in range(args.steps)]
        wevs = [[torch.cuda.Event(enable_timing=True) for _ in range(2)] for _ in range(args.steps)]
        for i in range(args.steps):
            ops = fill(evs[i], wevs[i])
        torch.cuda.synchronize()
    fill_s = max_over_ranks(sum(e[0].elapsed_time(e[1]) for e in evs) / 1e3)
    walk_s = sum(e[0].elapsed_time(e[1]) for e in wevs) / 1e3 if rank == 0 else 0.0
    walk_s = max_over_ranks(walk_s)
    tot_s = fill_s + walk_s
    shard_kern = sh.table.kernel()

    # cross-shard check: every shard's columns against an unsharded solve of
    # the same chain on rank 0's GPU (and that against the reference digest)
    mine = sh.table.download()
    my_dig = table_digest(*mine)
    del mine
    sh.table._host = None
    digs = gather((lo, hi, my_dig))
    check = None
    if rank == 0:
        with rotor.DpTable(menu, 1, M, device=local) as t:
            o, k, v = t.download()
            ok = all(table_digest(np.ascontiguousarray(o[:, a:b]), np.ascontiguousarray(k[:, a:b]),
                                  np.ascontiguousarray(v[:, a:b])) == d for a, b, d in digs)
            g = golden(3) if cfg == 3 else (golden("5twin") if twin else None)
            ref_ok = (table_digest(o, k, v) == g["digest"]) if g else None
            del o, k, v
            t._host = None
            check = {"shard_columns_equal_unsharded": ok, "schedule_equal_unsharded":
                     ops == t.backtrack(0, L - 1, M), "unsharded_equals_reference": ref_ok,
                     "shards": [[a, b] for a, b, _ in digs]}

    # end to end through the public API: every rank builds its shard from the
    # host menu (H2D), shards exchange IPC handles and link, fill, rank 0 walks
    # and copies the schedule back
    sh.close()
    e2e = []
    h2d = 0
    for it in range(args.warmup + args.steps):
        torch.cuda.synchronize()
        barrier()
        t0 = time.perf_counter()
        s2 = rotor.ProcessShard(menu, 1, M, world, rank, device=local)
        hs, ins = rotor.link_process_shards(s2, gather)
        s2.zero()
        barrier()
        s2.launch()
        s2.sync()
        barrier()
        if rank == 0:
            s2.backtrack(hs, ins, 0, L - 1, M)
        dt = time.perf_counter() - t0
        h2d = s2.table.h2d_bytes()
        s2.close()
        if it >= args.warmup:
            e2e.append(dt)
    e2e_s = max_over_ranks(sum(e2e))
    h2d_all = sum(gather(h2d))
    if rank == 0:
        peaks, peak_src = measured_peaks()
        cells = cells_of(L, M)
        ab = alg_bytes(L, M)
        hbm = float(peaks.get("hbm_gbs", FALLBACK_HBM_GBS))
        per_fill = fill_s / args.steps
        line = {
            "metric": METRIC if cfg == 3 else METRIC_SHARDED,
            "value": cells * args.steps / tot_s, "unit": "cells/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot_s / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "int64 (stored as u32, overflow-proven)",
            "data": "synthetic (SURVEY.md 8(d) generator)",
            "config": {"workload": (workload_name(cfg) if cfg == 3 else
                                    f"config5{'-twin' if twin else ''}: L={L}, B={B}, M={M}")
                       + f"; budget axis in {world} shard(s), one per GPU, halo pushed in-kernel "
                         f"over peer memory, rank 0 walks across the shards",
                       "L": L, "B": B, "M": M, "shard0_range": [lo, hi],
                       "fill_ms": 1e3 * per_fill, "walk_ms": 1e3 * walk_s / args.steps,
                       "schedule_ops": len(ops or [])},
            "e2e": {"value": cells * args.steps / e2e_s, "unit": "cells/s",
                    "h2d_bytes_per_step": h2d_all, "d2h_bytes_per_step": 12 * len(ops or []) + 32,
                    "ms_per_step": 1e3 * e2e_s / args.steps,
                    "path": "per rank rkr_shard_create (host menu) + IPC link + fill; rank 0 "
                            "rkr_shard_backtrack, schedule copied back"},
            "gpu_launches": args.steps * (world + 1),
            "roofline": {"bound": "hbm", "achieved": ab / per_fill / 1e9 / world, "peak": hbm,
                         "unit": "GB/s", "frac": ab / per_fill / 1e9 / world / hbm, "traffic": None,
                         "kernel": (FILL_KERNELS[shard_kern] if shard_kern != "tiles" else
                                    "fill_tiles_batch (K1t budget-shard tile jobs)")
                                   + ", one launch per shard per step; halo pushed in-kernel",
                         "alg_bytes_per_fill": ab,
                         "peak_source": peak_src + " hbm_gbs per GPU (algorithmic bytes)"},
            "clocks": sampler.summary(),
            "shard_check": check,
        }
        print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", type=int, default=3, choices=[1, 2, 3, 4, 5])
    ap.add_argument("--no-cpu-baseline", action="store_true", help="skip the CPU leg (tuning runs)")
    ap.add_argument("--no-ncu", action="store_true", help="skip the live ncu counter pass")
    ap.add_argument("--ncu-probe", action="store_true", help=argparse.SUPPRESS)
    ap.add_argument("--tune", default="", help="A/B: comma-separated rkr_exec.tune flags (rotor.TUNE)")
    ap.add_argument("--tile-rows", type=int, default=0, help="A/B: K1t rows per warp (0 = auto)")
    args = ap.parse_args()
    if args.tune or args.tile_rows:
        from paper_2307_01236_b200 import rotor
        flags = [f for f in args.tune.split(",") if f]
        with rotor.tuning(*flags, tile_rows=args.tile_rows):
            return run(args)
    return run(args)


def run(args):
    if args.ncu_probe:
        ncu_probe_child(args.config)
        return
    args.warmup = max(args.warmup, 3) if args.impl == "b200" else args.warmup
    world, rank, local = dist_setup()
    if args.config == 4:
        if args.impl == "reference":
            reference_arm_sweep(args, world, rank)
        else:
            b200_arm_sweep(args, world, rank, local)
    elif args.impl == "reference":
        if args.config == 5:
            if rank == 0:
                print(json.dumps({"impl": "reference", "metric": METRIC_SHARDED, "unavailable":
                                  "config 5 needs ~550 GB / ~107 h on the reference CPU solver"}))
            return
        reference_arm(args, world, rank)
    elif args.config == 5 or (args.config == 3 and world > 1):
        b200_arm_sharded(args, world, rank, local)
    else:
        b200_arm(args, world, rank, local)


if __name__ == "__main__":
    main()
