"""In-tree build of librkr.so (sm_100a) and the C++ API test program.

    python -m paper_2307_01236_b200.build
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "librkr.so")
SOURCES = [os.path.join(CSRC, f) for f in ("rkr_kernels.cu", "rkr_persist.cu", "rkr_tiles.cu",
                                            "rkr_table.cu", "rkr_batch.cu", "rkr_shard.cu",
                                            "rkr_replay.cu")]
DEPS = SOURCES + [os.path.join(CSRC, h) for h in ("rkr_internal.h", "rkr_host.h", "rkr_walk.cuh")] + [
    os.path.join(ROOT, "include", "rkr.h")]

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-lineinfo", "-O3", "-std=c++17",
    "-Xcompiler", "-fPIC,-O2",
    "-shared",
]


def _stale(target: str, deps) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def build_lib(force: bool = False, verbose: bool = False) -> str:
    if force or _stale(LIB, DEPS):
        cmd = ["nvcc", *NVCC_FLAGS, "-o", LIB + ".tmp", *SOURCES]
        if verbose:
            cmd.insert(1, "-Xptxas=-v")
        subprocess.run(cmd, check=True)
        os.replace(LIB + ".tmp", LIB)
    return LIB


PROBE_SRC = os.path.join(ROOT, "tools", "l2probe.cu")
PROBE_LIB = os.path.join(ROOT, "tools", "libl2probe.so")


def build_probe(force: bool = False) -> str:
    """tools/libl2probe.so: the L2 read-bandwidth micro-benchmark bench.py's
    roofline uses (measurement infrastructure, not the solver)."""
    if force or _stale(PROBE_LIB, [PROBE_SRC]):
        subprocess.run(["nvcc", *NVCC_FLAGS, "-o", PROBE_LIB + ".tmp", PROBE_SRC], check=True)
        os.replace(PROBE_LIB + ".tmp", PROBE_LIB)
    return PROBE_LIB


CPP_TEST_SRC = os.path.join(ROOT, "tests", "cpp", "test_chain_dp_b200.cpp")
CPP_TEST_BIN = os.path.join(ROOT, "tests", "cpp", "test_chain_dp_b200")


def build_cpp_tests(force: bool = False) -> str:
    hdrs = [os.path.join(ROOT, "include", "remat_b200", f) for f in
            ("chain_dp.hpp", "types.hpp", "errors.hpp", "device_error.hpp")]
    hdrs.append(os.path.join(ROOT, "include", "remat", "chain_dp.hpp"))
    if force or _stale(CPP_TEST_BIN, [CPP_TEST_SRC, LIB, *hdrs]):
        subprocess.run(
            ["g++", "-std=c++20", "-O1", "-I", os.path.join(ROOT, "include"), CPP_TEST_SRC,
             "-o", CPP_TEST_BIN, "-L", HERE, "-lrkr",
             "-Wl,-rpath,$ORIGIN/../../paper_2307_01236_b200"],
            check=True)
    return CPP_TEST_BIN


if __name__ == "__main__":
    build_lib(force="--force" in sys.argv, verbose="-v" in sys.argv)
    build_cpp_tests(force="--force" in sys.argv)
    build_probe(force="--force" in sys.argv)
    print(LIB)
